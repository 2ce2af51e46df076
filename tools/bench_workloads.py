"""Secondary workloads of BASELINE.json (the headline bench is bench.py, config 3):

  --workload config2   batch of 256 blocks at 128^2 and at 512^2 (mixed Wishart /
                       spectrum-controlled, kappa(A_hat) ~ 1e6): root + residual check
  --workload config4   32000 x 1024 embedding: blocked one-sided statistics (32 row
                       blocks, R_b^{-1/2}) + D fallback for the vocab dim; variant
                       "unblocked": one R with K = 32000 (block size 32768)
  --workload resnet50  f3: ResNet-50 tensors of order 1..4 (HWIO conv
                       kernels, fc, BN vectors), block 1024: per-mode statistics,
                       roots (p = 2k'), mode-product preconditioning

Every phase is timed with CUDA events on the launching stream after warm-up;
prints one JSON line per workload (no oracle on the timed path).

    python tools/bench_workloads.py --workload config2 [--steps 3 --warmup 2]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2002_09018_b200 as shp  # noqa: E402
import synth  # noqa: E402


MODE = {"auto": "auto", "auto7": "auto7", "auto6": "auto6", "fp64": None, "ozaki": "ozaki", "ozaki7": "ozaki7",
        "ozaki6": "ozaki6", "hybrid": -1}


def timed(fn, steps, warmup, stream):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.mean(ts))


def config2(args, dev, stream):
    out = {"workload": "config2_batch256", "results": []}
    for n in (128, 512):
        A = torch.empty((256, n, n), dtype=torch.float32, device=dev)
        A[0::2] = synth.wishart_batch_device(n, 128, synth.BASE_SEED + 2 + n, dev)
        A[1::2] = torch.from_numpy(synth.psd_batch(n, 2, synth.BASE_SEED + 2 + n, "spectrum")).to(dev).repeat(64, 1, 1)
        X = torch.empty_like(A)
        info = shp.new_info(256, dev)
        t_root = timed(lambda: shp.inverse_pth_root_batched(A, 4, X=X, info=info, fp64_iters=MODE[args.root_precision]),
                       args.steps, args.warmup, stream)
        res_box = {}

        def resid():
            res_box["r"] = shp.root_residual_batched(A, X, 4, info)
        t_res = timed(resid, args.steps, args.warmup, stream)
        inf = shp.info_to_numpy(info)
        r = res_box["r"].cpu().numpy()
        iters = inf["iters"].astype(np.float64)
        flops = float(iters.sum()) * 4 * n * n * (n + 1) + 256 * 100 * 2.0 * n * n
        out["results"].append({
            "n": n, "batch": 256, "root_ms": t_root, "roots_per_s": 256 / (t_root * 1e-3),
            "root_tflops_sym": flops / (t_root * 1e-3) / 1e12, "residual_ms": t_res,
            "iters_mean": float(iters.mean()), "status_counts": {str(k): int((inf["status"] == k).sum()) for k in range(4)},
            "residual_over_sqrt_n_max": float(r.max() / np.sqrt(n)),
            "residual_note": "||X^p A_hat - I||_F of the stored fp32 root (dominated by its fp32 rounding)"})
    return out


def config4(args, dev, stream):
    out = {"workload": "config4_embedding_32000x1024", "results": []}
    G = synth.vocab_gradient_device(synth.VOCAB, synth.D_MODEL, synth.BASE_SEED + 4, dev)
    for variant, block in (("blocked_b1024", 1024), ("unblocked_K32000", 32768)):
        plan = shp.make_plan([tuple(G.shape)], block, 8192, 1)
        D = torch.zeros_like(G)
        P = torch.zeros_like(G)
        table = shp.TensorTable([G], [D], [P])
        stats = torch.zeros(plan.stats_elems, dtype=torch.float32, device=dev)
        roots = torch.zeros_like(stats)
        gn = torch.zeros(plan.n_blocks, dtype=torch.float64, device=dev)
        sc = torch.zeros(plan.n_blocks, dtype=torch.float32, device=dev)
        for _ in range(8):
            shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
        t_stats = timed(lambda: shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn), args.steps, args.warmup,
                        stream)
        box = {}

        def roots_fn():
            box["i"] = shp.refresh_group_roots(plan, stats, roots, 0, fp64_iters=MODE[args.root_precision])
        t_roots = timed(roots_fn, args.steps, args.warmup, stream)
        t_prec = timed(lambda: shp.precondition(table, plan, roots, gn, sc), args.steps, args.warmup, stream)
        iters = np.concatenate([shp.info_to_numpy(i)["iters"] for _, i in box["i"]])
        K = sum(int(b["rows"]) for b in plan.blocks)
        out["results"].append({
            "variant": variant, "blocks": plan.n_blocks, "roots_p2": int(sum(int(g["count"]) for g in plan.groups)),
            "stats_ms": t_stats, "stats_tflops_sym": 1024.0 * 1025 * K / (t_stats * 1e-3) / 1e12,
            "roots_ms": t_roots, "precondition_ms": t_prec, "iters_mean": float(iters.mean())})
    return out


def resnet50(args, dev, stream):
    named = synth.resnet50_shapes()
    shapes = [s for _, s in named]
    plan = shp.make_tensor_plan(shapes, args.block_size, 8192, 1)
    Gs = [torch.from_numpy(synth.conv_gradient(s, synth.BASE_SEED + 26 + i)).to(dev) for i, s in enumerate(shapes)]
    Ds = [torch.zeros_like(G) for G in Gs]
    Ps = [torch.zeros_like(G) for G in Gs]
    table = shp.TTensorTable(Gs, Ds, Ps)
    stats = torch.zeros(plan.stats_elems, dtype=torch.float32, device=dev)
    roots = torch.zeros_like(stats)
    nb = plan.n_blocks
    gn = torch.zeros(nb, dtype=torch.float64, device=dev)
    sc = torch.zeros(nb, dtype=torch.float32, device=dev)
    for _ in range(8):
        shp.tensor_stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
    t_stats = timed(lambda: shp.tensor_stats_update(table, plan, stats, 1.0, 1.0, -1, gn), args.steps, args.warmup,
                    stream)
    box = {}

    def roots_fn():
        box["i"] = shp.refresh_group_roots(plan, stats, roots, 0, fp64_iters=MODE[args.root_precision])
    t_roots = timed(roots_fn, args.steps, args.warmup, stream)
    t_prec = timed(lambda: shp.tensor_precondition(table, plan, roots, gn, sc), args.steps, args.warmup, stream)
    iters = np.concatenate([shp.info_to_numpy(i)["iters"] for _, i in box["i"]])
    status = np.concatenate([shp.info_to_numpy(i)["status"] for _, i in box["i"]])
    # algorithmic work: statistic e(e+1) K per kept mode (symmetric-minimal); mode products 2 e numel
    st_fl = pr_fl = 0.0
    for b in plan.blocks:
        numel = int(np.prod(b["extent"]))
        for i in range(int(b["order"])):
            if b["p"][i]:
                e = int(b["extent"][i])
                st_fl += float(e) * (e + 1) * (numel // e)  # symmetric-minimal
                pr_fl += 2.0 * e * numel
    groups = {}
    for g in plan.groups:
        key = f"p{int(g['p'])}"
        groups[key] = groups.get(key, 0) + int(g["count"])
    return {"workload": f"resnet50_b{args.block_size}", "tensors": len(shapes),
            "params": int(sum(int(np.prod(s)) for s in shapes)), "blocks": nb, "roots": groups,
            "stats_ms": t_stats, "stats_tflops_sym": st_fl / (t_stats * 1e-3) / 1e12,
            "roots_ms": t_roots, "precondition_ms": t_prec, "precondition_tflops": pr_fl / (t_prec * 1e-3) / 1e12,
            "shampoo_step_ms": t_stats + t_prec, "amortized_step_ms_kappa500": t_stats + t_prec + t_roots / 500,
            "iters_mean": float(iters.mean()), "status_counts": {str(k): int((status == k).sum()) for k in range(4)}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", required=True, choices=["config2", "config4", "resnet50"])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--block-size", type=int, default=1024)
    ap.add_argument("--root-precision", default="auto", choices=sorted(MODE))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    fn = {"config2": config2, "config4": config4, "resnet50": resnet50}[args.workload]
    out = fn(args, dev, stream)
    out.update({"steps": args.steps, "warmup": args.warmup, "data": "synthetic", "gpu": torch.cuda.get_device_name(),
                "root_precision": args.root_precision})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
