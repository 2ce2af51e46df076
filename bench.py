"""bench.py -- the hot path of distributed Shampoo on B200, one JSON line.

Roots run in the "auto" precision by default: the Ozaki root (every Newton
product on the INT8 tensor cores with exact int32 accumulation of 7-slice
splits, fp64-level accuracy) for blocks of n >= 512 (all of
this workload), FP64 DMMA below; --root-precision fp64 / ozaki / ozaki6 / hybrid force one
(auto6: 6 slices for n >= 512).

Workload (BASELINE.json configs[2], the configuration the metric is quoted on):
Transformer-Big (99 matrix parameters, 375.1M of P:494's 375.4M), block size
1024, max_precond_dim 8192 -> 360 blocks, 528 inverse-4th roots + 96
inverse-square roots of 1024^2 statistics.  One STEP = the whole hot path:
  a2 statistics (owned blocks) + D + graft numerator
  a3-a6 root refresh of every owned statistic (power iteration + coupled Newton)
  a7 NCCL all-gather of the packed roots (N > 1)
  a8-a9 preconditioned gradient + graft scale for every block.
value = inverse-4th-roots of 1024^2 blocks completed per second of step time
(whole job, all ranks; the step time also contains everything else above).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "inverse-4th-roots/sec @1024² blocks (1/2/4/8 B200); Shampoo step ms, Transformer-Big"
UNIT = "roots/s"
BLOCK = 1024
MAX_PRECOND = 8192
KAPPA_REFRESH = 500  # root refresh interval of the paper's Transformer runs
FP64_DMMA_PEAK_TFLOPS = 37.1  # measured: tools/microbench/fp64_pipes.cu (profiles/r01_fp64_pipes.txt)
# dram__bytes_read.sum + dram__bytes_write.sum of root_kernel per 1024^2 p=4 matrix (20 iterations), from the
# ncu --set full capture in profiles/r01_ncu_root_kernel.txt (148-matrix launch: 323.6 GB)
ROOT_TRAFFIC_BYTES_PER_MATRIX = (191.679e9 + 128.690e9) / 148  # profiles/root_r01h_ncu_summary.txt
def _int8_peak():
    """int8 dense peak = 2 x the measured bf16 peak of MEASURED_PEAKS.json (nominal int8:bf16 ratio 2).  The
    Ozaki GEMM launches run inside a ~1 s step, so the SUSTAINED bf16 figure is the denominator (B200_PROFILING:
    burst for a kernel timed alone, sustained for a kernel inside a long step); fallback: the burst figure
    measured on this pool earlier (1687.1), then NVIDIA's nominal 4.5 POPS."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        if mp.get("bf16_tflops_sustained"):
            return 2 * float(mp["bf16_tflops_sustained"]), "sustained", 2 * float(mp.get("bf16_tflops") or 0) or None
        if mp.get("bf16_tflops"):
            return 2 * float(mp["bf16_tflops"]), "burst", 2 * float(mp["bf16_tflops"])
    except (OSError, ValueError):
        pass
    return 2 * 1687.1, "burst (earlier measurement; MEASURED_PEAKS.json absent)", 2 * 1687.1
# dram read + write per Ozaki GEMM launch per 1024^2 matrix: the mean over the four product launches of one S = 5
# iteration (the schedule's majority: 55 of the 88 GEMM launches of a 528-root call), from the ncu --set full capture
# of the final kernel with tiled planes (profiles/r02/r02zb_ncu_gemm5_full_tiled_summary.txt, 148 matrices): X T
# 2.751 GB, T T sliced 1.515 GB, T^2 T^2 sliced 1.518 GB, T^4 M 2.764 GB -> 18.6 / 10.2 / 10.3 / 18.7 MB per matrix =
# the algorithmic planes + output (18 / 10 / 10 / 18 MB: no re-reads).  S = 7 launches move 22.8 / 14.4 / 14.4 / 22.8
# MB (r02a_ncu_gemm7_full_summary.txt).
OZAKI_TRAFFIC_BYTES_PER_MATRIX_STAGE = (2.751 + 1.515 + 1.518 + 2.764) / 4 * 1e9 / 148
# the arithmetic of the dominant phase (the roots): fp64 iterates, products per the root precision
DTYPE = {"auto": "f64 iterates, int8 Ozaki products S=7..5 per iteration (exact int32 accumulation)",
         "auto7": "f64 iterates, int8 Ozaki S=7 products (exact int32 accumulation)",
         "auto6": "f64 iterates, int8 Ozaki S=6 products (exact int32 accumulation)",
         "ozaki": "f64 iterates, int8 Ozaki products S=7..5 per iteration (exact int32 accumulation)",
         "ozaki7": "f64 iterates, int8 Ozaki S=7 products (exact int32 accumulation)",
         "ozaki6": "f64 iterates, int8 Ozaki S=6 products (exact int32 accumulation)",
         "fp64": "f64 (FP64 DMMA)", "hybrid": "f64 DMMA, then 3xTF32 (tf32 tcgen05) tail"}
EMPTY_LAUNCH_MS = 0.05  # an Ozaki GEMM launch with no active matrix returns in a few microseconds
ROOT_MODE = {"auto": "auto", "auto7": "auto7", "auto6": "auto6", "fp64": None, "ozaki": "ozaki", "ozaki7": "ozaki7",
             "ozaki6": "ozaki6", "hybrid": -1}
# (max slices, scheduled?) of the Ozaki modes
ROOT_SLICES = {"auto": (7, True), "auto7": (7, False), "auto6": (6, False), "ozaki": (7, True), "ozaki7": (7, False),
               "ozaki6": (6, False)}
ROOT_LABEL = {"auto": "auto: ozaki (INT8 tcgen05, per-iteration slice schedule 7..5 of reading #29, exact int32 "
                      "accumulation) for n >= 512, fp64 DMMA below",
              "auto7": "auto7: ozaki (INT8 tcgen05, 7 slices, exact int32 accumulation) for n >= 512, fp64 DMMA below",
              "auto6": "auto6: ozaki (INT8 tcgen05, 6 slices, exact int32 accumulation) for n >= 512, fp64 DMMA below",
              "fp64": "fp64 DMMA", "ozaki": "ozaki: INT8 tcgen05, slice schedule 7..5, exact int32 accumulation",
              "ozaki7": "ozaki7: INT8 tcgen05, 7 slices, exact int32 accumulation",
              "ozaki6": "ozaki6: INT8 tcgen05, 6 slices, exact int32 accumulation",
              "hybrid": "hybrid fp64 DMMA -> 3xTF32 tcgen05 (auto switch)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tol", type=float, default=1e-7)
    ap.add_argument("--block-size", type=int, default=BLOCK,
                    help="config 5 sweep (128..4096); the metric is quoted at 1024")
    ap.add_argument("--max-precond-dim", type=int, default=MAX_PRECOND)
    ap.add_argument("--root-precision", default="auto", choices=sorted(ROOT_MODE),
                    help="auto: ozaki for n >= 512, fp64 below; fp64: FP64 DMMA; ozaki: INT8 tensor cores "
                         "with fp64-level accuracy (7 slices, §6.3c); ozaki6 / auto6: 6 slices (21 slice "
                         "products, roots ~3e-5 from the fp64 oracle, reading #27); "
                         "hybrid: FP64 DMMA then a 3xTF32 tcgen05 tail (§6.3b)")
    ap.add_argument("--hybrid", action="store_true", help="alias of --root-precision hybrid")
    ap.add_argument("--shard", default="layers", choices=["layers", "roots"],
                    help="N > 1: layers -- whole tensors per rank (their statistics, roots and P; one all-gather of P "
                         "per step, reading #30); roots -- every root LPT-assigned on its own, the roots all-gathered "
                         "and every rank preconditioning every block")
    ap.add_argument("--gather", default="allgather", choices=["overlapped", "allgather"],
                    help="N > 1: one all_gather_into_tensor after all roots (default), or per-group owner broadcasts "
                         "overlapping the next group's roots (measured equal at N = 2, 4: DESIGN §8)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _cpu_warm(_):
    from oracle import root  # noqa: F401


def _cpu_root(seed: int):
    import time as _t

    from oracle import root as oroot
    A = synth.wishart(BLOCK, seed).astype(np.float64)
    t0 = _t.perf_counter()
    _, info = oroot.inverse_pth_root(A, 4)
    return _t.perf_counter() - t0, info.iters


def oracle_root_baseline(seconds: float = 15.0, n: int = 1024):
    """The CPU fp64 oracle (as it stands) on a bounded sample of the workload, one independent 1024^2 root per host
    core (one BLAS thread each) -- the paper's "distributed to all CPU cores available" (
    BASELINE.md §3).  Rounds of `cores` roots until ~`seconds` have passed."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    old = {v: os.environ.get(v) for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
    for v in old:
        os.environ[v] = "1"  # inherited by the spawned workers before they import numpy
    try:
        with mp.get_context("spawn").Pool(cores) as pool:
            pool.map(_cpu_warm, range(cores))  # worker imports outside the timed sample
            t0 = time.perf_counter()
            done, iters, rnd = 0, [], 0
            while True:
                res = pool.map(_cpu_root, [synth.BASE_SEED + 2 + rnd * cores + i for i in range(cores)])
                done += cores
                iters += [r[1] for r in res]
                rnd += 1
                if time.perf_counter() - t0 >= seconds or rnd >= 4:
                    break
            dt = time.perf_counter() - t0
    finally:
        for v, x in old.items():
            if x is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = x
    return {"value": done / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{done} inverse-4th-roots of {n}^2 Wishart statistics (kappa~1e6), numpy fp64 coupled Newton, "
                      f"one root per core ({cores} processes x 1 BLAS thread), {np.mean(iters):.0f} iterations, "
                      f"{dt:.1f} s"}


# ------------------------------------------------------------------ reference arm

def run_reference(args):
    """The reference arm for this tier: the fp64 oracle, as it stands, on the box's host cores -- every step one
    round of independent 1024^2 inverse-4th-roots of the workload's kind, one per core (the paper's roots "distributed
    to all CPU cores"), a bounded sample of the Transformer-Big refresh.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"  # inherited by the spawned workers before they import numpy
    samples, iters = [], []
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_cpu_warm, range(cores))
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_root, [synth.BASE_SEED + 2 + i * cores + q for q in range(cores)])
            if i >= args.warmup:
                samples.append(time.perf_counter() - t0)
                iters += [r[1] for r in res]
    t = float(np.mean(samples))
    value = cores / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"transformer_big_b{BLOCK}_full_step",
                       "step": f"bounded sample: {cores} independent {BLOCK}^2 inverse-4th-roots (Wishart, kappa~1e6), "
                               "one per host core", "block_size": BLOCK},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{cores} x {args.steps} roots of {BLOCK}^2, one per core (1 BLAS thread each), "
                                       f"{np.mean(iters):.0f} iterations"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def main():
    args = parse()
    if args.hybrid:
        args.root_precision = "hybrid"
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2002_09018_b200 as shp
    from paper_2002_09018_b200 import dist as sdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    names_shapes = synth.transformer_big_shapes()
    shapes = [s for _, s in names_shapes]
    B = args.block_size
    layers = args.shard == "layers"
    plan = shp.make_plan(shapes, B, args.max_precond_dim, world, owners="tensor" if layers else "root")
    n_p4 = int(sum((plan.blocks["p_left"] == 4).sum() + (plan.blocks["p_right"] == 4).sum() for _ in [0]))
    # gradients (device), vocab tensors row-sparse (Zipf ids), others low-rank + noise
    Gs = []
    for i, (name, (m, n)) in enumerate(names_shapes):
        seed = synth.BASE_SEED + 3 + i
        if m == synth.VOCAB:
            Gs.append(synth.vocab_gradient_device(m, n, seed, dev))
        else:
            Gs.append(synth.lowrank_gradient_device(m, n, seed, dev))
    Ds = [torch.zeros_like(G) for G in Gs]
    nb = plan.n_blocks
    if layers:
        # whole tensors per rank: statistics, D, graft numerator, roots and P of this rank's tensors only; every
        # P (and graft scale) in one flat buffer of equal rank segments -> one all-gather per step
        ls = sdist.LayerShards(plan, world)
        mine = ls.sub[rank]
        flatP = torch.zeros(ls.numel, dtype=torch.float32, device=dev)
        Ps = ls.p_views(flatP)
        gnum = torch.zeros(max(1, mine.n_blocks), dtype=torch.float64, device=dev)
        gscale = ls.scales_of(flatP, rank)
        stats_plan, only = mine, -1
        seg = slice(rank * plan.segment_elems, (rank + 1) * plan.segment_elems)
    else:
        Ps = [torch.zeros_like(G) for G in Gs]
        gnum = torch.zeros(nb, dtype=torch.float64, device=dev)
        gscale = torch.zeros(nb, dtype=torch.float32, device=dev)
        stats_plan, only = plan, (rank if world > 1 else -1)
        seg = slice(0, plan.stats_elems)
    table = shp.TensorTable(Gs, Ds, Ps)
    stats = torch.zeros(plan.stats_elems, dtype=torch.float32, device=dev)
    roots = torch.zeros_like(stats)
    roots_lo = torch.zeros_like(stats)
    # statistics accumulated over 8 steps before the timed refreshes (config 3 recipe)
    for _ in range(8):
        shp.stats_update(table, stats_plan, stats, 1.0, 1.0, only, gnum)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    launches = [0]

    def step(ev=None, tbl=None, before_stats=None, after_stats=None, before_precond=None, after_precond=None):
        tbl = table if tbl is None else tbl
        if before_stats:
            before_stats()
        if ev:
            ev[0].record(stream)
        shp.stats_update(tbl, stats_plan, stats, 1.0, 1.0, only, gnum)
        if after_stats:
            after_stats()
        launches[0] += shp.last_launch_count()
        if ev:
            ev[1].record(stream)
        if world > 1 and args.gather == "overlapped" and not layers:
            # each group's roots go out (NCCL broadcasts from their owners) while the next group computes
            infos, nl = sdist.refresh_gather_overlapped(plan, stats, roots, rank, world, tol=args.tol,
                                                        fp64_iters=ROOT_MODE[args.root_precision])
            launches[0] += nl
            if ev:
                ev[2].record(stream)
        else:
            infos = shp.refresh_group_roots(plan, stats, roots, rank, tol=args.tol,
                                            fp64_iters=ROOT_MODE[args.root_precision])
            launches[0] += shp.last_refresh_launch_count()
            if ev:
                ev[2].record(stream)
            if not layers:
                sdist.all_gather_roots(plan, roots, rank, world)
        # once per refresh: the roots' TF32 remainder for the tensor cores (layers: this rank's segment only)
        shp.tf32_split(roots[seg], roots_lo[seg])
        launches[0] += 1
        if ev:
            ev[3].record(stream)
        if before_precond:
            before_precond()
        shp.precondition(tbl, stats_plan, roots, gnum, gscale, roots_lo=roots_lo)
        launches[0] += shp.last_launch_count()
        if ev:
            ev[4].record(stream)
        if layers:
            ls.gather(flatP, rank)  # every rank's P and graft scales (one NCCL all-gather of equal segments)
        if ev:
            ev[5].record(stream)
        if after_precond:
            after_precond()
        return infos

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # timed region: barrier + sync on both sides, CUDA events on the launching stream
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    # per-group root launch timing (the dominant kernel) on the same stream
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches[0] = 0
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    all_infos = []
    for k in range(args.steps):
        all_infos.append(step(evs[k]))
    end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = start.elapsed_time(end)
    phase = np.array([[evs[k][i].elapsed_time(evs[k][i + 1]) for i in range(5)] for k in range(args.steps)])
    t_local = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms = float(t_local.item())
    ms_per_step = total_ms / args.steps

    # dominant kernel: the p=4 root launch (one cooperative kernel per call), timed alone on the stream
    g4 = sorted([g for g in plan.groups_of(rank) if int(g["p"]) == 4], key=lambda g: -int(g["count"]) * int(g["n"]) ** 3)
    roof = None
    iters_mean = None
    slices, scheduled = ROOT_SLICES.get(args.root_precision, (None, False))
    if g4 and slices and (args.root_precision.startswith("ozaki") or int(g4[0]["n"]) >= shp.OZAKI_MIN_N):
        # the INT8 GEMM dominates: every launch bracketed by CUDA events on its stream
        g = g4[0]
        cnt, off, stride = int(g["count"]), int(g["offset"]), int(g["stride"])
        gn_ = int(g["n"])
        gld = (gn_ + 3) // 4 * 4
        info = shp.new_info(cnt, dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        shp.profile_begin()
        e0.record(stream)
        shp.inverse_pth_root_ptr(stats.data_ptr() + 4 * off, gld, stride, roots.data_ptr() + 4 * off, gld, stride,
                                 cnt, gn_, 4, info, tol=args.tol, device=dev,
                                 fp64_iters="ozaki" if scheduled else f"ozaki{slices}")
        e1.record(stream)
        torch.cuda.synchronize()
        gemm_ms, gemm_launches = shp.profile_end("ozaki_gemm")
        rk_ms, _ = shp.profile_end("root_kernel")
        per_launch = shp.profile_launch_ms("ozaki_gemm")
        # launches after every matrix of the batch converged return at once (a few us): the per-launch figure
        # is taken over the launches that did work
        working = per_launch[per_launch > EMPTY_LAUNCH_MS]
        call_ms = e0.elapsed_time(e1)
        inf = shp.info_to_numpy(info)
        iters_mean = float(inf["iters"].sum()) / cnt
        n = gn_
        # algorithmic int8 ops: per symmetric product S(S+1)/2 slice products of n^2 (n+1) (upper triangle incl.
        # diagonal, 2 ops per multiply-add), 4 products per iteration, S per iteration from the library's schedule
        ops = shp.ozaki_int8_ops(inf["iters"], n, 4, 1e-6, None if scheduled else 0.0, slices)
        achieved = ops / (gemm_ms * 1e-3) / 1e12
        peak, peak_kind, peak_burst = _int8_peak()
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS (int8)",
                "frac": achieved / peak, "traffic": OZAKI_TRAFFIC_BYTES_PER_MATRIX_STAGE * cnt,
                "traffic_note": "dram read+write bytes per GEMM launch (mean of the 4 product launches of an "
                                "S = 5 iteration, the schedule's majority), ncu --set full of the same kernel (148 "
                                "matrices, r02zb) scaled to this batch: the algorithmic planes + output, no re-reads",
                "kernel": f"oz::gemm_kernel (INT8 tcgen05 Ozaki products, batch {cnt} x {n}^2, p=4)",
                "kernel_ms": float(working.mean()) if working.size else None,
                "kernel_launches": int(working.size), "kernel_launches_total": gemm_launches,
                "kernel_ms_empty_launches_total": float(per_launch[per_launch <= EMPTY_LAUNCH_MS].sum()),
                "ops_per_launch": ops / max(1, int(working.size)),
                "root_call_ms": call_ms, "gemm_share_of_root_call": gemm_ms / call_ms,
                "root_kernel_ms_power_iteration_and_setup": rk_ms,
                "fp64_equivalent_tflops": (float(inf["iters"].sum()) * 4 * n * n * (n + 1)
                                           + cnt * 100 * 2.0 * n * n) / (call_ms * 1e-3) / 1e12,
                "peak_source": f"int8 dense = 2 x the {peak_kind} bf16 TF/s of MEASURED_PEAKS.json (nominal "
                               f"int8:bf16 ratio 2; NVIDIA nominal 4.5 POPS)", "slices": slices, "slice_schedule": [shp.ozaki_iteration_slices(k, 4, n, 1e-6, None if scheduled else 0.0, slices)
                                                        for k in range(int(inf["iters"].max()))],
                "frac_vs_burst_peak": (achieved / peak_burst) if peak_burst else None,
                "peak_note": "the sustained bf16 figure was measured at ~1290 MHz under a bf16 GEMM's power draw; "
                             "this int8 kernel runs at ~1550-1650 MHz under the cap, and at b >= 2048 exceeds the "
                             "sustained-derived figure (profiles/r01z_block_sweep.jsonl) -- frac_vs_burst_peak is "
                             "the stricter bound"}
    elif g4:
        g = g4[0]
        cnt, off, stride = int(g["count"]), int(g["offset"]), int(g["stride"])
        info = shp.new_info(cnt, dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gn_ = int(g["n"])
        gld = (gn_ + 3) // 4 * 4
        shp.inverse_pth_root_ptr(stats.data_ptr() + 4 * off, gld, stride, roots.data_ptr() + 4 * off, gld, stride,
                                 cnt, gn_, 4, info, tol=args.tol, device=dev)
        e1.record(stream)
        torch.cuda.synchronize()
        kms = e0.elapsed_time(e1)
        inf = shp.info_to_numpy(info)
        iters_mean = float(inf["iters"].mean())
        n = gn_
        # algorithmic flops: 4 symmetric products per iteration, n^2 (n+1) flops each (upper triangle
        # incl. diagonal x 2n), + the power iteration (100 x 2 n^2)
        flops = float(inf["iters"].sum()) * 4 * n * n * (n + 1) + cnt * 100 * 2.0 * n * n
        achieved = flops / (kms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_DMMA_PEAK_TFLOPS,
                "traffic": ROOT_TRAFFIC_BYTES_PER_MATRIX * cnt if n == 1024 else None,
                "traffic_note": "bytes per launch, ncu capture of the same kernel (148 matrices) scaled per matrix",
                "kernel": f"root_kernel (FP64 DMMA coupled Newton, batch {cnt} x {n}^2, p=4)",
                "kernel_ms": kms, "flops_per_launch": flops,
                "peak_source": "FP64 DMMA.8x8x4 peak measured on this pool's B200 by tools/microbench/fp64_pipes.cu "
                               "(MEASURED_PEAKS.json has no FP64 entry)"}

    # every root of every timed step: status / iteration histograms (a status-2 root leaves X untouched and
    # status 1 did not reach tol -- the line says how many of the counted roots are which)
    st_hist, it_hist = {}, {}
    for infos in all_infos:
        for _, info in infos:
            a = shp.info_to_numpy(info)
            for v in a["status"]:
                st_hist[int(v)] = st_hist.get(int(v), 0) + 1
            for v in a["iters"]:
                it_hist[int(v)] = it_hist.get(int(v), 0) + 1
    n_p4_total = n_p4  # every p=4 root of the plan is computed once per step (owner-sharded)
    value = n_p4_total / (ms_per_step * 1e-3)

    # e2e: through the public API with host buffers (pinned), every step's H2D of the gradients and D2H of P and
    # the graft scales inside the timed region, on a copy stream: the gradients of step k+1 land in a second
    # device buffer while step k's roots run (the refresh reads only the statistics), P_k leaves while step
    # k+1 runs (its preconditioning waits for that copy) -- a prefetching input pipeline, no copy skipped
    e2e = None
    if not args.no_e2e:
        hostG = [torch.empty(G.shape, dtype=torch.float32, pin_memory=True) for G in Gs]
        for h, G in zip(hostG, Gs):
            h.copy_(G)
        if layers:  # every P and graft scale in one flat buffer: one D2H copy
            hostP = [torch.empty(flatP.shape, dtype=torch.float32, pin_memory=True)]
            hscale = None
        else:
            hostP = [torch.empty(P.shape, dtype=torch.float32, pin_memory=True) for P in Ps]
            hscale = torch.empty(nb, dtype=torch.float32, pin_memory=True)
        Gs2 = [torch.empty_like(G) for G in Gs]
        tables = [table, shp.TensorTable(Gs2, Ds, Ps)]
        bufs = [Gs, Gs2]
        copy = torch.cuda.Stream(device=dev)
        ev_h2d = [torch.cuda.Event() for _ in range(args.steps)]
        ev_pre = [torch.cuda.Event() for _ in range(args.steps)]
        ev_d2h = [torch.cuda.Event() for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)

        def h2d(k):
            with torch.cuda.stream(copy):
                copy.wait_event(s0)
                if k >= 2:
                    copy.wait_event(ev_pre[k - 2])  # buffer k % 2 last read by step k-2's preconditioning
                for h, G in zip(hostG, bufs[k % 2]):
                    G.copy_(h, non_blocking=True)
                ev_h2d[k].record(copy)

        def d2h(k):
            with torch.cuda.stream(copy):
                copy.wait_event(ev_pre[k])
                for h, P in zip(hostP, [flatP] if layers else Ps):
                    h.copy_(P, non_blocking=True)
                if hscale is not None:
                    hscale.copy_(gscale, non_blocking=True)
                ev_d2h[k].record(copy)

        h2d(0)
        for k in range(args.steps):
            step(tbl=tables[k % 2],
                 before_stats=lambda k=k: stream.wait_event(ev_h2d[k]),
                 after_stats=(lambda k=k: h2d(k + 1)) if k + 1 < args.steps else None,
                 before_precond=(lambda k=k: stream.wait_event(ev_d2h[k - 1])) if k >= 1 else None,
                 after_precond=lambda k=k: (ev_pre[k].record(stream), d2h(k)))
        stream.wait_event(ev_d2h[args.steps - 1])
        s1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([s0.elapsed_time(s1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item()) / args.steps
        bi = sum(G.numel() * 4 for G in Gs)
        bo = flatP.numel() * 4 if layers else sum(P.numel() * 4 for P in Ps) + nb * 4
        e2e = {"value": n_p4_total / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo, "ms_per_step": e2e_ms}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = oracle_root_baseline()
        ph = phase.mean(axis=0)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": DTYPE[args.root_precision], "data": "synthetic",
            "config": {"workload": f"transformer_big_b{B}_full_step", "model": "Transformer-Big (P:494) shapes",
                       "block_size": B, "max_precond_dim": args.max_precond_dim, "blocks": nb,
                       "roots_p4": n_p4_total, "roots_p2": int(sum(int(g["count"]) for g in plan.groups if int(g["p"]) == 2)),
                       "eps_rel": 1e-6, "tol": args.tol, "power_iters": 100,
                       "parallelism": (f"layer-shard{world}" if layers else f"root-shard{world}"),
                       "root_exchange": ("none: whole tensors per rank, one all_gather_into_tensor of P + graft "
                                         "scales per step" if layers else
                                         ("per-group owner broadcasts overlapping the next group's roots "
                                          "(phase 'roots' includes them)") if args.gather == "overlapped"
                                         else "one all_gather_into_tensor of the roots") if world > 1 else None,
                       "root_precision": ROOT_LABEL[args.root_precision], "l2": "inputs larger than L2 (stats 2.6 GB, roots 2.6 GB, G 1.5 GB)"},
            "phase_ms": {"stats": ph[0], "roots": ph[1], "root_allgather_and_split": ph[2], "precondition": ph[3],
                         "p_allgather": ph[4]},
            "shampoo_step_ms": ph[0] + ph[3] + ph[4],
            "amortized_step_ms_kappa500": ph[0] + ph[3] + ph[4] + (ph[1] + ph[2]) / KAPPA_REFRESH,
            "root_phase_roots_per_s": n_p4_total / (ph[1] * 1e-3),
            "newton_iters_mean": iters_mean,
            "root_status_hist": {str(k): v for k, v in sorted(st_hist.items())},
            "root_iters_hist": {str(k): v for k, v in sorted(it_hist.items())},
            "roots_failed": st_hist.get(2, 0) + st_hist.get(3, 0),
            "gpu_launches": launches[0],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
