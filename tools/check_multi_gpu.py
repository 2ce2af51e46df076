"""Multi-GPU check of row e (run under torchrun, NCCL): owner-sharded statistics +
roots + all-gather must give roots bit-identical to a single-GPU computation.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tools/check_multi_gpu.py [--root-precision auto|fp64|ozaki|ozaki6]

--root-precision defaults to "auto", the bench's path (INT8 Ozaki root for n >= 512).
"""

import argparse

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2002_09018_b200 as shp  # noqa: E402
import synth  # noqa: E402
from paper_2002_09018_b200 import dist as sdist  # noqa: E402


MODES = {"auto": "auto", "auto6": "auto6", "fp64": None, "ozaki": "ozaki", "ozaki6": "ozaki6"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--root-precision", default="auto", choices=sorted(MODES))
    ap.add_argument("--full", action="store_true", help="the whole Transformer-Big plan (bench.py's workload)")
    ap.add_argument("--shard", default="roots", choices=["roots", "layers"],
                    help="roots: gathered roots vs 1 GPU; layers: whole tensors per rank, gathered P vs 1 GPU")
    args = ap.parse_args()
    mode = MODES[args.root_precision]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    shapes = [s for _, s in synth.transformer_big_shapes()]
    if not args.full:
        shapes = shapes[3:40]  # attention + FFN blocks (no vocab)
    Gs = [synth.lowrank_gradient_device(m, n, synth.BASE_SEED + 3 + i, dev) for i, (m, n) in enumerate(shapes)]
    if args.shard == "layers":
        return check_layers(args, rank, world, dev, shapes, Gs, mode)
    table = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs])
    # sharded
    plan = shp.make_plan(shapes, 1024, 8192, world)
    stats = torch.zeros(plan.stats_elems, device=dev)
    roots = torch.zeros_like(stats)
    for _ in range(2):
        shp.stats_update(table, plan, stats, 1.0, 1.0, rank)
    sdist.refresh_roots(plan, stats, roots, rank, world, fp64_iters=mode)
    torch.cuda.synchronize()
    # single-GPU reference on every rank (same kernels, whole plan)
    plan1 = shp.make_plan(shapes, 1024, 8192, 1)
    table1 = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs])
    stats1 = torch.zeros(plan1.stats_elems, device=dev)
    roots1 = torch.zeros_like(stats1)
    for _ in range(2):
        shp.stats_update(table1, plan1, stats1, 1.0, 1.0, -1)
    shp.refresh_group_roots(plan1, stats1, roots1, 0, fp64_iters=mode)
    torch.cuda.synchronize()
    bad = 0
    for b, b1 in zip(plan.blocks, plan1.blocks):
        for side in ("left", "right"):
            if b[f"p_{side}"]:
                n = int(b["rows"] if side == "left" else b["cols"])
                ld = int(b[f"{side}_ld"])
                o, o1 = int(b[f"{side}_off"]), int(b1[f"{side}_off"])
                if not torch.equal(roots[o:o + n * ld], roots1[o1:o1 + n * ld]):
                    bad += 1
    t = torch.tensor([bad], device=dev)
    dist.all_reduce(t)
    if rank == 0:
        n_roots = int((plan.blocks["p_left"] > 0).sum() + (plan.blocks["p_right"] > 0).sum())
        print(f"world {world}, root precision {args.root_precision} ({mode}), {len(shapes)} tensors: {n_roots} roots, mismatching (summed over ranks) = {int(t.item())}", flush=True)
    dist.destroy_process_group()
    if int(t.item()) != 0:
        raise SystemExit(1)


def check_layers(args, rank, world, dev, shapes, Gs, mode):
    """Layer-granular step (reading #30): each rank its tensors' statistics, roots and P, one all-gather of P;
    every gathered P (and graft scale) must equal the single-GPU step's bit for bit."""
    plan = shp.make_plan(shapes, 1024, 8192, world, owners="tensor")
    ls = sdist.LayerShards(plan, world)
    mine = ls.sub[rank]
    flat = torch.zeros(ls.numel, device=dev)
    Ds = [torch.zeros_like(G) for G in Gs]
    table = shp.TensorTable(Gs, Ds, ls.p_views(flat))
    stats = torch.zeros(plan.stats_elems, device=dev)
    roots = torch.zeros_like(stats)
    gn = torch.zeros(max(1, mine.n_blocks), dtype=torch.float64, device=dev)
    for _ in range(2):
        shp.stats_update(table, mine, stats, 1.0, 1.0, -1, gn)
    shp.refresh_group_roots(plan, stats, roots, rank, fp64_iters=mode)
    shp.precondition(table, mine, roots, gn, ls.scales_of(flat, rank), roots_lo=shp.tf32_split(roots))
    ls.gather(flat, rank)
    sc = torch.zeros(plan.n_blocks, device=dev)
    ls.unpack_scales(flat, sc)
    torch.cuda.synchronize()
    # single-GPU reference on every rank
    plan1 = shp.make_plan(shapes, 1024, 8192, 1)
    P1 = [torch.zeros_like(G) for G in Gs]
    table1 = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs], P1)
    stats1 = torch.zeros(plan1.stats_elems, device=dev)
    roots1 = torch.zeros_like(stats1)
    gn1 = torch.zeros(plan1.n_blocks, dtype=torch.float64, device=dev)
    sc1 = torch.zeros(plan1.n_blocks, device=dev)
    for _ in range(2):
        shp.stats_update(table1, plan1, stats1, 1.0, 1.0, -1, gn1)
    shp.refresh_group_roots(plan1, stats1, roots1, 0, fp64_iters=mode)
    shp.precondition(table1, plan1, roots1, gn1, sc1, roots_lo=shp.tf32_split(roots1))
    torch.cuda.synchronize()
    bad = sum(int(not torch.equal(a, b)) for a, b in zip(ls.p_views(flat), P1)) + int(not torch.equal(sc, sc1))
    t = torch.tensor([bad], device=dev)
    dist.all_reduce(t)
    if rank == 0:
        loads = [sum(int(g["count"]) for g in plan.groups_of(r)) for r in range(world)]
        print(f"world {world}, layers, root precision {args.root_precision}, {len(shapes)} tensors, roots per rank "
              f"{loads}: tensors with a differing P or scale array (summed over ranks) = {int(t.item())}", flush=True)
    dist.destroy_process_group()
    if int(t.item()) != 0:
        raise SystemExit(1)


if __name__ == "__main__":
    main()
