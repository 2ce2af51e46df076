"""f1 measurement: Transformer-Big Shampoo steps with the delayed, amortised root
refresh (kappa = 500 as in the paper's runs) -- step ms while a refresh is
in flight vs the plain step (statistics + preconditioning) and vs a synchronous
refresh every step.  One JSON line.

    python tools/bench_delayed.py [--kappa 500] [--steps 20]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_09018_b200 as shp  # noqa: E402
import synth  # noqa: E402
from paper_2002_09018_b200.schedule import DelayedRefresh  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kappa", type=int, default=500)
ap.add_argument("--steps", type=int, default=20)
args = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = [s for _, s in synth.transformer_big_shapes()]
plan = shp.make_plan(shapes, 1024, 8192, 1)
Gs = [synth.lowrank_gradient_device(m, n, synth.BASE_SEED + 3 + i, dev) for i, (m, n) in enumerate(shapes)]
Ps = [torch.zeros_like(G) for G in Gs]
table = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs], Ps)
stats = torch.zeros(plan.stats_elems, device=dev)
roots = torch.zeros_like(stats)
gn = torch.zeros(plan.n_blocks, dtype=torch.float64, device=dev)
sc = torch.zeros(plan.n_blocks, device=dev)
for _ in range(8):
    shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
shp.refresh_group_roots(plan, stats, roots, 0)  # bootstrap roots
dr = DelayedRefresh(plan, stats, roots, kappa=args.kappa)


def timed(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for t in range(n):
        fn(t)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


roots_lo = shp.tf32_split(roots)


def plain(t):
    shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
    shp.precondition(table, plan, roots, gn, sc, roots_lo=roots_lo)


def delayed(t):
    shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
    dr.step(t)
    shp.precondition(table, plan, dr.current, gn, sc, roots_lo=dr.current_lo)


def synchronous(t):
    shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
    shp.refresh_group_roots(plan, stats, roots, 0)
    shp.tf32_split(roots, roots_lo)
    shp.precondition(table, plan, roots, gn, sc, roots_lo=roots_lo)


for fn in (plain, delayed):
    timed(fn, 3)  # warm-up
dr = DelayedRefresh(plan, stats, roots, kappa=args.kappa)
ms_plain = timed(plain, args.steps)
ms_delayed = timed(delayed, args.steps)  # steps 0..steps-1 of a kappa window: every one carries a chunk
ms_sync = timed(synchronous, 2)
chunk = dr.chunk
print(json.dumps({"f1": "delayed amortised refresh", "kappa": args.kappa, "roots_per_step_chunk": chunk,
                  "step_ms_plain": ms_plain, "step_ms_with_refresh_chunk": ms_delayed,
                  "step_ms_synchronous_refresh": ms_sync,
                  "refresh_overhead_per_step_ms": ms_delayed - ms_plain,
                  "amortised_refresh_ms_if_spread_evenly": (ms_sync - ms_plain) / args.kappa}))
