"""Run the Transformer-Big statistics call (config 3, b = 1024, all 624 L/R) for
timing / ncu.   python tools/profile_stats.py [--reps 3]"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_09018_b200 as shp  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = [s for _, s in synth.transformer_big_shapes()]
plan = shp.make_plan(shapes, 1024, 8192, 1)
Gs = [synth.lowrank_gradient_device(m, n, 7 + i, dev) for i, (m, n) in enumerate(shapes)]
table = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs])
stats = torch.zeros(plan.stats_elems, device=dev)
gn = torch.zeros(plan.n_blocks, dtype=torch.float64, device=dev)
for r in range(args.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
flops = 0
for b in plan.blocks:
    r, c = int(b["rows"]), int(b["cols"])
    if b["p_left"]:
        flops += r * (r + 1) * c
    if b["p_right"]:
        flops += c * (c + 1) * r
print(f"stats: {ms:.3f} ms, {flops / 1e9:.0f} GF algorithmic (symmetric-minimal), {flops / ms / 1e9:.1f} TFLOP/s, "
      f"launches {shp.last_launch_count()}")
