"""Run the Transformer-Big preconditioned-gradient call (config 3, b = 1024) on
random symmetric roots, for timing / ncu.   python tools/profile_precondition.py [--reps 3]"""

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
Ps = [torch.zeros_like(G) for G in Gs]
table = shp.TensorTable(Gs, [torch.ones_like(G) for G in Gs], Ps)
roots = torch.randn(plan.stats_elems, device=dev) * 0.03
gn = torch.ones(plan.n_blocks, dtype=torch.float64, device=dev)
sc = torch.zeros(plan.n_blocks, device=dev)
for r in range(args.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    shp.precondition(table, plan, roots, gn, sc)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
flops = 0
for b in plan.blocks:
    r, c = int(b["rows"]), int(b["cols"])
    if b["p_left"]:
        flops += 2 * r * r * c
    if b["p_right"]:
        flops += 2 * r * c * c
print(f"precondition: {ms:.3f} ms, {flops / 1e9:.0f} GF algorithmic (dense), {flops / ms / 1e9:.1f} TFLOP/s, "
      f"launches {shp.last_launch_count()}")
