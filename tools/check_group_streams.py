"""The bench's two root calls (528 p = 4 and 96 p = 2 roots of 1024^2, Transformer-Big statistics) one after the
other on one stream, against the p = 2 call on a second stream concurrent with the p = 4 call: is there idle GPU
time the second call can fill?  Prints both times (CUDA events, best of --reps) and whether the roots are
bit-identical.

    python tools/check_group_streams.py [--reps 3]
"""

import argparse
import json
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
Gs = []
for i, (m, n) in enumerate(shapes):
    seed = synth.BASE_SEED + 3 + i
    Gs.append(synth.vocab_gradient_device(m, n, seed, dev) if m == synth.VOCAB
              else synth.lowrank_gradient_device(m, n, seed, dev))
table = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs])
plan = shp.make_plan(shapes, 1024, 8192, 1)
stats = torch.zeros(plan.stats_elems, device=dev)
for _ in range(4):
    shp.stats_update(table, plan, stats, 1.0, 1.0, -1)
groups = list(range(len(plan.groups)))
subs = [shp.Plan(plan.shapes, plan.block_size, plan.max_precond_dim, 1, plan.blocks, plan.groups[g:g + 1],
                 plan.stats_elems, plan.segment_elems) for g in groups]
main = torch.cuda.current_stream()
side = torch.cuda.Stream(device=dev)


def serial(out):
    shp.refresh_group_roots(plan, stats, out, 0, fp64_iters="auto")


def concurrent(out):
    ev = torch.cuda.Event()
    ev.record(main)
    side.wait_event(ev)
    # the largest group on the main stream, the others on the side stream
    order = sorted(groups, key=lambda g: -int(plan.groups[g]["count"]) * int(plan.groups[g]["n"]) ** 3)
    shp.refresh_group_roots(subs[order[0]], stats, out, 0, fp64_iters="auto", stream=main)
    with torch.cuda.stream(side):
        for g in order[1:]:
            shp.refresh_group_roots(subs[g], stats, out, 0, fp64_iters="auto", stream=side)
    done = torch.cuda.Event()
    done.record(side)
    main.wait_event(done)


res = {}
outs = {}
for name, fn in (("serial", serial), ("concurrent", concurrent), ("serial2", serial)):
    out = torch.zeros_like(stats)
    fn(out)  # warm-up (workspaces)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        fn(out)
        e1.record(main)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[name] = best
    outs[name] = out
print(json.dumps({"groups": [(int(g["n"]), int(g["p"]), int(g["count"])) for g in plan.groups], "ms": res,
                  "bit_identical": bool(torch.equal(outs["serial"], outs["concurrent"]))}), flush=True)
