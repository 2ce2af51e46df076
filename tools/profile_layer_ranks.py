"""Per-rank root time of a layer-granular plan, measured on ONE GPU (no collectives): for W ranks, every rank's
owned (n, p) groups are refreshed in turn with CUDA events around each batched call -- the balance of the plan
and the per-call fixed costs (power iteration, launches) that stop the roots phase from shrinking as 1/W.

    python tools/profile_layer_ranks.py [--world 4 8] [--owners tensor root]
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
ap.add_argument("--world", type=int, nargs="+", default=[1, 4, 8])
ap.add_argument("--owners", nargs="+", default=["tensor"])
args = ap.parse_args()
dev = torch.device("cuda", 0)
names_shapes = synth.transformer_big_shapes()
shapes = [s for _, s in names_shapes]
Gs = []
for i, (m, n) in enumerate(shapes):  # bench.py's gradient recipe
    seed = synth.BASE_SEED + 3 + i
    Gs.append(synth.vocab_gradient_device(m, n, seed, dev) if m == synth.VOCAB
              else synth.lowrank_gradient_device(m, n, seed, dev))
table = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs])
for owners in args.owners:
    for W in args.world:
        plan = shp.make_plan(shapes, 1024, 8192, W, owners=owners)
        stats = torch.zeros(plan.stats_elems, device=dev)
        roots = torch.zeros_like(stats)
        for _ in range(8):
            shp.stats_update(table, plan, stats, 1.0, 1.0, -1)
        shp.refresh_group_roots(plan, stats, roots, 0, fp64_iters="auto")  # warm-up
        torch.cuda.synchronize()
        ranks = []
        for r in range(W):
            calls = []
            for gi in range(len(plan.groups)):
                g = plan.groups[gi]
                if int(g["owner"]) != r:
                    continue
                one = shp.Plan(plan.shapes, plan.block_size, plan.max_precond_dim, W, plan.blocks,
                               plan.groups[gi:gi + 1], plan.stats_elems, plan.segment_elems)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                shp.refresh_group_roots(one, stats, roots, r, fp64_iters="auto")
                e1.record()
                torch.cuda.synchronize()
                calls.append({"n": int(g["n"]), "p": int(g["p"]), "count": int(g["count"]),
                              "ms": e0.elapsed_time(e1)})
            ranks.append({"rank": r, "roots": sum(c["count"] for c in calls), "ms": sum(c["ms"] for c in calls),
                          "calls": calls})
        tot = sum(x["ms"] for x in ranks)
        print(json.dumps({"owners": owners, "world": W, "max_rank_ms": max(x["ms"] for x in ranks),
                          "ideal_ms": tot / W, "balance": tot / W / max(x["ms"] for x in ranks),
                          "ranks": ranks}), flush=True)
