"""Robustness of the root kernels when they share the GPU with the training step (f1's setting).

A batch of Ozaki roots runs on one stream while the Shampoo step's kernels (statistics: DMMA; preconditioning:
tcgen05 3xTF32) run in a loop on another; the roots must be bit-identical to the same call made alone, with the
same statuses.  Stream priorities are varied: with a higher-priority training stream the GPU may preempt the
running root kernels (compute preemption) -- the case the delayed refresh relies on.

    python tools/check_concurrency.py [--batch 32] [--trials 4] [--work both|stats|precondition]
Prints one JSON line per (priority setting, work) and exits 1 on any mismatch.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2002_09018_b200 as shp  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--trials", type=int, default=4)
ap.add_argument("--loops", type=int, default=40)
ap.add_argument("--precision", default="ozaki")
ap.add_argument("--works", default="both,stats,precondition")
ap.add_argument("--settings", default="hi_lo,equal,lo_hi")
args = ap.parse_args()
dev = torch.device("cuda", 0)
A = synth.wishart_batch_device(args.n, args.batch, synth.BASE_SEED + 2, dev)
X_ref, info_ref = shp.inverse_pth_root_batched(A, 4, fp64_iters=args.precision)
torch.cuda.synchronize()
inf_ref = shp.info_to_numpy(info_ref)

# the training step's kernels on a slice of Transformer-Big
shapes = [s for _, s in synth.transformer_big_shapes()][3:27]
plan = shp.make_plan(shapes, 1024, 8192, 1)
Gs = [synth.lowrank_gradient_device(m, n, synth.BASE_SEED + 3 + i, dev) for i, (m, n) in enumerate(shapes)]
Ps = [torch.zeros_like(G) for G in Gs]
table = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs], Ps)
stats = torch.zeros(plan.stats_elems, device=dev)
gn = torch.zeros(plan.n_blocks, dtype=torch.float64, device=dev)
sc = torch.zeros(plan.n_blocks, device=dev)
shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
roots = torch.zeros_like(stats)
shp.refresh_group_roots(plan, stats, roots, 0, fp64_iters="auto")
roots_lo = shp.tf32_split(roots)
torch.cuda.synchronize()

lo, hi = torch.cuda.Stream.priority_range()
bad_total = 0
for setting in args.settings.split(","):
    pr, pt = {"hi_lo": (lo, hi), "equal": (0, 0), "lo_hi": (hi, lo)}[setting]
    rs = torch.cuda.Stream(device=dev, priority=pr)
    ts = torch.cuda.Stream(device=dev, priority=pt)
    for work in args.works.split(","):
        mism, st_hist, max_rel = 0, {}, 0.0
        for trial in range(args.trials):
            torch.cuda.synchronize()
            with torch.cuda.stream(ts):
                # the training stream starts first so the roots launch into a busy GPU
                shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
            with torch.cuda.stream(rs):
                X, info = shp.inverse_pth_root_batched(A, 4, fp64_iters=args.precision)
            with torch.cuda.stream(ts):
                for _ in range(args.loops):
                    if work in ("both", "stats"):
                        shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
                    if work in ("both", "precondition"):
                        shp.precondition(table, plan, roots, gn, sc, roots_lo=roots_lo)
            torch.cuda.synchronize()
            inf = shp.info_to_numpy(info)
            for s in inf["status"]:
                st_hist[int(s)] = st_hist.get(int(s), 0) + 1
            for i in range(args.batch):
                if not torch.equal(X[i], X_ref[i]) or inf[i]["status"] != inf_ref[i]["status"]:
                    mism += 1
                    d = (X[i].double() - X_ref[i].double()).norm() / X_ref[i].double().norm()
                    max_rel = max(max_rel, float(d) if torch.isfinite(d) else float("inf"))
        bad_total += mism
        print(json.dumps({"setting": setting, "root_stream_priority": pr, "train_stream_priority": pt, "work": work,
                          "batch": args.batch, "trials": args.trials, "mismatching_roots": mism,
                          "max_rel_diff": max_rel, "status_hist": {str(k): v for k, v in sorted(st_hist.items())},
                          "status_ref": {str(k): int((inf_ref["status"] == k).sum()) for k in np.unique(inf_ref["status"])}}),
              flush=True)
sys.exit(1 if bad_total else 0)
