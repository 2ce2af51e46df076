"""f1 measurement: Transformer-Big Shampoo steps while the delayed, pipelined
root refresh runs (kappa = 500 as in the paper's runs).

The training step (statistics + preconditioning, the Shampoo step of the
metric) runs on a HIGH-priority stream; ``DelayedRefresh`` enqueues each step's
chunk of roots (the bench's precision, "auto" = Ozaki) on its own
LOWEST-priority stream, so the refresh fills what the step leaves idle
("pipelined and runs asynchronously without blocking the training
loop").  For each chunk size the script times the whole refresh window (every
chunk step plus the gather step) against the same number of plain steps; the
refresh's cost per step of a kappa window is (window - plain) / kappa.

    python tools/bench_delayed.py [--kappa 500] [--chunks 2,8,32]
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
ap.add_argument("--chunks", default="2,8,32", help="roots per step (busiest rank)")
ap.add_argument("--precision", default="auto")
ap.add_argument("--plain-steps", type=int, default=30)
args = ap.parse_args()
dev = torch.device("cuda", 0)
names_shapes = synth.transformer_big_shapes()
shapes = [s for _, s in names_shapes]
plan = shp.make_plan(shapes, 1024, 8192, 1)
Gs = []
for i, (m, n) in enumerate(shapes):  # bench.py's gradient recipe
    seed = synth.BASE_SEED + 3 + i
    Gs.append(synth.vocab_gradient_device(m, n, seed, dev) if m == synth.VOCAB
              else synth.lowrank_gradient_device(m, n, seed, dev))
Ps = [torch.zeros_like(G) for G in Gs]
table = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs], Ps)
stats = torch.zeros(plan.stats_elems, device=dev)
roots = torch.zeros_like(stats)
gn = torch.zeros(plan.n_blocks, dtype=torch.float64, device=dev)
sc = torch.zeros(plan.n_blocks, device=dev)
for _ in range(8):
    shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
shp.refresh_group_roots(plan, stats, roots, 0, fp64_iters=args.precision)  # bootstrap roots
roots_lo = shp.tf32_split(roots)
torch.cuda.synchronize()
lo_prio, hi_prio = torch.cuda.Stream.priority_range()
train = torch.cuda.Stream(device=dev, priority=hi_prio)


def timed(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(train):
        e0.record(train)
        for t in range(n):
            fn(t)
        e1.record(train)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def plain(t):
    shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
    shp.precondition(table, plan, roots, gn, sc, roots_lo=roots_lo)


def synchronous(t):
    shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
    shp.refresh_group_roots(plan, stats, roots, 0, fp64_iters=args.precision)
    shp.tf32_split(roots, roots_lo)
    shp.precondition(table, plan, roots, gn, sc, roots_lo=roots_lo)


timed(plain, 3)  # warm-up
ms_plain = timed(plain, args.plain_steps) / args.plain_steps
ms_sync = timed(synchronous, 2) / 2
out = {"f1": "delayed pipelined refresh on a lowest-priority stream, step on a highest-priority stream",
       "kappa": args.kappa, "precision": args.precision, "stream_priorities": [lo_prio, hi_prio],
       "step_ms_plain": ms_plain, "step_ms_synchronous_refresh": ms_sync,
       "refresh_ms_synchronous": ms_sync - ms_plain,
       "amortised_floor_ms_per_step": (ms_sync - ms_plain) / args.kappa, "chunks": []}
for chunk in [int(c) for c in args.chunks.split(",")]:
    with torch.cuda.stream(train):
        dr = DelayedRefresh(plan, stats, roots.clone(), kappa=args.kappa, chunk=chunk, fp64_iters=args.precision)

    def delayed(t, dr=dr):
        shp.stats_update(table, plan, stats, 1.0, 1.0, -1, gn)
        dr.step(t)
        shp.precondition(table, plan, dr.current, gn, sc, roots_lo=dr.current_lo)

    timed(delayed, 1)  # warm-up step 0 (snapshot + first chunk)
    with torch.cuda.stream(train):
        dr = DelayedRefresh(plan, stats, roots.clone(), kappa=args.kappa, chunk=chunk, fp64_iters=args.precision)
    ms_window = timed(lambda t, dr=dr: delayed(t, dr), dr.n_steps)  # every chunk step, the last one gathers
    assert dr.ready and dr.refreshes == 1
    st = [int(s) for _, _, _, info in dr.infos for s in shp.info_to_numpy(info)["status"]]
    # the gathered roots against a synchronous refresh of the same snapshot (bit-identity)
    ref = torch.zeros_like(roots)
    shp.refresh_group_roots(plan, dr.snapshot, ref, 0, fp64_iters=args.precision)
    torch.cuda.synchronize()
    mism, bad_info = 0, []
    for g, i0, cnt, info in dr.infos:
        nn, stride, off0 = int(g["n"]), int(g["stride"]), int(g["offset"])
        inf = shp.info_to_numpy(info)
        for q in range(cnt):
            o = off0 + (i0 + q) * stride
            if not torch.equal(dr.next[o:o + nn * ((nn + 3) // 4 * 4)], ref[o:o + nn * ((nn + 3) // 4 * 4)]):
                mism += 1
            if inf[q]["status"] != 0:
                bad_info.append({"n": nn, "p": int(g["p"]), "index": i0 + q, "status": int(inf[q]["status"]),
                                 "iters": int(inf[q]["iters"]), "lambda": float(inf[q]["lambda_max"]),
                                 "err": float(inf[q]["err"])})
    extra = ms_window - dr.n_steps * ms_plain
    out["chunks"].append({"roots_per_step": chunk, "window_steps": dr.n_steps, "window_ms": ms_window,
                          "step_ms_during_window": ms_window / dr.n_steps,
                          "refresh_cost_ms": extra, "cost_per_step_ms_over_kappa": extra / args.kappa,
                          "step_delta_frac_over_kappa": extra / args.kappa / ms_plain,
                          "refresh_cost_vs_synchronous": extra / (ms_sync - ms_plain),
                          "statuses": {str(s): st.count(s) for s in sorted(set(st))},
                          "roots_differing_from_synchronous_refresh": mism, "nonzero_status": bad_info[:20]})
print(json.dumps(out), flush=True)
