"""CPU baseline per BASELINE.md §3: the fp64 oracle (as it stands) on the box's host cores, one independent root
per core -- the paper's design of distributing root work "to all CPU cores available in the training system"
(P:285-288).  A baseline only, not a target.

Reports, as one JSON line: the CPU model (lscpu) and core count; seconds per root and aggregate roots/s at
n in {64, 128, 512, 1024} (p = 4, eps_rel = 1e-6, Wishart statistics of kappa ~1e6, iteration counts); config 1
(64x64 from a 64x32 gradient: statistics + 2 roots + preconditioned gradient + graft) end to end; config 3
(Transformer-Big) statistics + preconditioning on a sample of blocks run one per core, extrapolated to all 360
blocks (labelled so).

    python tools/cpu_baseline.py [--sizes 64 128 512 1024] [--config3-blocks 0]
"""

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _init():
    # one BLAS thread per worker (set in the environment before numpy loads; threadpoolctl as a second guard)
    import threadpoolctl
    global _LIMITS
    _LIMITS = threadpoolctl.threadpool_limits(1)


def _root(args):
    n, seed = args
    import numpy as np

    import synth
    from oracle import root as oroot
    A = synth.wishart(n, seed).astype(np.float64)
    t0 = time.perf_counter()
    _, info = oroot.inverse_pth_root(A, 4)
    return time.perf_counter() - t0, info.iters


def _config3_block(bi):
    import numpy as np

    import synth
    from oracle import plan as oplan
    from oracle import precondition as opre
    from oracle import root as oroot  # noqa: F401
    from oracle import stats as ostats
    shapes = [s for _, s in synth.transformer_big_shapes()]
    pl = oplan.plan(shapes, 1024, 8192, 1)
    b = pl.blocks[bi]
    m, n = shapes[b.tensor_id]
    seed = synth.BASE_SEED + 3 + b.tensor_id
    G = synth.vocab_gradient(m, n, seed) if m == synth.VOCAB else synth.lowrank_gradient(m, n, seed)
    D = [np.zeros((m, n), np.float32) if t == b.tensor_id else None for t in range(len(shapes))]
    Gs = [G if t == b.tensor_id else None for t in range(len(shapes))]
    stats = np.zeros(pl.stats_elems, np.float32)
    t0 = time.perf_counter()
    num, _ = ostats.stats_update(Gs, D, pl, stats, 1.0, 1.0, blocks=[bi])
    t1 = time.perf_counter()
    Gb = G[b.row0:b.row0 + b.rows, b.col0:b.col0 + b.cols]
    XL = np.eye(b.rows) if b.p_left else None    # identity roots: the preconditioning cost, not the roots'
    XR = np.eye(b.cols) if b.p_right else None
    P = opre.precondition_block(Gb, XL, XR, D[b.tensor_id][b.row0:b.row0 + b.rows, b.col0:b.col0 + b.cols])
    opre.graft_scale(float(num[bi]), float(np.sum(P * P)))
    return t1 - t0, time.perf_counter() - t1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[64, 128, 512, 1024])
    ap.add_argument("--config3-blocks", type=int, default=-1, help="sample size (default: one per core)")
    args = ap.parse_args()
    import numpy as np

    import synth
    cores = len(os.sched_getaffinity(0))
    try:
        model = [ln.split(":", 1)[1].strip() for ln in subprocess.run(["lscpu"], capture_output=True, text=True)
                 .stdout.splitlines() if ln.startswith("Model name")][0]
    except (OSError, IndexError):
        model = "unknown"
    out = {"kind": "oracle", "cpu_model": model, "cores": cores, "threads_per_root": 1, "roots": []}
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"  # inherited by the spawned workers before they import numpy
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores, initializer=_init) as pool:
        pool.map(_root, [(16, 1)] * cores)  # warm the workers (imports)
        for n in args.sizes:
            t0 = time.perf_counter()
            res = pool.map(_root, [(n, synth.BASE_SEED + 2 + i) for i in range(cores)])
            wall = time.perf_counter() - t0
            per = [r[0] for r in res]
            out["roots"].append({"n": n, "p": 4, "roots": cores, "wall_s": wall, "roots_per_s": cores / wall,
                                 "s_per_root_median": float(np.median(per)),
                                 "iters_mean": float(np.mean([r[1] for r in res]))})
            print(json.dumps(out["roots"][-1]), file=sys.stderr, flush=True)
        # config 3: statistics + preconditioning, one block per core, extrapolated to 360 blocks
        shapes = [s for _, s in synth.transformer_big_shapes()]
        from oracle import plan as oplan
        nb = len(oplan.plan(shapes, 1024, 8192, 1).blocks)
        k = cores if args.config3_blocks < 0 else args.config3_blocks
        if k > 0:
            sample = [int(x) for x in np.linspace(0, nb - 1, k)]
            t0 = time.perf_counter()
            res = pool.map(_config3_block, sample)
            wall = time.perf_counter() - t0
            out["config3_stats_precondition"] = {
                "sample_blocks": k, "wall_s": wall, "stats_s_mean": float(np.mean([r[0] for r in res])),
                "precondition_s_mean": float(np.mean([r[1] for r in res])),
                "extrapolated_step_s_all_360_blocks": wall * nb / k, "label": "extrapolated from the sample"}
    # config 1 end to end (one process)
    from oracle import plan as oplan
    from oracle import precondition as opre
    from oracle import root as oroot
    from oracle import stats as ostats
    G = synth.gaussian((64, 32), synth.BASE_SEED + 1)
    t0 = time.perf_counter()
    pl = oplan.plan([G.shape], 1024, 8192, 1)
    st = np.zeros(pl.stats_elems, np.float32)
    D = [np.zeros(G.shape, np.float32)]
    num, _ = ostats.stats_update([G], D, pl, st, 1.0, 1.0)
    b = pl.blocks[0]
    roots = np.zeros(pl.stats_elems)
    for nn, off, ld in ((b.rows, b.left_off, b.left_ld), (b.cols, b.right_off, b.right_ld)):
        A = st[off:off + nn * ld].reshape(nn, ld)[:, :nn].astype(np.float64)
        roots[off:off + nn * ld].reshape(nn, ld)[:, :nn] = oroot.inverse_pth_root(A, 4)[0]
    opre.precondition_plan([G], D, pl, roots, num)
    out["config1_end_to_end_ms"] = (time.perf_counter() - t0) * 1e3
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
