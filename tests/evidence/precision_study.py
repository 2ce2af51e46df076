"""Precision study for the coupled-Newton root (evidence for DESIGN.md §7.2).

Emulates the product precision of candidate tensor-core paths by rounding the
matmul OPERANDS (and, for fp32-storage variants, the iterates) and runs the
same coupled Newton iteration as the oracle on fp32 Wishart statistics
(kappa(A_hat) ~ 1e6 with eps_rel = 1e-6).  Reference: eigh of the same A_hat.

  fp64      : the shipped path (FP64 DMMA)
  bf16      : operands rounded to bf16 (8-bit significand), fp32 accumulate/storage
  tf32      : operands rounded to tf32 (11-bit significand), fp32 accumulate/storage
  3xtf32    : hi = tf32(x), lo = tf32(x - hi); hi*hi + hi*lo + lo*hi, fp32 storage
  3xtf32t   : the measured tcgen05 semantics: operands truncated to tf32, hi = trunc(x),
              lo = trunc(x - hi), fp32 accumulation
  hybN      : first N iterations fp64, then 3xtf32 (hybNt: then 3xtf32t)

    python tests/evidence/precision_study.py [--n 256] [--seeds 2] > profiles/r01_precision_study.txt
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import synth  # noqa: E402
from oracle import root as oroot  # noqa: E402


def round_mantissa(x, bits):
    """Round-to-nearest-even of fp32 values to `bits` explicit mantissa bits."""
    x32 = np.asarray(x, np.float32)
    u = x32.view(np.uint32).astype(np.uint64)
    drop = 23 - bits
    half = np.uint64(1 << (drop - 1))
    lsb = (u >> np.uint64(drop)) & np.uint64(1)
    u = (u + half - np.uint64(1) + lsb) >> np.uint64(drop) << np.uint64(drop)
    return (u.astype(np.uint32)).view(np.float32)


def mm(a, b, mode):
    if mode == "fp64":
        return a @ b
    a32, b32 = np.asarray(a, np.float32), np.asarray(b, np.float32)
    if mode == "bf16":
        return (round_mantissa(a32, 7).astype(np.float64) @ round_mantissa(b32, 7).astype(np.float64)).astype(np.float32)
    if mode == "tf32":
        return (round_mantissa(a32, 10).astype(np.float64) @ round_mantissa(b32, 10).astype(np.float64)).astype(np.float32)
    if mode == "3xtf32":
        ah = round_mantissa(a32, 10)
        al = round_mantissa(a32 - ah, 10)
        bh = round_mantissa(b32, 10)
        bl = round_mantissa(b32 - bh, 10)
        f = lambda x, y: x.astype(np.float64) @ y.astype(np.float64)
        return (f(ah, bh) + f(ah, bl) + f(al, bh)).astype(np.float32)
    if mode == "3xtf32t":
        # the measured tcgen05 kind::tf32 semantics (profiles/r01_tf32_probe.txt): operands TRUNCATED
        # to tf32; hi = trunc(x), lo = x - hi (exact in fp32) is truncated again by the MMA; the three
        # passes accumulate in fp32 (TF32 x TF32 products are exact in fp32)
        ah = trunc_mantissa(a32, 10)
        al = trunc_mantissa(a32 - ah, 10)
        bh = trunc_mantissa(b32, 10)
        bl = trunc_mantissa(b32 - bh, 10)
        return (al @ bh + ah @ bl) + ah @ bh
    raise ValueError(mode)


def trunc_mantissa(x, bits):
    """Truncation (round toward zero) of fp32 values to `bits` explicit mantissa bits."""
    u = np.asarray(x, np.float32).view(np.uint32)
    mask = np.uint32((0xFFFFFFFF << (23 - bits)) & 0xFFFFFFFF)
    return (u & mask).view(np.float32)


def newton(A, p, mode, eps=1e-6, tol=1e-7, max_iter=60, fp64_iters=0):
    n = A.shape[0]
    lam = oroot.power_iteration(A)
    I = np.eye(n)
    Ahat = A + eps * lam * I
    c = lam * (1 + eps)
    M = Ahat / c
    X = oroot.c_pow_neg_inv_p(c, p) * I
    best = (np.inf, X, 0)
    for k in range(max_iter + 1):
        err = float(np.max(np.abs(M - I)))
        if err < best[0]:
            best = (err, X, k)
        if err <= tol or k == max_iter:
            break
        cur = "fp64" if k < fp64_iters else mode
        T = ((p + 1) * I - M) / p
        X = mm(X, T, cur).astype(np.float64)
        Tp = T
        q = p
        while q > 1:
            Tp = mm(Tp, Tp, cur).astype(np.float64)
            q //= 2
        M = mm(Tp, M, cur).astype(np.float64)
        if cur != "fp64":
            X = X.astype(np.float32).astype(np.float64)
            M = M.astype(np.float32).astype(np.float64)
    return best[1], best[2], Ahat


def main():
    np.seterr(all="ignore")  # bf16 / tf32 iterations overflow; that is the result being shown
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--seeds", type=int, default=2)
    ap.add_argument("--modes", default="fp64:0,bf16:0,tf32:0,3xtf32:0,3xtf32:6,3xtf32:8")
    args = ap.parse_args()
    modes = [(m.split(":")[0], int(m.split(":")[1])) for m in args.modes.split(",")]
    print(f"# coupled Newton, p=4, eps_rel=1e-6, n={args.n}, fp32 Wishart(n/2) statistics (kappa(A_hat)~1e6)")
    print("# relative Frobenius error of X vs eigh(A_hat)^(-1/4); north-star bar 1e-3")
    print(f"{'mode':>12} {'seed':>5} {'iters':>6} {'rel_err':>10}  verdict")
    for s in range(args.seeds):
        A = synth.wishart(args.n, synth.BASE_SEED + 100 + s).astype(np.float64)
        for mode, k in modes:
            X, it, Ahat = newton(A, 4, mode, fp64_iters=k)
            w, V = np.linalg.eigh(Ahat)
            ref = (V * w ** -0.25) @ V.T
            err = np.linalg.norm(X - ref) / np.linalg.norm(ref)
            name = mode if k == 0 else (f"hyb{k}" + ("t" if mode.endswith("t") else ""))
            print(f"{name:>12} {s:>5} {it:>6} {err:>10.2e}  {'pass' if err <= 1e-3 else 'REJECT'}", flush=True)


if __name__ == "__main__":
    main()
