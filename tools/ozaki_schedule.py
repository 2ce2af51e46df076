"""Host emulation of a per-iteration slice schedule for the Ozaki root (reading #29).

Why a schedule can drop slices late in the iteration: an error F made in M_k
reaches the root as X_k (M_k + F)^(-1/p) instead of X_k M_k^(-1/p) (the rest of
the iteration drives M to I and multiplies X by M_k^(-1/p)), i.e. relative to
the root it is amplified by ~ 1/(p lambda_min(M_k)).  lambda_min(M_0) >=
eps_rel / (1 + eps_rel) (the ridge) and the scalar recurrence
m <- m ((p+1-m)/p)^p grows it by g = ((p+1)/p)^p (2.44 for p = 4) per
iteration until it nears 1, so the amplification bound falls geometrically
with k and later products need fewer bits.  The bound is a-priori (from
eps_rel, p and k only), never from the matrix.

Schedule tested here (S_k = slices of every product of iteration k):
  m_k = min(1, eps_rel g^k); S_k = the smallest S in [S_min, S_max] with
  2^-(7S - 1) / (p m_k) <= budget.
The X-update product X_k T_k is not amplified (X only accumulates T's), so it
may take its own slice count (--sx).

Emulates exactly what csrc/ozaki.cuh computes (row exponent, one rounding to
7S - 1 bits, balanced base-128 digits, pairs s + t <= S + 1 exact, one fp64
sum per output), numpy only, and compares with the exact root (eigh).

    python tools/ozaki_schedule.py [--n 512] [--budget 1e-9 1e-10] [--kinds wishart spectrum]
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from tools.ozaki_precision import oz_mul  # noqa: E402


def schedule(k, p, eps_rel, budget, s_min=4, s_max=7):
    g = ((p + 1) / p) ** p
    m = min(1.0, eps_rel * g ** k)
    for S in range(s_min, s_max + 1):
        if 2.0 ** -(7 * S - 1) / (p * m) <= budget:
            return S
    return s_max


def newton(A_hat, c, p, sched, sx, tol=1e-7, max_iter=100):
    n = A_hat.shape[0]
    I = np.eye(n)
    X = I * (1.0 / np.sqrt(np.sqrt(c)) if p == 4 else c ** (-1.0 / p))
    M = A_hat / c
    best = (np.inf, X, 0)
    work = 0
    used = []
    for k in range(max_iter):
        err = np.abs(M - I).max()
        if err < best[0]:
            best = (err, X, k)
        if err <= tol:
            break
        S = sched(k)
        Sx = min(S, sx) if sx else S
        used.append((S, Sx))
        T = ((p + 1) * I - M) / p
        X = oz_mul(X, T, Sx)
        work += Sx * (Sx + 1) // 2
        Tp = T
        for _ in range(int(np.log2(p))):
            Tp = oz_mul(Tp, Tp, S)
            work += S * (S + 1) // 2
        M = oz_mul(Tp, M, S)
        work += S * (S + 1) // 2
    return best, work, used


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--budget", type=float, nargs="+", default=[1e-9])
    ap.add_argument("--sx", type=int, nargs="+", default=[0], help="cap on the X-update's slices (0: none)")
    ap.add_argument("--kinds", nargs="+", default=["wishart", "spectrum"])
    ap.add_argument("--eps-rel", type=float, default=1e-6)
    ap.add_argument("--s-min", type=int, default=5)
    ap.add_argument("--full", action="store_true", help="also the all-S=7 reference run")
    args = ap.parse_args()
    n, p = args.n, args.p
    for kind in args.kinds:
        A = (synth.wishart(n, synth.BASE_SEED + 2) if kind == "wishart" else synth.spectrum(n, synth.BASE_SEED + 2))
        A = A.astype(np.float64)
        w, Q = np.linalg.eigh(A)
        lam = w[-1]
        A_hat = A + args.eps_rel * lam * np.eye(n)
        c = lam * (1 + args.eps_rel)
        wh = w + args.eps_rel * lam
        X_true = (Q * wh ** (-1.0 / p)) @ Q.T
        nrm = np.linalg.norm(X_true)
        X32 = None
        print(f"{kind} n={n} p={p} kappa={wh[-1] / wh[0]:.3g}", flush=True)
        runs = [("all S=7", lambda k: 7, 0)] if args.full else []
        for b in args.budget:
            for sx in args.sx:
                runs.append((f"budget {b:g}, X cap {sx or '-'}", lambda k, b=b: schedule(k, p, args.eps_rel, b, args.s_min), sx))
        for name, sched, sx in runs:
            (err, X, k), work, used = newton(A_hat, c, p, sched, sx)
            r = np.linalg.norm(X - X_true) / nrm
            X32 = X.astype(np.float32).astype(np.float64)
            r32 = np.linalg.norm(X32 - X_true) / nrm
            full = k * (p.bit_length() + 1) * 28
            print(f"  {name}: {k} it, max|M-I| {err:.1e}, root err {r:.2e} (fp32-rounded {r32:.2e}), "
                  f"slice products {work} = {work / max(full, 1):.2f} of all-S=7; S_k {[u[0] for u in used]}"
                  f" Sx_k {[u[1] for u in used]}", flush=True)


if __name__ == "__main__":
    main()
