"""Host emulation of the Ozaki root for choosing the slice count S.

Emulates exactly what csrc/ozaki.cuh computes -- per-row exponent e_i of
max_k |A_ik|, one rounding V = rint(A_ik 2^(6 + 7(S-1) - e_i)), balanced
base-128 digits, the pairs s + t <= S + 1 accumulated exactly (the digit
products are integer-valued fp64 matmuls, exact while |sum| < 2^53), one
fp64 sum per output with weights 2^-(12 + 7d) -- inside the coupled Newton
iteration (reading #1), and compares the result with the exact
root of the same regularised matrix from numpy's eigh.  numpy only (no
oracle, no GPU): the evidence for the precision choice, not a parity check.

    python tools/ozaki_precision.py [--n 1024] [--slices 5 6 7] [--kinds wishart spectrum]
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def slices(A, S):
    mx = np.abs(A).max(axis=1)
    e = np.zeros(A.shape[0], dtype=np.int64)
    nz = mx > 0
    e[nz] = np.frexp(mx[nz])[1]
    V = np.rint(np.ldexp(A, (6 + 7 * (S - 1) - e)[:, None])).astype(np.int64)
    digs = []
    for _ in range(S - 1):
        d = ((V + 64) & 127) - 64
        digs.append(d)
        V = (V - d) >> 7
    digs.append(V)
    digs.reverse()  # digs[0] most significant
    return [d.astype(np.float64) for d in digs], np.ldexp(1.0, e)


def oz_mul(A, B, S):
    """C = A @ B for symmetric-or-not A, B: A sliced by rows, B by columns."""
    da, sa = slices(A, S)
    db, sb = slices(B.T.copy(), S)
    acc = [np.zeros((A.shape[0], B.shape[1])) for _ in range(S)]
    for s in range(S):
        for t in range(S - s):
            acc[s + t] += da[s] @ db[t].T
    C = np.zeros_like(acc[0])
    for d in range(S - 1, -1, -1):
        C = C + acc[d] * 2.0 ** -(12 + 7 * d)
    return C * sa[:, None] * sb[None, :]


def newton(A_hat, c, p, mul, tol=1e-7, max_iter=100):
    n = A_hat.shape[0]
    I = np.eye(n)
    X = I * (1.0 / np.sqrt(np.sqrt(c)) if p == 4 else c ** (-1.0 / p))
    M = A_hat / c
    best = (np.inf, X, 0)
    for k in range(max_iter):
        err = np.abs(M - I).max()
        if err < best[0]:
            best = (err, X, k)
        if err <= tol:
            break
        T = ((p + 1) * I - M) / p
        X = mul(X, T)
        Tp = T
        for _ in range(int(np.log2(p))):
            Tp = mul(Tp, Tp)
        M = mul(Tp, M)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--slices", type=int, nargs="+", default=[5, 6, 7])
    ap.add_argument("--kinds", nargs="+", default=["wishart", "spectrum"])
    ap.add_argument("--eps-rel", type=float, default=1e-6)
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
        err64, X64, k64 = newton(A_hat, c, p, lambda a, b: a @ b)
        X32 = X64.astype(np.float32).astype(np.float64)
        print(f"{kind} n={n} p={p} kappa={wh[-1] / wh[0]:.3g}: fp64 newton {k64} it, root err "
              f"{np.linalg.norm(X64 - X_true) / nrm:.2e} (fp32-rounded {np.linalg.norm(X32 - X_true) / nrm:.2e})",
              flush=True)
        for S in args.slices:
            err, X, k = newton(A_hat, c, p, lambda a, b, S=S: oz_mul(a, b, S))
            print(f"  S={S} ({S * (S + 1) // 2} slice products): {k} it, max|M-I| {err:.1e}, root err "
                  f"{np.linalg.norm(X - X_true) / nrm:.2e}", flush=True)


if __name__ == "__main__":
    main()
