"""Oracle: lambda_max by power iteration, ridge, coupled-Newton inverse p-th root
and the root residual (rows a3-a6).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy, fp64; ``A @ B``
(a library matmul) is the only primitive used for products.

The paper names the method -- "the Schur-Newton algorithm ... can compute the
inverse p'th root as a sequence of matrix-vector and matrix-matrix products"
(P:206-210), in double precision -- but prints no formula.  The
iteration, ridge, scaling and stopping rule below are the readings recorded in
DESIGN.md §3 (#1-#4, #16), taken from SPEC.md S:131-132 / S:163-164:

  power iteration (reading #3): v0[i] = splitmix64(i) mapped to [-1, 1),
      v = v0/|v0|; repeat `power_iters` times: w = A v; lam = v.w;
      if |w| == 0: break; v = w/|w|.      lam_hat = last lam.
  degenerate (reading #18): lam_hat non-finite -> status 2, X untouched;
      lam_hat <= 0 -> status 3, X = I.
  ridge + scale (reading #2, "eps I"): A_hat = A + eps_rel*lam_hat*I,
      c = lam_hat*(1+eps_rel), M_0 = A_hat/c, X_0 = c^{-1/p} I with
      c^{-1/4} = 1/sqrt(sqrt(c)), c^{-1/2} = 1/sqrt(c).
  iterate (reading #1), k = 0, 1, ...:
      err_k = max_ij |M_k - I|
      if err_k is not finite                           -> X untouched   (status 2)
      if err_k <= tol                                   -> return X_k   (status 0)
      if k >= 1 and err_k >= err_{k-1} and err_{k-1} < 1e-2
                                                         -> return X_{k-1} (status 1)
      if k == max_iter                                   -> return X_k   (status 1)
      T = ((p+1) I - M_k)/p;  X_{k+1} = X_k T;  M_{k+1} = T^p M_k
      (T^p by repeated squaring: T^2, T^4 = (T^2)^2, ...)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64_start(n: int) -> np.ndarray:
    """Deterministic power-iteration start vector v0 in [-1, 1) (reading #3).

    z = i + 0x9E3779B97F4A7C15; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
    z = (z ^ z>>27) * 0x94D049BB133111EB; z ^= z>>31;
    v0[i] = (z>>11) * 2^-53 * 2 - 1    (all uint64 arithmetic wraps)
    """
    v = np.empty(n, np.float64)
    for i in range(n):
        z = (i + 0x9E3779B97F4A7C15) & MASK64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        z = z ^ (z >> 31)
        v[i] = float(z >> 11) * (2.0 ** -53) * 2.0 - 1.0
    return v


def power_iteration(A: np.ndarray, iters: int = 100) -> float:
    """Rayleigh-quotient estimate of lambda_max(A) after `iters` power steps."""
    A = np.asarray(A, np.float64)
    v = splitmix64_start(A.shape[0])
    v = v / np.sqrt(np.dot(v, v))
    lam = 0.0
    for _ in range(iters):
        w = A @ v
        lam = float(np.dot(v, w))
        nw = float(np.sqrt(np.dot(w, w)))
        if nw == 0.0:
            break
        v = w / nw
    return lam


def c_pow_neg_inv_p(c: float, p: int) -> float:
    """c^{-1/p} by IEEE sqrt chains (exact scale equivariance for c -> 16^k c)."""
    if p == 1:
        return 1.0 / c
    if p == 2:
        return 1.0 / np.sqrt(c)
    if p == 4:
        return 1.0 / np.sqrt(np.sqrt(c))
    if p == 8:
        return 1.0 / np.sqrt(np.sqrt(np.sqrt(c)))
    raise ValueError("p must be 1, 2, 4 or 8")


def matrix_power_by_squaring(T: np.ndarray, p: int) -> np.ndarray:
    out = T
    q = p
    while q > 1:
        out = out @ out
        q //= 2
    return out


@dataclass
class RootInfo:
    iters: int
    status: int  # 0 ok, 1 not converged (best iterate), 2 non-finite, 3 degenerate
    lambda_max: float
    err: float


STAGNATION_GATE = 1e-2


def inverse_pth_root(A, p: int, eps_rel: float = 1e-6, tol: float = 1e-7, max_iter: int = 100,
                     power_iters: int = 100, X_prev=None):
    """Return (X, RootInfo) with X ~ (A + eps_rel*lam_hat*I)^{-1/p} in fp64.

    ``X_prev`` is returned unchanged (status 2) when lam_hat is non-finite.
    """
    if p not in (1, 2, 4, 8):
        raise ValueError("p must be 1, 2, 4 or 8")
    A = np.asarray(A, np.float64)
    n = A.shape[0]
    lam = power_iteration(A, power_iters)
    if not np.isfinite(lam):
        return X_prev, RootInfo(0, 2, lam, float("nan"))
    I = np.eye(n)
    if lam <= 0.0:
        return I.copy(), RootInfo(0, 3, lam, float("nan"))
    Ahat = A + (eps_rel * lam) * I
    c = lam * (1.0 + eps_rel)
    M = Ahat / c
    X = c_pow_neg_inv_p(c, p) * I
    X_last = None
    err_last = float("inf")
    k = 0
    while True:
        err = float(np.max(np.abs(M - I)))
        if not np.isfinite(err):            # overflow / NaN mid-iteration: treat as non-finite input
            return X_prev, RootInfo(k, 2, lam, err)
        if err <= tol:
            return X, RootInfo(k, 0, lam, err)
        if k >= 1 and err >= err_last and err_last < STAGNATION_GATE:
            return X_last, RootInfo(k - 1, 1, lam, err_last)
        if k == max_iter:
            return X, RootInfo(k, 1, lam, err)
        T = ((p + 1) * I - M) / p
        X_last, err_last = X, err
        X = X @ T
        M = matrix_power_by_squaring(T, p) @ M
        k += 1


def residual(A, X, p: int, eps_rel: float, lam: float) -> float:
    """Independent root check ||X^p A_hat - I||_F with A_hat = A + eps_rel*lam*I
    (the "residual check" of config 2; invariant named by the north star)."""
    A = np.asarray(A, np.float64)
    X = np.asarray(X, np.float64)
    n = A.shape[0]
    Ahat = A + (eps_rel * lam) * np.eye(n)
    return float(np.linalg.norm(matrix_power_by_squaring(X, p) @ Ahat - np.eye(n)))
