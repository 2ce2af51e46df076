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
      c^{-1/4} = 1/sqrt(sqrt(c)), c^{-1/2} = 1/sqrt(c) (sqrt chains for
      p = 2^j), c ** (-1/p) otherwise (reading #22: any integer p in [1, 16]).
  iterate (reading #1), k = 0, 1, ...:
      err_k = max_ij |M_k - I|
      if err_k is not finite                           -> X untouched   (status 2)
      if err_k <= tol                                   -> return X_k   (status 0)
      if k >= 1 and err_k >= err_{k-1} and err_{k-1} < 1e-2
                                                         -> return X_{k-1} (status 1)
      if k == max_iter                                   -> return X_k   (status 1)
      T = ((p+1) I - M_k)/p;  X_{k+1} = X_k T;  M_{k+1} = T^p M_k
      (T^p by numpy's matrix_power, a library primitive)
  rational exponent (f4, "L^{-1/2p} G R^{-1/2q}"; reading #23):
      X = (A_hat^{-1/p})^r, the converged root raised to the integer power r.
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


MAX_P = 16


def valid_p(p: int) -> bool:
    return isinstance(p, (int, np.integer)) and 1 <= p <= MAX_P


def c_pow_neg_inv_p(c: float, p: int) -> float:
    """c^{-1/p}: IEEE sqrt chains for p = 2^j (exact scale equivariance for
    c -> 16^k c), the library power otherwise."""
    if not valid_p(p):
        raise ValueError(f"p must be an integer in [1, {MAX_P}]")
    if p & (p - 1) == 0:
        x = c
        q = p
        while q > 1:
            x = np.sqrt(x)
            q //= 2
        return 1.0 / x
    return float(c ** (-1.0 / p))


def matrix_power(T: np.ndarray, p: int) -> np.ndarray:
    return np.linalg.matrix_power(T, p)


matrix_power_by_squaring = matrix_power  # historical name (p = 2^j)


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
    if not valid_p(p):
        raise ValueError(f"p must be an integer in [1, {MAX_P}]")
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
        M = matrix_power(T, p) @ M
        k += 1


def inverse_root(A, p: int, r: int = 1, eps_rel: float = 1e-6, tol: float = 1e-7, max_iter: int = 100,
                 power_iters: int = 100, X_prev=None):
    """X ~ A_hat^{-r/p} = (A_hat^{-1/p})^r (f4: rational exponents r/p, 1 <= r <= p).
    Statuses / info are those of the p-th root; status 2 returns X_prev."""
    if not (isinstance(r, (int, np.integer)) and 1 <= r <= p):
        raise ValueError("need 1 <= r <= p")
    X, info = inverse_pth_root(A, p, eps_rel, tol, max_iter, power_iters, X_prev)
    if info.status == 2 or r == 1:
        return X, info
    return matrix_power(X, r), info


def residual(A, X, p: int, eps_rel: float, lam: float) -> float:
    """Independent root check ||X^p A_hat - I||_F with A_hat = A + eps_rel*lam*I
    (the "residual check" of config 2; invariant named by the north star)."""
    A = np.asarray(A, np.float64)
    X = np.asarray(X, np.float64)
    n = A.shape[0]
    Ahat = A + (eps_rel * lam) * np.eye(n)
    return float(np.linalg.norm(matrix_power(X, p) @ Ahat - np.eye(n)))
