"""Pins for the root oracle (rows a3-a6): SPEC worked examples, closed forms,
eigendecomposition (numpy eigh) cross-checks, the decoupled scalar recurrence,
exact scale equivariance, orthogonal similarity, the residual invariant and
the degenerate cases.  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import root as oroot
from synth import gaussian, spectrum, wishart

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def eig_root(Ahat, p):
    w, V = np.linalg.eigh(Ahat)
    return (V * w ** (-1.0 / p)) @ V.T


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ------------------------------------------------------------ power iteration

def test_splitmix_start_vector_known_values():
    # splitmix64(0) first output is the published constant 0xE220A8397B1DCDAF
    # (Steele, Lea, Flood 2014 reference sequence for seed 0); v0 = (z>>11)*2^-53*2 - 1.
    z = 0xE220A8397B1DCDAF
    v = oroot.splitmix64_start(3)
    assert v[0] == (z >> 11) * 2.0 ** -53 * 2 - 1
    assert np.all(np.abs(v) <= 1.0) and len(set(v.tolist())) == 3


def test_power_iteration_diagonal_and_rank_one():
    d = np.array([3.0, 1.0, 0.5, 0.25])
    assert oroot.power_iteration(np.diag(d)) == pytest.approx(3.0, rel=1e-14)
    u = gaussian((16,), 7).astype(np.float64)
    u /= np.linalg.norm(u)
    s, delta = 10.0, 1e-3
    A = s * np.outer(u, u) + delta * np.eye(16)
    assert oroot.power_iteration(A) == pytest.approx(s + delta, rel=1e-13)


@pytest.mark.parametrize("n", [32, 128])
def test_power_iteration_rayleigh_bound(n):
    A = wishart(n, 100 + n).astype(np.float64)
    lam = oroot.power_iteration(A)
    true = np.linalg.eigvalsh(A)[-1]
    assert lam <= true * (1 + 1e-14)           # a Rayleigh quotient never exceeds lambda_max
    assert lam >= true * (1 - 2e-2)            # and is close after 100 steps (small top gap)


def test_power_iteration_zero_matrix():
    assert oroot.power_iteration(np.zeros((5, 5))) == 0.0


# ------------------------------------------------------------ worked examples

def _golden_roots():
    with open(os.path.join(GOLDEN, "root_cases.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _golden_roots(), ids=["identity5", "diag16_81"])
def test_spec_worked_examples(case):
    if case["A"] == "identity":
        A = np.eye(case["n"])
        X, info = oroot.inverse_pth_root(A, case["p"], eps_rel=case["eps_rel"])
        want = (1 + case["eps_rel"]) ** (-1.0 / case["p"]) * np.eye(case["n"])
        np.testing.assert_allclose(X, want, rtol=case["rtol"], atol=0)
        assert info.iters <= case["max_iters"] and info.status == 0
    else:
        X, info = oroot.inverse_pth_root(np.array(case["A"]), case["p"], eps_rel=case["eps_rel"], tol=1e-14)
        np.testing.assert_allclose(X, np.array(case["X"]), atol=case["atol"], rtol=0)
        assert info.status == 0


# ------------------------------------------------------------ closed forms

@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_scalar_n1(p):
    a = 7.25
    eps = 1e-6
    X, info = oroot.inverse_pth_root(np.array([[a]]), p, eps_rel=eps, tol=1e-14)
    assert X[0, 0] == pytest.approx((a * (1 + eps)) ** (-1.0 / p), rel=1e-14)
    assert info.lambda_max == a


@pytest.mark.parametrize("p", [2, 4])
def test_rank_one_plus_delta(p):
    n = 24
    u = gaussian((n,), 8).astype(np.float64)
    u /= np.linalg.norm(u)
    s, delta, eps = 50.0, 1e-3, 1e-6
    A = s * np.outer(u, u) + delta * np.eye(n)
    X, info = oroot.inverse_pth_root(A, p, eps_rel=eps, tol=1e-13)
    r = eps * info.lambda_max
    P = np.outer(u, u)
    want = (s + delta + r) ** (-1.0 / p) * P + (delta + r) ** (-1.0 / p) * (np.eye(n) - P)
    assert rel(X, want) < 1e-11
    assert info.lambda_max == pytest.approx(s + delta, rel=1e-13)


def test_diagonal_decouples_into_scalar_recurrences():
    # With A diagonal every iterate is diagonal, and each entry follows
    #   m <- m ((p+1-m)/p)^p,  x <- x (p+1-m)/p   (the scalar form of S:131).
    d = np.array([1.0, 0.5, 1e-3, 1e-6])
    p, eps, tol = 4, 1e-6, 1e-9
    X, info = oroot.inverse_pth_root(np.diag(d), p, eps_rel=eps, tol=tol)
    lam = 1.0
    c = lam * (1 + eps)
    m = (d + eps * lam) / c
    x = np.full(4, c ** -0.25)
    k = 0
    while np.max(np.abs(m - 1)) > tol:
        t = (p + 1 - m) / p
        x, m, k = x * t, m * t ** p, k + 1
    assert info.iters == k and info.status == 0
    np.testing.assert_allclose(np.diag(X), x, rtol=1e-13)
    assert np.count_nonzero(X - np.diag(np.diag(X))) == 0


# ------------------------------------------------------------ eigh cross-checks

@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_matches_eigh_wishart_kappa_1e6(p):
    # config 1's L: 64x64 rank-32 Wishart, kappa(A_hat) ~ 1e6 after the ridge
    G = gaussian((64, 32), 200209019)
    A = G.astype(np.float64) @ G.astype(np.float64).T
    X, info = oroot.inverse_pth_root(A, p, eps_rel=1e-6, tol=1e-12)
    Ahat = A + 1e-6 * info.lambda_max * np.eye(64)
    w = np.linalg.eigvalsh(Ahat)
    assert w[-1] / w[0] > 5e5
    assert rel(X, eig_root(Ahat, p)) < 1e-8
    assert info.status == 0 and 15 <= info.iters <= 40


def test_matches_eigh_spectrum_kappa_1e8():
    # random 64x64 with condition 1e8 (ridge caps kappa(A_hat) near 1e6)
    A = spectrum(64, 5).astype(np.float64)
    X, info = oroot.inverse_pth_root(A, 4, eps_rel=1e-6, tol=1e-12)
    Ahat = A + 1e-6 * info.lambda_max * np.eye(64)
    assert rel(X, eig_root(Ahat, 4)) < 1e-6


def test_default_tolerance_is_within_1e6_of_exact():
    A = wishart(96, 31).astype(np.float64)
    X, info = oroot.inverse_pth_root(A, 4)  # defaults: eps 1e-6, tol 1e-7
    Ahat = A + 1e-6 * info.lambda_max * np.eye(96)
    assert rel(X, eig_root(Ahat, 4)) < 1e-6


# ------------------------------------------------------------ invariants

def test_scale_equivariance_bit_exact():
    A = wishart(32, 9).astype(np.float64)
    X1, i1 = oroot.inverse_pth_root(A, 4)
    X2, i2 = oroot.inverse_pth_root(A * 16.0 ** 3, 4)
    assert i1.iters == i2.iters
    assert np.array_equal(X2, X1 / 8.0)  # (16^3)^{-1/4} = 1/8 exactly


def test_orthogonal_similarity():
    A = wishart(40, 12).astype(np.float64)
    Q, _ = np.linalg.qr(gaussian((40, 40), 13).astype(np.float64))
    X1, _ = oroot.inverse_pth_root(A, 4, tol=1e-12)
    X2, _ = oroot.inverse_pth_root(Q @ A @ Q.T, 4, tol=1e-12)
    assert rel(X2, Q @ X1 @ Q.T) < 1e-8


def test_residual_invariant():
    A = wishart(64, 14).astype(np.float64)
    X, info = oroot.inverse_pth_root(A, 4, tol=1e-12)
    res = oroot.residual(A, X, 4, 1e-6, info.lambda_max)
    assert res < 1e-6
    # a root perturbed by 1e-4 must show up in the residual
    assert oroot.residual(A, X * (1 + 1e-4), 4, 1e-6, info.lambda_max) > 1e-4


# ------------------------------------------------------------ degenerate cases

def test_non_finite_input_keeps_previous_root():
    A = wishart(8, 3).astype(np.float64)
    A[2, 3] = A[3, 2] = np.nan
    prev = np.full((8, 8), 7.0)
    X, info = oroot.inverse_pth_root(A, 4, X_prev=prev)
    assert info.status == 2 and X is prev


def test_zero_matrix_is_degenerate_identity():
    X, info = oroot.inverse_pth_root(np.zeros((6, 6)), 4)
    assert info.status == 3 and np.array_equal(X, np.eye(6))


def test_max_iter_not_converged_returns_iterate():
    A = wishart(32, 4).astype(np.float64)
    X, info = oroot.inverse_pth_root(A, 4, max_iter=3)
    assert info.status == 1 and info.iters == 3 and info.err > 1e-2


def test_stagnation_returns_previous_best():
    # tol below what fp64 can reach: the iteration must stop at the first
    # non-decrease (after err < 1e-2) and return the previous iterate.
    A = wishart(48, 21).astype(np.float64)
    X, info = oroot.inverse_pth_root(A, 4, tol=0.0, max_iter=200)
    assert info.status == 1 and info.iters < 60 and info.err < 1e-12
    Ahat = A + 1e-6 * info.lambda_max * np.eye(48)
    assert rel(X, eig_root(Ahat, 4)) < 1e-9


# ------------------------------------------------------------ any integer p, rational r/p (f3, f4)

def eig_power(Ahat, e):
    w, V = np.linalg.eigh(Ahat)
    return (V * w ** e) @ V.T


@pytest.mark.parametrize("p", [3, 5, 6, 7, 12, 16])
def test_general_p_matches_eigh(p):
    # p = 2k for rank-k tensors (f3: p = 6 for rank 3); the coupled iteration
    # converges for any integer p while spec(M_0) lies in (0, p+1) (Appendix A)
    G = gaussian((48, 24), 200209021)
    A = G.astype(np.float64) @ G.astype(np.float64).T
    X, info = oroot.inverse_pth_root(A, p, eps_rel=1e-6, tol=1e-12)
    Ahat = A + 1e-6 * info.lambda_max * np.eye(48)
    assert info.status == 0
    assert rel(X, eig_root(Ahat, p)) < 1e-8


@pytest.mark.parametrize("p", [3, 6])
def test_general_p_scalar_closed_form(p):
    a, eps = 7.25, 1e-6
    X, info = oroot.inverse_pth_root(np.array([[a]]), p, eps_rel=eps, tol=1e-14)
    assert X[0, 0] == pytest.approx((a * (1 + eps)) ** (-1.0 / p), rel=1e-14)


@pytest.mark.parametrize("p,r", [(8, 3), (8, 1), (6, 2), (3, 2), (5, 4), (4, 4)])
def test_rational_rank_one_plus_delta(p, r):
    # closed form of A_hat^{-r/p} for s uu^T + delta I
    n = 20
    u = gaussian((n,), 18).astype(np.float64)
    u /= np.linalg.norm(u)
    s, delta, eps = 50.0, 1e-3, 1e-6
    A = s * np.outer(u, u) + delta * np.eye(n)
    X, info = oroot.inverse_root(A, p, r, eps_rel=eps, tol=1e-13)
    rr = eps * info.lambda_max
    P = np.outer(u, u)
    e = -r / p
    want = (s + delta + rr) ** e * P + (delta + rr) ** e * (np.eye(n) - P)
    assert rel(X, want) < 1e-11


@pytest.mark.parametrize("p,r", [(8, 3), (6, 5), (16, 7)])
def test_rational_matches_eigh_and_inverse_identity(p, r):
    A = wishart(40, 77).astype(np.float64)
    X, info = oroot.inverse_root(A, p, r, tol=1e-12)
    Ahat = A + 1e-6 * info.lambda_max * np.eye(40)
    assert rel(X, eig_power(Ahat, -r / p)) < 1e-8
    # X^p A_hat^r = I (the defining identity of A_hat^{-r/p}); checked at a
    # ridge that keeps kappa(A_hat)^r within fp64 (kappa ~ 1e2)
    if r > 5:
        return  # kappa^r beyond fp64
    X, info = oroot.inverse_root(A, p, r, eps_rel=1e-2, tol=1e-13)
    Ahat = A + 1e-2 * info.lambda_max * np.eye(40)
    Y = np.linalg.matrix_power(X, p) @ np.linalg.matrix_power(Ahat, r)
    assert np.linalg.norm(Y - np.eye(40)) / np.sqrt(40) < 1e-4  # a wrong exponent gives O(1)


def test_rational_r1_is_the_pth_root_and_complementary_pair():
    A = wishart(32, 5).astype(np.float64)
    X1, _ = oroot.inverse_root(A, 8, 1, tol=1e-12)
    Xp, _ = oroot.inverse_pth_root(A, 8, tol=1e-12)
    assert np.array_equal(X1, Xp)
    # (1/8) + (3/8) = 1/2: X_{1/8} X_{3/8} = A_hat^{-1/2}
    X3, info = oroot.inverse_root(A, 8, 3, tol=1e-12)
    Ahat = A + 1e-6 * info.lambda_max * np.eye(32)
    assert rel(X1 @ X3, eig_power(Ahat, -0.5)) < 1e-8


def test_invalid_p_and_r():
    with pytest.raises(ValueError):
        oroot.inverse_pth_root(np.eye(3), 17)
    with pytest.raises(ValueError):
        oroot.inverse_root(np.eye(3), 4, 5)
    with pytest.raises(ValueError):
        oroot.inverse_root(np.eye(3), 4, 0)


def test_residual_general_p():
    A = wishart(40, 15).astype(np.float64)
    X, info = oroot.inverse_pth_root(A, 6, tol=1e-12)
    assert oroot.residual(A, X, 6, 1e-6, info.lambda_max) < 1e-6
