"""Pins for the statistics oracle (row a2): exact integer cases, the sequential
fp64 contract (order-sensitive constructions), Alg. 1's EMA unrolled, trace
identity, D = diagonal of the full AdaGrad accumulator, non-finite rejection.
CPU only."""

from fractions import Fraction

import numpy as np
import pytest

from oracle import plan as oplan
from oracle import stats as ostats
from synth import gaussian


def _left(G, decay=1.0, weight=1.0, L0=None):
    m, n = G.shape
    L = np.zeros((m, m), np.float32) if L0 is None else L0.copy()
    ostats.stats_left(G, 0, 0, m, n, L, decay, weight)
    return L


def _right(G, decay=1.0, weight=1.0, R0=None):
    m, n = G.shape
    R = np.zeros((n, n), np.float32) if R0 is None else R0.copy()
    ostats.stats_right(G, 0, 0, m, n, R, decay, weight)
    return R


def test_integer_gradients_exact():
    # Small integers: every sum is exact in fp64 and fp32, so L = G G^T and
    # R = G^T G exactly (pins indices / transposes of P:151-159).
    g = np.random.default_rng(1).integers(-3, 4, size=(7, 11))
    G = g.astype(np.float32)
    assert np.array_equal(_left(G), (g @ g.T).astype(np.float32))
    assert np.array_equal(_right(G), (g.T @ g).astype(np.float32))
    S = np.random.default_rng(2).integers(-5, 6, size=(7, 7))
    L0 = (S + S.T).astype(np.float32)  # statistics are symmetric; the upper triangle is read
    # decay 0.5 / weight 2: exact in binary
    assert np.array_equal(_left(G, 0.5, 2.0, L0), (0.5 * L0 + 2.0 * (g @ g.T)).astype(np.float32))


def test_block_views_and_ragged_blocks():
    g = np.random.default_rng(3).integers(-2, 3, size=(10, 13))
    G = g.astype(np.float32)
    L = np.zeros((4, 8), np.float32)  # padded leading dim
    ostats.stats_left(G, 6, 5, 4, 8, L, 1.0, 1.0)
    sub = g[6:10, 5:13]
    assert np.array_equal(L[:, :4], (sub @ sub.T).astype(np.float32))
    assert np.all(L[:, 4:] == 0)
    R = np.zeros((8, 8), np.float32)
    ostats.stats_right(G, 6, 5, 4, 8, R, 1.0, 1.0)
    assert np.array_equal(R, (sub.T @ sub).astype(np.float32))


def test_sequential_ascending_order_contract():
    # Products [1, 2^-24, 2^-55 x 8]: the ascending fp64 chain absorbs each 2^-55
    # (below half an ulp of 1) and ends on the fp32 tie 1 + 2^-24 -> 1.0f; any
    # descending / tree order or a single rounding would give 1 + 2^-23.
    a = np.array([1.0, 2.0 ** -12] + [2.0 ** -27] * 8, np.float32)
    b = np.array([1.0, 2.0 ** -12] + [2.0 ** -28] * 8, np.float32)
    G = np.stack([a, b])
    L = _left(G)
    assert L[0, 1] == np.float32(1.0) and L[1, 0] == np.float32(1.0)
    exact = sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b))
    assert exact > Fraction(1) + Fraction(1, 2 ** 24)  # the contract is NOT the exactly rounded sum
    # Products [1, 2^-24, 2^-24]: fp64 accumulation gives 1 + 2^-23 exactly
    # (an fp32 accumulator would tie-round twice to 1.0).
    c = np.array([1.0, 2.0 ** -12, 2.0 ** -12], np.float32)
    L2 = _left(np.stack([c, c]))
    assert L2[0, 1] == np.float32(1.0 + 2.0 ** -23)


def test_epilogue_rounding_sequence():
    # t1 = weight*acc; t2 = decay*L; r = t1 + t2 (each RN in fp64), then (float) r.
    G = np.array([[3.0, 1.0]], np.float32)  # acc = 10
    L0 = np.array([[np.float32(0.1)]], np.float32)
    decay, weight = 0.999, 0.001
    want = np.float32(weight * 10.0 + decay * float(np.float32(0.1)))
    assert _left(G, decay, weight, L0)[0, 0] == want


def test_unrolled_two_step_ema():
    # beta2 = 0.999, L0 = eps I: L_2 = b^2 eps I + b(1-b) G1G1^T + (1-b) G2G2^T (Alg. 1)
    G1 = gaussian((6, 9), 11)
    G2 = gaussian((6, 9), 12)
    b, eps = 0.999, 1e-6
    L = (eps * np.eye(6)).astype(np.float32)
    L = _left(G1, b, 1 - b, L)
    L = _left(G2, b, 1 - b, L)
    g1, g2 = G1.astype(np.float64), G2.astype(np.float64)
    want = b * b * eps * np.eye(6) + b * (1 - b) * g1 @ g1.T + (1 - b) * g2 @ g2.T
    np.testing.assert_allclose(L, want, rtol=1e-6, atol=1e-8)


def test_zero_gradient_leaves_state_unchanged():
    L0 = _left(gaussian((5, 8), 3))
    assert np.array_equal(_left(np.zeros((5, 8), np.float32), 1.0, 1.0, L0), L0)


def test_trace_identity_and_symmetry():
    # tr(L) = tr(R) = sum_s ||G_s||_F^2 (from zero, beta2 = 1)
    Gs = [gaussian((12, 20), 20 + s) for s in range(4)]
    L = np.zeros((12, 12), np.float32)
    R = np.zeros((20, 20), np.float32)
    for G in Gs:
        L = _left(G, 1.0, 1.0, L)
        R = _right(G, 1.0, 1.0, R)
    fro = sum(float(np.sum(G.astype(np.float64) ** 2)) for G in Gs)
    assert abs(np.trace(L.astype(np.float64)) - fro) <= 1e-6 * fro
    assert abs(np.trace(R.astype(np.float64)) - fro) <= 1e-6 * fro
    assert np.array_equal(L, L.T) and np.array_equal(R, R.T)


def test_diag_is_diagonal_of_full_adagrad():
    # D = diag(sum_s vec(G_s) vec(G_s)^T), brute force on a tiny shape
    Gs = [gaussian((3, 4), 40 + s) for s in range(5)]
    D = np.zeros((3, 4), np.float32)
    H = np.zeros((12, 12))
    nums = []
    for G in Gs:
        nums.append(ostats.diag_update(G, 0, 0, 3, 4, D))
        v = G.astype(np.float64).reshape(-1)  # row-major vec
        H += np.outer(v, v)
    np.testing.assert_allclose(D.reshape(-1), np.diag(H), rtol=1e-6)
    # graft numerator of the last step: ||D^{-1/2} o G||^2
    g = Gs[-1].astype(np.float64)
    np.testing.assert_allclose(nums[-1], np.sum(g * g / D.astype(np.float64)), rtol=1e-12)


def test_diag_floor_and_zero():
    D = np.zeros((2, 3), np.float32)
    G = np.zeros((2, 3), np.float32)
    assert ostats.diag_update(G, 0, 0, 2, 3, D) == 0.0 and np.all(D == 0)  # floor 1e-30, no NaN


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_block_rejected(bad):
    shapes = [(8, 8), (4, 6)]
    pl = oplan.plan(shapes, 4, 4096, 1)
    Gs = [gaussian(s, 50 + i) for i, s in enumerate(shapes)]
    Gs[0][5, 6] = bad  # inside block (row-block 1, col-block 1) of tensor 0
    Ds = [np.zeros(s, np.float32) for s in shapes]
    stats = np.zeros(pl.stats_elems, np.float32)
    num, status = ostats.stats_update(Gs, Ds, pl, stats, 1.0, 1.0)
    bad_blocks = [i for i, b in enumerate(pl.blocks) if b.tensor_id == 0 and b.row0 == 4 and b.col0 == 4]
    assert list(np.nonzero(status)[0]) == bad_blocks and status[bad_blocks[0]] == 2
    b = pl.blocks[bad_blocks[0]]
    assert np.all(stats[b.left_off:b.left_off + 16] == 0) and np.all(Ds[0][4:8, 4:8] == 0)
    assert num[bad_blocks[0]] == 0.0
    assert np.all(np.isfinite(stats))


def test_only_owner_updates_owned_statistics():
    shapes = [(8, 8)]
    pl = oplan.plan(shapes, 4, 4096, 2)
    G = [gaussian((8, 8), 60)]
    full = np.zeros(pl.stats_elems, np.float32)
    ostats.stats_update(G, [np.zeros((8, 8), np.float32)], pl, full, 1.0, 1.0)
    for r in range(2):
        part = np.zeros(pl.stats_elems, np.float32)
        D = np.zeros((8, 8), np.float32)
        ostats.stats_update(G, [D], pl, part, 1.0, 1.0, only_owner=r)
        seg = slice(r * pl.segment_elems, (r + 1) * pl.segment_elems)
        assert np.array_equal(part[seg], full[seg])
        other = np.ones(pl.stats_elems, bool)
        other[seg] = False
        assert np.all(part[other] == 0)
        assert np.all(D > 0)  # D always updated on every rank
