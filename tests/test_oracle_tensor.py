"""Pins for the tensor oracle (row f3): plan invariants and its reduction to the
(already pinned) matrix plan, brute-force mode statistics, the chunked
sequential contract by an order-sensitive construction, the Kronecker identity
of mode products, and the closed form of tensor Shampoo on a rank-one tensor
(exponents summing to -1/2).  CPU only."""

import itertools

import numpy as np
import pytest

import synth
from oracle import plan as oplan
from oracle import precondition as opre
from oracle import root as oroot
from oracle import stats as ostats
from oracle import tensor as ot


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


# ------------------------------------------------------------------- plan

def test_resnet50_parameter_count_and_plan_tiling():
    shapes = [s for _, s in synth.resnet50_shapes()]
    assert sum(int(np.prod(s)) for s in shapes) == 25_557_032
    pl = ot.plan(shapes, 1024, 8192, 4)
    covered = [np.zeros(s, np.int8) for s in shapes]
    for b in pl.blocks:
        covered[b.tensor_id][b.slices()] += 1
        kept = [b.p[i] for i in range(b.order) if b.p[i]]
        if kept:  # exponents -1/p of the kept modes sum to -1/2
            assert sum(1.0 / p for p in kept) == pytest.approx(0.5)
        assert all(b.extent[i] <= 1024 for i in range(b.order))
    assert all(np.all(c == 1) for c in covered)  # blocks tile every tensor exactly once
    # conv kernels [3,3,c,c]: 4 kept modes -> p = 8; [1,1,c,c']: the size-1 modes are skipped -> p = 4
    b0 = next(b for b in pl.blocks if b.tensor_id == 0)           # conv1 7x7x3x64
    assert b0.p[:4] == [8, 8, 8, 8]
    i11 = next(i for i, s in enumerate(shapes) if s == (1, 1, 64, 64))
    b11 = next(b for b in pl.blocks if b.tensor_id == i11)
    assert b11.p[:4] == [0, 0, 4, 4]
    ibn = next(i for i, s in enumerate(shapes) if len(s) == 1)
    bbn = next(b for b in pl.blocks if b.tensor_id == ibn)
    assert bbn.p[:1] == [2] and bbn.order == 1


@pytest.mark.parametrize("W", [1, 3])
def test_order2_plan_equals_matrix_plan(W):
    shapes = [s for _, s in synth.transformer_big_shapes()][:20] + [(1, 10), (300, 7), (2000, 1500)]
    pm = oplan.plan(shapes, 512, 4096, W)
    pt = ot.plan(shapes, 512, 4096, W)
    assert len(pm.blocks) == len(pt.blocks) and pm.stats_elems == pt.stats_elems
    for bm, bt in zip(pm.blocks, pt.blocks):
        assert (bm.row0, bm.col0, bm.rows, bm.cols) == (bt.origin[0], bt.origin[1], bt.extent[0], bt.extent[1])
        assert (bm.p_left, bm.p_right) == tuple(bt.p[:2])
        assert (bm.owner_left, bm.owner_right) == tuple(bt.owner[:2])
        assert (bm.left_off, bm.right_off) == tuple(bt.off[:2])
    assert [(g.owner, g.n, g.p, g.offset, g.count, g.stride) for g in pm.groups] == \
           [(g.owner, g.n, g.p, g.offset, g.count, g.stride) for g in pt.groups]


def test_plan_block_order_is_row_major_over_the_grid():
    pl = ot.plan([(5, 3, 7)], 2, 64, 1)
    origins = [tuple(b.origin[:3]) for b in pl.blocks]
    want = [(i, j, k) for i in (0, 2, 4) for j in (0, 2) for k in (0, 2, 4, 6)]
    assert origins == want
    assert pl.blocks[-1].extent[:3] == [1, 1, 1]


# ------------------------------------------------------------------ statistics

def _brute_mode_stat(B, mode):
    n = B.shape[mode]
    H = np.zeros((n, n))
    others = [range(d) for i, d in enumerate(B.shape) if i != mode]
    for a in range(n):
        for b in range(n):
            s = 0.0
            for rest in itertools.product(*others):
                ia = list(rest)
                ia.insert(mode, a)
                ib = list(rest)
                ib.insert(mode, b)
                s += float(B[tuple(ia)]) * float(B[tuple(ib)])
            H[a, b] = s
    return H


def test_mode_statistics_brute_force_order3_and_4():
    for shape in ((3, 4, 5), (2, 3, 2, 4)):
        G = synth.conv_gradient(shape, 11)
        pl = ot.plan([shape], 64, 64, 1)
        stats = np.zeros(pl.stats_elems, np.float32)
        D = [np.zeros(shape, np.float32)]
        ot.stats_update([G], D, pl, stats, 1.0, 1.0)
        b = pl.blocks[0]
        for i in range(len(shape)):
            H = ot.root_view(stats, b.off[i], b.extent[i], b.ld[i])
            want = _brute_mode_stat(G.astype(np.float64), i)
            assert np.max(np.abs(H - want)) <= 1e-6 * np.max(np.abs(want))
            assert np.array_equal(H, H.T)
            # trace identity: tr(H_i) = ||G||_F^2 for every mode
            assert np.trace(H.astype(np.float64)) == pytest.approx(float(np.sum(G.astype(np.float64) ** 2)), rel=1e-6)
        np.testing.assert_array_equal(D[0], (G.astype(np.float64) ** 2).astype(np.float32))


def test_order2_statistics_bit_exact_with_matrix_oracle():
    shapes = [(40, 70), (130, 33)]
    Gs = [synth.lowrank_gradient(m, n, 5 + m) for m, n in shapes]
    pm = oplan.plan(shapes, 64, 4096, 1)
    pt = ot.plan(shapes, 64, 4096, 1)
    sm = np.zeros(pm.stats_elems, np.float32)
    st = np.zeros(pt.stats_elems, np.float32)
    for step in range(2):
        Dm = [np.zeros(s, np.float32) for s in shapes]
        Dt = [np.zeros(s, np.float32) for s in shapes]
        nm, _ = ostats.stats_update(Gs, Dm, pm, sm, 0.9, 0.1)
        nt, _ = ot.stats_update(Gs, Dt, pt, st, 0.9, 0.1)
        assert np.array_equal(sm.view(np.uint32), st.view(np.uint32))
        assert all(np.array_equal(a, b) for a, b in zip(Dm, Dt))
        np.testing.assert_allclose(nt, nm, rtol=1e-13)


def test_chunked_contract_order_sensitive():
    # u = [2^30, 1 x (C-1) | 1 x C]: the sequential chunk 0 loses its ones
    # (ulp(2^60) = 256), chunk 1 sums them exactly: acc = 2^60 + 4096.  With the
    # old value -2^60 (decay = weight = 1) the stored result is the chunk-1 sum,
    # 4096.  One sequential sum would give 0; a descending one 8192.
    C = ot.STAT_CHUNK
    U = np.ones((1, 2 * C), np.float32)
    U[0, 0] = 2.0 ** 30
    S = np.array([[-(2.0 ** 60)]], np.float32)
    ostats.mode_stat(U, S, C, 1.0, 1.0)
    assert S[0, 0] == 4096.0
    S = np.array([[-(2.0 ** 60)]], np.float32)
    ostats.mode_stat(U, S, 4 * C, 1.0, 1.0)  # one chunk: the matrix contract
    assert S[0, 0] == 0.0


def test_non_finite_block_is_rejected():
    G = synth.conv_gradient((3, 4, 5), 3)
    G[1, 2, 3] = np.nan
    pl = ot.plan([G.shape], 64, 64, 1)
    stats = np.full(pl.stats_elems, 7.0, np.float32)
    D = [np.ones(G.shape, np.float32)]
    num, st = ot.stats_update([G], D, pl, stats, 1.0, 1.0)
    assert st[0] == 2 and num[0] == 0 and np.all(stats == 7.0) and np.all(D[0] == 1.0)


# ------------------------------------------------------------------ mode products, preconditioning

def test_mode_products_are_the_kronecker_product():
    g = synth.rng(21)
    G = g.standard_normal((3, 4, 5))
    A, B, C = g.standard_normal((3, 3)), g.standard_normal((4, 4)), g.standard_normal((5, 5))
    P = ot.mode_product(ot.mode_product(ot.mode_product(G, A, 0), B, 1), C, 2)
    np.testing.assert_allclose(P.reshape(-1), np.kron(np.kron(A, B), C) @ G.reshape(-1), rtol=1e-12, atol=1e-12)
    # order 2: X_L G X_R with symmetric roots
    M = g.standard_normal((4, 6))
    XL = g.standard_normal((4, 4))
    XL = XL + XL.T
    XR = g.standard_normal((6, 6))
    XR = XR + XR.T
    np.testing.assert_allclose(ot.mode_product(ot.mode_product(M, XL, 0), XR, 1),
                               opre.precondition_block(M, XL, XR), rtol=1e-12, atol=1e-12)


def _full_step(shapes, Gs, eps=1e-6):
    pl = ot.plan(shapes, 1024, 8192, 1)
    stats = np.zeros(pl.stats_elems, np.float32)
    Ds = [np.zeros(s, np.float32) for s in shapes]
    num, _ = ot.stats_update(Gs, Ds, pl, stats, 1.0, 1.0)
    roots = np.zeros(pl.stats_elems)
    for b in pl.blocks:
        for i in range(b.order):
            if b.p[i]:
                A = ot.root_view(stats, b.off[i], b.extent[i], b.ld[i]).astype(np.float64)
                X, info = oroot.inverse_pth_root(A, b.p[i], eps_rel=eps, tol=1e-13)
                roots[b.off[i]:b.off[i] + b.extent[i] * b.ld[i]].reshape(b.extent[i], b.ld[i])[:, :b.extent[i]] = X
    return pl, Ds, num, roots


@pytest.mark.parametrize("shape", [(12,), (6, 9), (3, 4, 5), (3, 3, 4, 6)])
def test_rank_one_tensor_closed_form(shape):
    # one step on G = a o b o c ...: every mode statistic is ||G||^2 u_i u_i^T, so
    # X_i u_i = (||G||^2 (1+eps))^{-1/p} u_i with p = 2k and P = G / sqrt(||G||^2 (1+eps))
    g = synth.rng(31)
    G = np.ones(())
    for d in shape:
        G = np.multiply.outer(G, g.standard_normal(d) + 2.0)
    G = G.astype(np.float32)
    # (ridge 1e-2: dominates the fp32 rounding of the stored rank-one statistic)
    pl, Ds, num, roots = _full_step([shape], [G], eps=1e-2)
    Ps, scales, dens = ot.precondition_plan([G], Ds, pl, roots, num)
    Gd = G.astype(np.float64)
    want = Gd / np.sqrt(np.sum(Gd ** 2) * (1 + 1e-2))
    assert rel(Ps[0], want) < 1e-6
    # grafting identity: ||scale * P|| = sqrt(num)
    assert np.sqrt(dens[0]) * scales[0] == pytest.approx(np.sqrt(num[0]), rel=1e-10)


def test_order2_precondition_equals_matrix_oracle():
    shapes = [(70, 50)]
    Gs = [synth.lowrank_gradient(70, 50, 8)]
    pl, Ds, num, roots = _full_step(shapes, Gs)
    Pt, st, _ = ot.precondition_plan(Gs, Ds, pl, roots, num)
    pm = oplan.plan(shapes, 1024, 8192, 1)
    Pm, sm, _ = opre.precondition_plan(Gs, Ds, pm, roots, num)
    np.testing.assert_allclose(Pt[0], Pm[0], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(st, sm, rtol=1e-12)


def test_diagonal_only_block():
    # a (1, 1, 1, 9000) tensor with max_precond_dim 4096: no kept mode -> D^{-1/2} o G
    shape = (1, 1, 1, 9000)
    G = synth.gaussian(shape, 4)
    pl = ot.plan([shape], 9000, 4096, 1)
    assert len(pl.blocks) == 1 and not any(pl.blocks[0].p)
    Ds = [np.zeros(shape, np.float32)]
    num, _ = ot.stats_update([G], Ds, pl, np.zeros(0, np.float32), 1.0, 1.0)
    Ps, sc, _ = ot.precondition_plan([G], Ds, pl, np.zeros(0), num)
    np.testing.assert_allclose(Ps[0], np.sign(G), rtol=1e-6)
    assert sc[0] == pytest.approx(1.0)
