"""GPU parity: the CUDA path (through the C ABI) against the CPU fp64 oracle on
identical seeded inputs.  Bars (BASELINE.json north star):
  * plan, statistics L/R and D: bit-exact;
  * roots: relative Frobenius error <= 1e-3 (north star); the FP64-DMMA path
    is additionally held to 2e-6 (fp32 output rounding + fp64 iteration);
  * preconditioned gradient: relative Frobenius error <= 1e-3 (held to 2e-5:
    3xTF32 tcgen05 products, ~1e-6 measured);
  * graft numerator / scale: relative 1e-9 / 1e-5.
"""

import numpy as np
import pytest
import torch

import synth
from oracle import plan as oplan
from oracle import precondition as opre
from oracle import root as oroot
from oracle import stats as ostats

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def shp():
    import paper_2002_09018_b200 as shp
    return shp


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def bits(x):
    return np.asarray(x, np.float32).view(np.uint32)


# ---------------------------------------------------------------- statistics

def _run_stats_both(shp, shapes, Gs_np, block_size, decay, weight, steps=1, W=1, only_owner=-1, stats0=None):
    pl_o = oplan.plan(shapes, block_size, 8192, W)
    pl = shp.make_plan(shapes, block_size, 8192, W)
    stats_o = np.zeros(pl_o.stats_elems, np.float32) if stats0 is None else stats0.copy()
    Ds_o = [np.zeros(s, np.float32) for s in shapes]
    Gd = [torch.from_numpy(G).to(DEV) for G in Gs_np[0]]
    Dd = [torch.zeros(s, dtype=torch.float32, device=DEV) for s in shapes]
    table = shp.TensorTable(Gd, Dd)
    stats = torch.from_numpy(stats_o.copy()).to(DEV)
    gn = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    bs = torch.full((pl.n_blocks,), -1, dtype=torch.int32, device=DEV)
    for s in range(steps):
        for G, g in zip(Gd, Gs_np[s]):
            G.copy_(torch.from_numpy(g))
        shp.stats_update(table, pl, stats, decay, weight, only_owner, gn, bs)
        num_o, st_o = ostats.stats_update(Gs_np[s], Ds_o, pl_o, stats_o, decay, weight, only_owner)
    torch.cuda.synchronize()
    return (stats.cpu().numpy(), [D.cpu().numpy() for D in Dd], gn.cpu().numpy(), bs.cpu().numpy(),
            stats_o, Ds_o, num_o, st_o)


@pytest.mark.parametrize("decay,weight", [(1.0, 1.0), (0.999, 0.001)])
def test_stats_bit_exact_small(shp, decay, weight):
    shapes = [(64, 32), (300, 200), (1, 10), (130, 5), (257, 129)]
    Gs = [[synth.gaussian(s, 100 + 10 * st + i) for i, s in enumerate(shapes)] for st in range(2)]
    st, Ds, gn, bs, st_o, Ds_o, gn_o, bs_o = _run_stats_both(shp, shapes, Gs, 128, decay, weight, steps=2)
    assert np.array_equal(bits(st), bits(st_o))
    for D, Do in zip(Ds, Ds_o):
        assert np.array_equal(bits(D), bits(Do))
    np.testing.assert_allclose(gn, gn_o, rtol=1e-12)
    assert np.all(bs == 0) and np.all(bs_o == 0)


def test_stats_order_sensitive_rows(shp):
    # same construction as the oracle pin: ascending fp64 chain -> 1.0f, fp64 (not fp32) accumulation
    a = np.array([1.0, 2.0 ** -12] + [2.0 ** -27] * 8 + [0.0] * 22, np.float32)
    b = np.array([1.0, 2.0 ** -12] + [2.0 ** -28] * 8 + [0.0] * 22, np.float32)
    c = np.zeros(32, np.float32)
    c[:3] = [1.0, 2.0 ** -12, 2.0 ** -12]
    G = np.stack([a, b, c, c] + [synth.gaussian((32,), 7 + i) for i in range(4)])
    st, _, _, _, st_o, _, _, _ = _run_stats_both(shp, [G.shape], [[G]], 1024, 1.0, 1.0)
    assert np.array_equal(bits(st), bits(st_o))
    b = oplan.plan([G.shape], 1024, 8192, 1).blocks[0]
    L = st[b.left_off: b.left_off + 8 * b.left_ld].reshape(8, b.left_ld)
    assert L[0, 1] == np.float32(1.0) and L[2, 3] == np.float32(1.0 + 2.0 ** -23)


def test_stats_nonfinite_block_unchanged(shp):
    shapes = [(256, 256)]
    G = synth.gaussian(shapes[0], 5)
    G[200, 10] = np.nan
    st, Ds, gn, bs, st_o, Ds_o, gn_o, bs_o = _run_stats_both(shp, shapes, [[G]], 128, 1.0, 1.0)
    assert list(bs) == list(bs_o) and bs.tolist().count(2) == 1
    assert np.array_equal(bits(st), bits(st_o))
    assert np.array_equal(bits(Ds[0]), bits(Ds_o[0]))


@pytest.mark.parametrize("W", [2, 3])
def test_stats_only_owner(shp, W):
    shapes = [(256, 384), (128, 128)]
    Gs = [[synth.gaussian(s, 30 + i) for i, s in enumerate(shapes)]]
    for r in range(W):
        st, Ds, _, _, st_o, Ds_o, _, _ = _run_stats_both(shp, shapes, Gs, 128, 1.0, 1.0, W=W, only_owner=r)
        assert np.array_equal(bits(st), bits(st_o))
        assert np.array_equal(bits(Ds[0]), bits(Ds_o[0]))


def test_stats_transformer_big_sampled_blocks(shp):
    """Config 3 at full size (b = 1024, 360 blocks, 624 statistics, one launch
    sequence); the oracle recomputes sampled blocks one by one."""
    shapes = [s for _, s in synth.transformer_big_shapes()]
    pl = shp.make_plan(shapes, 1024, 8192, 1)
    pl_o = oplan.plan(shapes, 1024, 8192, 1)
    Gd = [synth.lowrank_gradient_device(m, n, synth.BASE_SEED + 3 + i, DEV) for i, (m, n) in enumerate(shapes)]
    Dd = [torch.zeros_like(G) for G in Gd]
    stats = torch.zeros(pl.stats_elems, dtype=torch.float32, device=DEV)
    gn = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    shp.stats_update(shp.TensorTable(Gd, Dd), pl, stats, 1.0, 1.0, -1, gn)
    torch.cuda.synchronize()
    sample = [0, 31, 95, 96, 100, 359]  # vocab block, ragged vocab (256 rows), first attention, FFN...
    sample = [b for b in sample if b < pl.n_blocks]
    Gs_np = [None] * len(shapes)
    for bi in sample:
        t = pl_o.blocks[bi].tensor_id
        if Gs_np[t] is None:
            Gs_np[t] = Gd[t].cpu().numpy()
    Ds_o = [np.zeros(s, np.float32) if g is not None else None for s, g in zip(shapes, Gs_np)]
    stats_o = np.zeros(pl_o.stats_elems, np.float32)
    num_o, _ = ostats.stats_update(Gs_np, Ds_o, pl_o, stats_o, 1.0, 1.0, blocks=sample)
    st = stats.cpu().numpy()
    gnh = gn.cpu().numpy()
    for bi in sample:
        b = pl_o.blocks[bi]
        for p, n, off, ld in ((b.p_left, b.rows, b.left_off, b.left_ld), (b.p_right, b.cols, b.right_off, b.right_ld)):
            if p:
                seg = slice(off, off + n * ld)
                assert np.array_equal(bits(st[seg]), bits(stats_o[seg])), (bi, p)
        t = b.tensor_id
        Dg = Dd[t][b.row0:b.row0 + b.rows, b.col0:b.col0 + b.cols].cpu().numpy()
        assert np.array_equal(bits(Dg), bits(Ds_o[t][b.row0:b.row0 + b.rows, b.col0:b.col0 + b.cols]))
        assert abs(gnh[bi] - num_o[bi]) <= 1e-12 * abs(num_o[bi])


# --------------------------------------------------------------------- roots

def _roots_both(shp, As, p, eps=1e-6, tol=1e-7, max_iter=100):
    A = torch.from_numpy(np.ascontiguousarray(As)).to(DEV)
    X, info = shp.inverse_pth_root_batched(A, p, eps_rel=eps, tol=tol, max_iter=max_iter)
    torch.cuda.synchronize()
    Xg = X.cpu().numpy()
    inf = shp.info_to_numpy(info)
    outs = [oroot.inverse_pth_root(a.astype(np.float64), p, eps, tol, max_iter) for a in As]
    return Xg, inf, outs


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_root_config1_kappa_1e6(shp, p):
    G = synth.gaussian((64, 32), synth.BASE_SEED + 1)
    L = G.astype(np.float64) @ G.astype(np.float64).T
    R = G.astype(np.float64).T @ G.astype(np.float64)
    for A in (L.astype(np.float32), R.astype(np.float32)):
        Xg, inf, outs = _roots_both(shp, A[None], p)
        Xo, io = outs[0]
        assert rel(Xg[0], Xo) < 2e-6
        assert inf[0]["status"] == io.status == 0
        assert abs(int(inf[0]["iters"]) - io.iters) <= 1
        assert abs(inf[0]["lambda_max"] - io.lambda_max) <= 1e-12 * io.lambda_max


@pytest.mark.parametrize("n", [128, 200, 512])
def test_root_config2_batches(shp, n):
    count = 4 if n == 512 else 8
    As = synth.psd_batch(n, count, synth.BASE_SEED + 2 + n, "mixed")
    Xg, inf, outs = _roots_both(shp, As, 4)
    for i, (Xo, io) in enumerate(outs):
        assert rel(Xg[i], Xo) < 2e-6, i
        assert inf[i]["status"] == io.status
        assert abs(int(inf[i]["iters"]) - io.iters) <= 1


def test_root_1024_two_matrices(shp):
    As = synth.psd_batch(1024, 2, synth.BASE_SEED + 2, "wishart")
    Xg, inf, outs = _roots_both(shp, As, 4)
    for i, (Xo, io) in enumerate(outs):
        assert rel(Xg[i], Xo) < 2e-6
        assert inf[i]["status"] == 0 and abs(int(inf[i]["iters"]) - io.iters) <= 1


def test_root_edge_cases(shp):
    n = 40
    As = np.zeros((5, n, n), np.float32)
    As[0] = np.eye(n)                                    # identity -> (1+eps)^{-1/4} I, 0 iterations
    As[1] = synth.wishart(n, 3)
    As[2] = 0.0                                          # degenerate -> I, status 3
    As[3] = synth.wishart(n, 4)
    As[3][5, 7] = As[3][7, 5] = np.nan                   # non-finite -> untouched, status 2
    As[4] = np.diag(np.linspace(1.0, 2.0, n)).astype(np.float32) * 16.0 ** 3
    A = torch.from_numpy(As).to(DEV)
    X = torch.full_like(A, 7.0)
    from paper_2002_09018_b200 import info_to_numpy
    X, info = shp.inverse_pth_root_batched(A, 4, X=X)
    torch.cuda.synchronize()
    Xg, inf = X.cpu().numpy(), info_to_numpy(info)
    assert inf[0]["status"] == 0 and inf[0]["iters"] == 0
    np.testing.assert_allclose(Xg[0], (1 + 1e-6) ** -0.25 * np.eye(n), rtol=1e-7, atol=0)
    assert inf[2]["status"] == 3 and np.array_equal(Xg[2], np.eye(n, dtype=np.float32))
    assert inf[3]["status"] == 2 and np.all(Xg[3] == 7.0)
    for i in (1, 4):
        Xo, io = oroot.inverse_pth_root(As[i].astype(np.float64), 4)
        assert rel(Xg[i], Xo) < 2e-6 and inf[i]["status"] == io.status


def test_root_n1_and_p_variants(shp):
    As = np.array([[[7.25]]], np.float32)
    for p in (1, 2, 4, 8):
        Xg, inf, outs = _roots_both(shp, As, p, tol=1e-14)
        assert abs(Xg[0, 0, 0] - (7.25 * (1 + 1e-6)) ** (-1.0 / p)) <= 2e-7 * Xg[0, 0, 0]


def test_root_not_converged_and_stagnation(shp):
    As = synth.psd_batch(64, 2, 77, "wishart")
    Xg, inf, outs = _roots_both(shp, As, 4, max_iter=3)
    for i, (Xo, io) in enumerate(outs):
        assert inf[i]["status"] == io.status == 1 and inf[i]["iters"] == io.iters == 3
        assert rel(Xg[i], Xo) < 1e-5
    Xg, inf, outs = _roots_both(shp, As, 4, tol=0.0, max_iter=200)  # tol unreachable -> stagnation guard
    for i, (Xo, io) in enumerate(outs):
        assert inf[i]["status"] == 1 and inf[i]["iters"] < 60
        assert rel(Xg[i], Xo) < 2e-6


def test_root_determinism(shp):
    As = torch.from_numpy(synth.psd_batch(256, 3, 11, "mixed")).to(DEV)
    X1, _ = shp.inverse_pth_root_batched(As, 4)
    X2, _ = shp.inverse_pth_root_batched(As, 4)
    torch.cuda.synchronize()
    assert torch.equal(X1, X2)


def test_residual_kernel_vs_oracle(shp):
    from paper_2002_09018_b200 import info_to_numpy
    for n, p in ((64, 4), (200, 2), (130, 8)):
        As = synth.psd_batch(n, 2, 900 + n, "mixed")
        outs = [oroot.inverse_pth_root(a.astype(np.float64), p) for a in As]
        # roots are symmetric by contract; symmetrize the oracle's (rounding-asymmetric) fp64 roots
        Xo32 = np.stack([((o[0] + o[0].T) * 0.5).astype(np.float32) for o in outs])
        info = np.zeros(2, shp.ROOT_INFO_DTYPE)
        info["lambda_max"] = [o[1].lambda_max for o in outs]
        info_d = torch.from_numpy(info.view(np.uint8).copy()).to(DEV)
        res = shp.root_residual_batched(torch.from_numpy(As).to(DEV), torch.from_numpy(Xo32).to(DEV), p, info_d)
        res = res.cpu().numpy()
        for i, o in enumerate(outs):
            want = oroot.residual(As[i], Xo32[i], p, 1e-6, o[1].lambda_max)
            assert abs(res[i] - want) <= 1e-6 * max(want, 1e-12), (n, p, res[i], want)
    # GPU roots satisfy the invariant as well as the oracle's root rounded to fp32
    # does: with kappa ~ 1e6 the fp32 storage of X alone makes ||X^p A_hat - I||_F
    # O(p * 2^-24 * kappa * sqrt(n)), so the bar is relative to that floor.
    As = synth.psd_batch(128, 2, 5, "wishart")
    X, info = shp.inverse_pth_root_batched(torch.from_numpy(As).to(DEV), 4)
    res = shp.root_residual_batched(torch.from_numpy(As).to(DEV), X, 4, info).cpu().numpy()
    for i in range(2):
        Xo, io = oroot.inverse_pth_root(As[i].astype(np.float64), 4)
        floor = oroot.residual(As[i], ((Xo + Xo.T) * 0.5).astype(np.float32), 4, 1e-6, io.lambda_max)
        assert res[i] < 3.0 * floor + 1e-9, (res[i], floor)


# -------------------------------------------------------------- precondition

def _pack_roots(pl_o, roots_fn):
    roots = np.zeros(pl_o.stats_elems, np.float32)
    for b in pl_o.blocks:
        for side, p, n, off, ld in ((0, b.p_left, b.rows, b.left_off, b.left_ld), (1, b.p_right, b.cols, b.right_off, b.right_ld)):
            if p:
                roots[off:off + n * ld].reshape(n, ld)[:, :n] = roots_fn(b, side, n)
    return roots


def test_precondition_with_oracle_roots(shp):
    # max_precond_dim 256, block 128: two-sided (ragged), right-only, left-only,
    # diagonal-only (both sides skipped) and a 1 x n row (right-only, p = 2)
    shapes = [(200, 240), (300, 100), (100, 300), (300, 300), (1, 50)]
    block = 128
    pl_o = oplan.plan(shapes, block, 256, 1)
    pl = shp.make_plan(shapes, block, 256, 1)
    kinds = {(b.p_left > 0, b.p_right > 0) for b in pl_o.blocks}
    assert kinds == {(True, True), (False, True), (True, False), (False, False)}
    Gs = [synth.gaussian(s, 60 + i) for i, s in enumerate(shapes)]
    Ds = [np.abs(synth.gaussian(s, 70 + i)) + 0.01 for i, s in enumerate(shapes)]

    def rf(b, side, n):
        M = synth.wishart(n, 1000 + b.block_index * 2 + side).astype(np.float64) + np.eye(n)
        return oroot.inverse_pth_root(M, b.p_left if side == 0 else b.p_right)[0].astype(np.float32)

    roots = _pack_roots(pl_o, rf)
    num = np.arange(1, pl_o.blocks.__len__() + 1, dtype=np.float64)
    Ps_o, sc_o, den_o = opre.precondition_plan(Gs, Ds, pl_o, roots.astype(np.float64), num)
    Gd = [torch.from_numpy(G).to(DEV) for G in Gs]
    Dd = [torch.from_numpy(D).to(DEV) for D in Ds]
    Pd = [torch.full(s, np.nan, dtype=torch.float32, device=DEV) for s in shapes]
    table = shp.TensorTable(Gd, Dd, Pd)
    sc = torch.zeros(pl.n_blocks, dtype=torch.float32, device=DEV)
    den = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    shp.precondition(table, pl, torch.from_numpy(roots).to(DEV), torch.from_numpy(num).to(DEV), sc, den)
    torch.cuda.synchronize()
    for t, (P, Po) in enumerate(zip(Pd, Ps_o)):
        Pg = P.cpu().numpy()
        for b in (bb for bb in pl_o.blocks if bb.tensor_id == t):
            sl = (slice(b.row0, b.row0 + b.rows), slice(b.col0, b.col0 + b.cols))
            assert rel(Pg[sl], Po[sl]) < 2e-5, (t, b.block_index)  # 3xTF32 tcgen05 / fp64 DMMA
    np.testing.assert_allclose(den.cpu().numpy(), den_o, rtol=1e-5)
    np.testing.assert_allclose(sc.cpu().numpy(), sc_o, rtol=1e-5)


def test_precondition_one_sided_rank_deficient(shp):
    """Right-only vocabulary blocks (rows <= cols: the INT8 Ozaki path, oz_precondition.cu) whose statistic is
    rank-deficient: G_b has a few nonzero rows, R_b = G_b^T G_b + the ridge has kappa ~1e6 and X_R is largest
    exactly where G_b's rows vanish, so P = G_b X_R cancels ~kappa^{1/2}.  With the ORACLE's roots (fp32) the
    product must match the oracle's fp64 product to fp32 rounding -- an fp32 accumulation (3xTF32) was 6.2e-3 off
    on such a block (r02c).  Ragged last block (rows 300 of 512), a block with 3 nonzero rows."""
    m, n, block = 1324, 512, 512
    G = np.zeros((m, n), np.float32)
    rng = np.random.default_rng(synth.BASE_SEED + 321)
    for r in rng.choice(512, 40, replace=False):           # block 0: 40 nonzero rows
        G[r] = rng.normal(0, 0.01, n)
    for r in 512 + rng.choice(512, 3, replace=False):      # block 1: 3 nonzero rows
        G[r] = rng.normal(0, 0.01, n)
    for r in 1024 + rng.choice(300, 12, replace=False):    # block 2 (ragged, 300 rows): 12 nonzero rows
        G[r] = rng.normal(0, 0.01, n)
    shapes = [(m, n)]
    pl_o = oplan.plan(shapes, block, 1024, 1)
    pl = shp.make_plan(shapes, block, 1024, 1)
    assert all(b.p_left == 0 and b.p_right == 2 for b in pl_o.blocks) and len(pl_o.blocks) == 3
    stats_o = np.zeros(pl_o.stats_elems, np.float32)
    D_o = [np.zeros(G.shape, np.float32)]
    num_o, _ = ostats.stats_update([G], D_o, pl_o, stats_o, 1.0, 1.0)

    def rf(b, side, nn):
        A = stats_o[b.right_off:b.right_off + nn * b.right_ld].reshape(nn, b.right_ld)[:, :nn].astype(np.float64)
        return oroot.inverse_pth_root(A, 2)[0].astype(np.float32)

    roots = _pack_roots(pl_o, rf)
    Ps_o, sc_o, den_o = opre.precondition_plan([G], D_o, pl_o, roots.astype(np.float64), num_o)
    Pd = torch.full(G.shape, np.nan, dtype=torch.float32, device=DEV)
    table = shp.TensorTable([torch.from_numpy(G).to(DEV)], [torch.from_numpy(D_o[0]).to(DEV)], [Pd])
    sc = torch.zeros(pl.n_blocks, dtype=torch.float32, device=DEV)
    shp.precondition(table, pl, torch.from_numpy(roots).to(DEV), torch.from_numpy(num_o).to(DEV), sc)
    torch.cuda.synchronize()
    Pg = Pd.cpu().numpy()
    for b in pl_o.blocks:
        sl = (slice(b.row0, b.row0 + b.rows), slice(b.col0, b.col0 + b.cols))
        err = rel(Pg[sl], Ps_o[0][sl])
        print(f"one-sided block {b.block_index} ({b.rows} rows): P rel err {err:.3e}")
        assert err < 1e-6, (b.block_index, err)
    np.testing.assert_allclose(sc.cpu().numpy(), sc_o, rtol=1e-5)


# ---------------------------------------------------------------- full chain

def test_full_step_config1_chain(shp):
    """Config 1: one 64x32 gradient -> statistics -> both inverse 4th roots ->
    preconditioned gradient + graft scale, each side computed independently."""
    G = synth.gaussian((64, 32), synth.BASE_SEED + 1)
    shapes = [G.shape]
    pl_o = oplan.plan(shapes, 1024, 8192, 1)
    pl = shp.make_plan(shapes, 1024, 8192, 1)
    # oracle chain
    stats_o = np.zeros(pl_o.stats_elems, np.float32)
    D_o = [np.zeros(G.shape, np.float32)]
    num_o, _ = ostats.stats_update([G], D_o, pl_o, stats_o, 1.0, 1.0)
    b = pl_o.blocks[0]
    roots_o = np.zeros(pl_o.stats_elems, np.float64)
    for n, off, ld in ((b.rows, b.left_off, b.left_ld), (b.cols, b.right_off, b.right_ld)):
        A = stats_o[off:off + n * ld].reshape(n, ld)[:, :n].astype(np.float64)
        roots_o[off:off + n * ld].reshape(n, ld)[:, :n] = oroot.inverse_pth_root(A, 4)[0]
    Ps_o, sc_o, _ = opre.precondition_plan([G], D_o, pl_o, roots_o, num_o)
    # GPU chain
    Gd = torch.from_numpy(G).to(DEV)
    Dd = torch.zeros_like(Gd)
    Pd = torch.zeros_like(Gd)
    table = shp.TensorTable([Gd], [Dd], [Pd])
    stats = torch.zeros(pl.stats_elems, dtype=torch.float32, device=DEV)
    roots = torch.zeros_like(stats)
    gn = torch.zeros(1, dtype=torch.float64, device=DEV)
    sc = torch.zeros(1, dtype=torch.float32, device=DEV)
    shp.stats_update(table, pl, stats, 1.0, 1.0, -1, gn)
    shp.refresh_group_roots(pl, stats, roots, 0)
    shp.precondition(table, pl, roots, gn, sc)
    torch.cuda.synchronize()
    assert np.array_equal(bits(stats.cpu().numpy()), bits(stats_o))
    assert rel(Pd.cpu().numpy(), Ps_o[0]) < 2e-5
    assert abs(sc.cpu().numpy()[0] - sc_o[0]) <= 1e-5 * sc_o[0]


def test_precondition_tcgen05_large_blocks(shp):
    """1024-blocks (the bench's geometry: 32 k-tiles, 8x8 output tiles per block,
    two-sided + right-only) through the tcgen05 3xTF32 path.  The roots are
    arbitrary symmetric matrices with random signs (P = X_L G X_R is a plain
    definition); their sums cancel ~sqrt(K)-fold per product, so the fp32 TMEM
    accumulation shows up at ~1e-5 here (bar 1e-3; the PSD-root cases above
    land near 1e-6)."""
    shapes = [(1024, 2048), (2048, 1024), (3000, 512)]
    pl_o = oplan.plan(shapes, 1024, 2048, 1)
    pl = shp.make_plan(shapes, 1024, 2048, 1)

    def rf(b, side, n):
        S = synth.gaussian((n, n), 5000 + 2 * b.block_index + side).astype(np.float64) / np.sqrt(n)
        return ((S + S.T) * 0.5).astype(np.float32)

    roots = _pack_roots(pl_o, rf)
    Gs = [synth.lowrank_gradient(m, n, 80 + i) for i, (m, n) in enumerate(shapes)]
    Ds = [np.ones(s, np.float32) for s in shapes]
    num = np.ones(len(pl_o.blocks))
    Ps_o, sc_o, den_o = opre.precondition_plan(Gs, Ds, pl_o, roots.astype(np.float64), num)
    Gd = [torch.from_numpy(G).to(DEV) for G in Gs]
    Pd = [torch.full(s, np.nan, dtype=torch.float32, device=DEV) for s in shapes]
    table = shp.TensorTable(Gd, [torch.from_numpy(D).to(DEV) for D in Ds], Pd)
    den = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    shp.precondition(table, pl, torch.from_numpy(roots).to(DEV), None, None, den)
    torch.cuda.synchronize()
    worst = 0.0
    for t, (P, Po) in enumerate(zip(Pd, Ps_o)):
        Pg = P.cpu().numpy()
        for b in (bb for bb in pl_o.blocks if bb.tensor_id == t):
            sl = (slice(b.row0, b.row0 + b.rows), slice(b.col0, b.col0 + b.cols))
            e = rel(Pg[sl], Po[sl])
            worst = max(worst, e)
            assert e < 1e-4, (t, b.block_index, e)
    print("worst block rel err", worst)
    np.testing.assert_allclose(den.cpu().numpy(), den_o, rtol=1e-4)


def test_precondition_determinism(shp):
    shapes = [(1024, 1024)]
    pl = shp.make_plan(shapes, 1024, 8192, 1)
    G = torch.from_numpy(synth.lowrank_gradient(1024, 1024, 3)).to(DEV)
    roots = torch.randn(pl.stats_elems, device=DEV)
    P1, P2 = torch.zeros_like(G), torch.zeros_like(G)
    shp.precondition(shp.TensorTable([G], [torch.ones_like(G)], [P1]), pl, roots)
    shp.precondition(shp.TensorTable([G], [torch.ones_like(G)], [P2]), pl, roots)
    torch.cuda.synchronize()
    assert torch.equal(P1, P2)


def test_precondition_with_precomputed_roots_split(shp):
    """shampoo_precondition_split with roots_lo = tf32_split(roots) (once per
    refresh) gives bit-identical P and scales to the per-call split; the split
    itself equals x - trunc_tf32(x) computed on the host."""
    shapes = [(1024, 1024), (300, 2048), (32000 // 16, 1024)]
    pl = shp.make_plan(shapes, 1024, 8192, 1)
    Gs = [torch.from_numpy(synth.lowrank_gradient(m, n, 7 + m)).to(DEV) for m, n in shapes]
    roots = torch.randn(pl.stats_elems, device=DEV) * 0.05
    lo = shp.tf32_split(roots)
    r = roots.cpu().numpy()
    want = r - (r.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    assert np.array_equal(lo.cpu().numpy().view(np.uint32), want.view(np.uint32))
    gn = torch.ones(pl.n_blocks, dtype=torch.float64, device=DEV)
    outs = []
    for roots_lo in (None, lo):
        Ps = [torch.zeros_like(G) for G in Gs]
        sc = torch.zeros(pl.n_blocks, device=DEV)
        shp.precondition(shp.TensorTable(Gs, [torch.ones_like(G) for G in Gs], Ps), pl, roots, gn, sc,
                         roots_lo=roots_lo)
        torch.cuda.synchronize()
        outs.append((Ps, sc))
    for P1, P2 in zip(outs[0][0], outs[1][0]):
        assert torch.equal(P1, P2)
    assert torch.equal(outs[0][1], outs[1][1])


def test_root_results_independent_of_batch_size(shp):
    """A root must not depend on which other matrices share its launch: small
    batches split each matrix's power iteration over several CTAs, large ones
    use one CTA per matrix; both reduce in the same fixed order."""
    As = synth.psd_batch(64, 200, 31, "mixed")
    Xs, _ = shp.inverse_pth_root_batched(torch.from_numpy(As[:3]).to(DEV), 4)
    Xl, _ = shp.inverse_pth_root_batched(torch.from_numpy(As).to(DEV), 4)
    torch.cuda.synchronize()
    assert torch.equal(Xs, Xl[:3])


@pytest.mark.parametrize("branch,beta1", [(True, 0.0), (True, 0.9), (False, 0.9)])
def test_momentum_step_vs_oracle(shp, branch, beta1):
    """f2: Alg. 1 tail (momentum, grafted step size, update) per block vs the oracle, two steps."""
    shapes = [(200, 240), (300, 100), (1, 50)]
    pl_o = oplan.plan(shapes, 128, 256, 1)
    pl = shp.make_plan(shapes, 128, 256, 1)
    W_o = [synth.gaussian(s, 300 + i) for i, s in enumerate(shapes)]
    M_o = [np.zeros(s, np.float32) for s in shapes]
    Pm_o = [np.zeros(s, np.float32) for s in shapes]
    Wd = [torch.from_numpy(w.copy()).to(DEV) for w in W_o]
    Md = [torch.zeros(s, dtype=torch.float32, device=DEV) for s in shapes]
    Pmd = [torch.zeros(s, dtype=torch.float32, device=DEV) for s in shapes]
    states = shp.StateTable(Wd, Md, Pmd)
    for step in range(2):
        Gs = [synth.gaussian(s, 400 + 10 * step + i) for i, s in enumerate(shapes)]
        Ds = [np.abs(synth.gaussian(s, 500 + 10 * step + i)) + 0.1 for i, s in enumerate(shapes)]
        Ps = [synth.gaussian(s, 600 + 10 * step + i) for i, s in enumerate(shapes)]
        table = shp.TensorTable([torch.from_numpy(g).to(DEV) for g in Gs], [torch.from_numpy(d).to(DEV) for d in Ds],
                                [torch.from_numpy(p).to(DEV) for p in Ps])
        eta = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
        shp.momentum_step(table, states, pl, beta1, 0.05, branch, eta)
        eta_o = []
        for b in pl_o.blocks:
            sl = (slice(b.row0, b.row0 + b.rows), slice(b.col0, b.col0 + b.cols))
            t = b.tensor_id
            eta_o.append(opre.momentum_step_block(W_o[t][sl], M_o[t][sl], Pm_o[t][sl], Gs[t][sl], Ds[t][sl],
                                                  Ps[t][sl], beta1, 0.05, branch))
        torch.cuda.synchronize()
        np.testing.assert_allclose(eta.cpu().numpy(), eta_o, rtol=1e-6)
        for t in range(len(shapes)):
            np.testing.assert_allclose(Md[t].cpu().numpy(), M_o[t], rtol=1e-6, atol=1e-7)
            np.testing.assert_allclose(Wd[t].cpu().numpy(), W_o[t], rtol=1e-6, atol=1e-7)
            if branch:
                np.testing.assert_allclose(Pmd[t].cpu().numpy(), Pm_o[t], rtol=1e-6, atol=1e-7)
