"""GPU parity for general root orders p in [1, 16] (f3: p = 2k for rank-k
tensors) and rational exponents A_hat^{-r/p} (f4, "L^{-1/2p} G
R^{-1/2q}"), through the C ABI, against the fp64 oracle.  Bars: roots <= 1e-3
relative Frobenius (north star), held to 2e-6 x r (fp32 output of an fp64
iteration, raised to the power r); iterations +-1; statuses equal."""

import numpy as np
import pytest
import torch

import synth
from oracle import plan as oplan
from oracle import root as oroot

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def shp():
    import paper_2002_09018_b200 as shp
    return shp


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _both(shp, As, p, r, eps=1e-6, tol=1e-7, max_iter=100):
    A = torch.from_numpy(np.ascontiguousarray(As)).to(DEV)
    X, info = shp.inverse_pth_root_batched(A, p, r=r, eps_rel=eps, tol=tol, max_iter=max_iter)
    torch.cuda.synchronize()
    outs = [oroot.inverse_root(a.astype(np.float64), p, r, eps, tol, max_iter) for a in As]
    return X.cpu().numpy(), shp.info_to_numpy(info), outs


@pytest.mark.parametrize("p", [3, 5, 6, 7, 16])
def test_general_p_mixed_batch(shp, p):
    As = synth.psd_batch(130, 4, synth.BASE_SEED + 40 + p, "mixed")  # ragged 130: 3 tiles per side
    Xg, inf, outs = _both(shp, As, p, 1)
    for i, (Xo, io) in enumerate(outs):
        assert rel(Xg[i], Xo) < 2e-6, (i, rel(Xg[i], Xo))
        assert inf[i]["status"] == io.status == 0
        assert abs(int(inf[i]["iters"]) - io.iters) <= 1


@pytest.mark.parametrize("p,r", [(8, 3), (8, 1), (6, 5), (3, 2), (4, 4), (16, 7)])
def test_rational_roots(shp, p, r):
    As = synth.psd_batch(200, 3, synth.BASE_SEED + 60 + 16 * p + r, "mixed")
    Xg, inf, outs = _both(shp, As, p, r)
    for i, (Xo, io) in enumerate(outs):
        assert rel(Xg[i], Xo) < 2e-6 * r, (i, rel(Xg[i], Xo))
        assert inf[i]["status"] == io.status
        assert abs(int(inf[i]["iters"]) - io.iters) <= 1


def test_rational_1024(shp):
    As = synth.psd_batch(1024, 2, synth.BASE_SEED + 2, "wishart")
    Xg, inf, outs = _both(shp, As, 8, 3)
    for i, (Xo, io) in enumerate(outs):
        assert rel(Xg[i], Xo) < 6e-6
        assert inf[i]["status"] == 0


def test_rational_edge_cases(shp):
    n = 40
    As = np.zeros((4, n, n), np.float32)
    As[0] = np.eye(n)
    As[1] = 0.0                                           # degenerate -> I (I^r = I), status 3
    As[2] = synth.wishart(n, 4)
    As[2][5, 7] = As[2][7, 5] = np.inf                    # non-finite -> untouched, status 2
    As[3] = synth.wishart(n, 5)
    A = torch.from_numpy(As).to(DEV)
    X = torch.full_like(A, 7.0)
    X, info = shp.inverse_pth_root_batched(A, 8, X=X, r=3)
    torch.cuda.synchronize()
    Xg, inf = X.cpu().numpy(), shp.info_to_numpy(info)
    np.testing.assert_allclose(Xg[0], (1 + 1e-6) ** (-3 / 8) * np.eye(n), rtol=1e-7, atol=0)
    assert inf[1]["status"] == 3 and np.array_equal(Xg[1], np.eye(n, dtype=np.float32))
    assert inf[2]["status"] == 2 and np.all(Xg[2] == 7.0)
    Xo, io = oroot.inverse_root(As[3].astype(np.float64), 8, 3)
    assert rel(Xg[3], Xo) < 6e-6


def test_split_plan_roots_through_groups(shp):
    """f4 end to end on the root side: a (1, 4) split plan (L^{-1/8}, R^{-3/8})
    refreshed group by group lands at the statistics offsets."""
    shapes = [(256, 256), (130, 300)]
    rng = np.random.default_rng(5)
    pl = shp.make_plan(shapes, 128, 4096, 1, (1, 4))
    pl_o = oplan.plan(shapes, 128, 4096, 1, (1, 4))
    stats = np.zeros(pl.stats_elems, np.float32)
    for b in pl_o.blocks:
        for n, off, ld in ((b.rows, b.left_off, b.left_ld), (b.cols, b.right_off, b.right_ld)):
            W = rng.standard_normal((n, max(1, n // 2))).astype(np.float32)
            S = (W.astype(np.float64) @ W.astype(np.float64).T).astype(np.float32)
            S = np.triu(S) + np.triu(S, 1).T
            stats[off:off + n * ld].reshape(n, ld)[:, :n] = S
    sd = torch.from_numpy(stats).to(DEV)
    roots = torch.zeros_like(sd)
    shp.refresh_group_roots(pl, sd, roots, 0)
    torch.cuda.synchronize()
    rg = roots.cpu().numpy()
    for b in pl_o.blocks:
        assert (b.p_left, b.r_left, b.p_right, b.r_right) == (8, 1, 8, 3)
        for n, off, ld, p, r in ((b.rows, b.left_off, b.left_ld, 8, 1), (b.cols, b.right_off, b.right_ld, 8, 3)):
            A = stats[off:off + n * ld].reshape(n, ld)[:, :n].astype(np.float64)
            Xo, _ = oroot.inverse_root(A, p, r)
            assert rel(rg[off:off + n * ld].reshape(n, ld)[:, :n], Xo) < 6e-6


@pytest.mark.parametrize("p", [3, 6])
def test_residual_general_p(shp, p):
    As = synth.psd_batch(100, 2, 91, "mixed")
    A = torch.from_numpy(As).to(DEV)
    X, info = shp.inverse_pth_root_batched(A, p)
    res = shp.root_residual_batched(A, X, p, info).cpu().numpy()
    inf = shp.info_to_numpy(info)
    for i in range(2):
        want = oroot.residual(As[i].astype(np.float64), X[i].cpu().numpy().astype(np.float64), p, 1e-6,
                              float(inf[i]["lambda_max"]))
        assert abs(res[i] - want) <= 1e-6 * max(1.0, want)
