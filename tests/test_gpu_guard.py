"""Guard-band checks (a stand-in for memcheck, which this pool does not
offer): every root precision writes exactly the n x n output of each matrix
of a padded, strided batch and leaves the padding / inter-matrix gaps and the
input untouched; the preconditioner leaves the padding columns of P alone."""

import numpy as np
import pytest
import torch

import synth
from oracle import root as oroot

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def shp():
    import paper_2002_09018_b200 as shp
    return shp


@pytest.mark.parametrize("mode", [None, "ozaki", -1])
@pytest.mark.parametrize("n", [130, 64])
def test_root_writes_only_its_outputs(shp, mode, n):
    batch, ld = 3, n + 6 + (n % 4 == 0) * 2
    ld = (ld + 3) // 4 * 4
    stride = ld * (n + 3) + 20
    As = synth.psd_batch(n, batch, 404 + n, "mixed")
    Abuf = torch.full((batch * stride + 64,), -3.0, dtype=torch.float32)
    Xbuf = torch.full((batch * stride + 64,), 7.0, dtype=torch.float32)
    for b in range(batch):
        Abuf[b * stride:b * stride + n * ld].view(n, ld)[:, :n] = torch.from_numpy(As[b])
    Ad, Xd = Abuf.to(DEV), Xbuf.to(DEV)
    A_before = Ad.clone()
    info = shp.new_info(batch, DEV)
    shp.inverse_pth_root_ptr(Ad.data_ptr(), ld, stride, Xd.data_ptr(), ld, stride, batch, n, 4, info, device=DEV,
                             fp64_iters=mode)
    torch.cuda.synchronize()
    assert torch.equal(Ad, A_before)
    X = Xd.cpu().numpy()
    inside = np.zeros(X.shape, bool)
    for b in range(batch):
        view = np.arange(X.size)[b * stride:b * stride + n * ld].reshape(n, ld)[:, :n]
        inside[view.ravel()] = True
        Xo, _ = oroot.inverse_pth_root(As[b].astype(np.float64), 4)
        Xg = X[b * stride:b * stride + n * ld].reshape(n, ld)[:, :n]
        assert np.linalg.norm(Xg - Xo) / np.linalg.norm(Xo) < 3e-4
    assert np.all(X[~inside] == 7.0)


def test_precondition_leaves_padding(shp):
    m, n, ldp = 300, 200, 212
    pl = shp.make_plan([(m, n)], 128, 4096, 1)
    G = torch.from_numpy(synth.lowrank_gradient(m, n, 9)).to(DEV)
    Pbig = torch.full((m, ldp), 5.0, device=DEV)
    P = Pbig[:, :n]
    D = torch.ones_like(G)
    roots = torch.randn(pl.stats_elems, device=DEV) * 0.05
    shp.precondition(shp.TensorTable([G], [D], [P]), pl, roots)
    torch.cuda.synchronize()
    assert torch.all(Pbig[:, n:] == 5.0)
    assert torch.all(torch.isfinite(P))
