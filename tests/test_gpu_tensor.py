"""GPU parity of the tensor path (row f3: order 1..4, per-mode statistics, mode
products, grafting) through the C ABI against oracle/tensor.py on the same
seeded inputs.  Bars: plan and statistics H_i / D bit-exact (chunked
sequential contract, reading #25); graft numerator 1e-12; preconditioned
gradient 1e-5 with the oracle's fp32 roots (fp64 products, fp32
intermediates) and 1e-3 end to end with GPU roots (north star)."""

import numpy as np
import pytest
import torch

import synth
from oracle import root as oroot
from oracle import tensor as ot

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


def _setup(shp, shapes, block, mpd=8192, seed=0):
    Gs = [synth.conv_gradient(s, synth.BASE_SEED + 26 + seed + i) for i, s in enumerate(shapes)]
    pl = shp.make_tensor_plan(shapes, block, mpd, 1)
    po = ot.plan(shapes, block, mpd, 1)
    Gd = [torch.from_numpy(G).to(DEV) for G in Gs]
    Dd = [torch.zeros(s, dtype=torch.float32, device=DEV) for s in shapes]
    Pd = [torch.zeros(s, dtype=torch.float32, device=DEV) for s in shapes]
    return Gs, pl, po, Gd, Dd, Pd


SHAPES = [(3, 3, 64, 40), (100,), (5, 130, 7), (70, 200), (40, 50, 120), (7, 7, 3, 64), (1, 1, 48, 33)]


@pytest.mark.parametrize("block", [1024, 32])
def test_tensor_stats_bit_exact(shp, block):
    Gs, pl, po, Gd, Dd, Pd = _setup(shp, SHAPES, block)
    stats = torch.zeros(pl.stats_elems, dtype=torch.float32, device=DEV)
    gn = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    bs = torch.full((pl.n_blocks,), -1, dtype=torch.int32, device=DEV)
    so = np.zeros(po.stats_elems, np.float32)
    Do = [np.zeros(s, np.float32) for s in SHAPES]
    table = shp.TTensorTable(Gd, Dd)
    for step, (decay, weight) in enumerate([(1.0, 1.0), (0.9, 0.1)]):
        if step:
            Gs = [synth.conv_gradient(s, 777 + i) for i, s in enumerate(SHAPES)]
            for G, g in zip(Gd, Gs):
                G.copy_(torch.from_numpy(g))
        shp.tensor_stats_update(table, pl, stats, decay, weight, -1, gn, bs)
        num_o, st_o = ot.stats_update(Gs, Do, po, so, decay, weight)
        torch.cuda.synchronize()
        assert np.array_equal(stats.cpu().numpy().view(np.uint32), so.view(np.uint32))
        for D, d in zip(Dd, Do):
            assert np.array_equal(D.cpu().numpy().view(np.uint32), d.view(np.uint32))
        np.testing.assert_allclose(gn.cpu().numpy(), num_o, rtol=1e-12)
        assert np.all(bs.cpu().numpy() == st_o)


def test_tensor_stats_non_finite_and_owner(shp):
    shapes = [(3, 4, 5), (6, 40, 3)]
    Gs, pl, po, Gd, Dd, Pd = _setup(shp, shapes, 1024)
    Gs[0][1, 2, 3] = np.inf
    Gd[0].copy_(torch.from_numpy(Gs[0]))
    stats = torch.full((pl.stats_elems,), 3.0, dtype=torch.float32, device=DEV)
    so = np.full(po.stats_elems, 3.0, np.float32)
    Do = [np.zeros(s, np.float32) for s in shapes]
    bs = torch.full((pl.n_blocks,), -1, dtype=torch.int32, device=DEV)
    shp.tensor_stats_update(shp.TTensorTable(Gd, Dd), pl, stats, 1.0, 1.0, -1, None, bs)
    _, st_o = ot.stats_update(Gs, Do, po, so, 1.0, 1.0)
    torch.cuda.synchronize()
    assert list(bs.cpu().numpy()) == list(st_o) == [2, 0]
    assert np.array_equal(stats.cpu().numpy().view(np.uint32), so.view(np.uint32))
    # owner filter: a world-2 plan, rank 1's statistics only
    pl2 = shp.make_tensor_plan(shapes, 1024, 8192, 2)
    po2 = ot.plan(shapes, 1024, 8192, 2)
    Gd[0].copy_(torch.from_numpy(np.nan_to_num(Gs[0], posinf=1.0)))
    Gs[0] = np.nan_to_num(Gs[0], posinf=1.0)
    stats = torch.zeros(pl2.stats_elems, dtype=torch.float32, device=DEV)
    so = np.zeros(po2.stats_elems, np.float32)
    shp.tensor_stats_update(shp.TTensorTable(Gd, Dd), pl2, stats, 1.0, 1.0, 1)
    ot.stats_update(Gs, [np.zeros(s, np.float32) for s in shapes], po2, so, 1.0, 1.0, only_owner=1)
    torch.cuda.synchronize()
    assert np.array_equal(stats.cpu().numpy().view(np.uint32), so.view(np.uint32))


def _oracle_roots(po, stats_np):
    roots = np.zeros(po.stats_elems, np.float32)
    for b in po.blocks:
        for i in range(b.order):
            if b.p[i]:
                n, off, ld = b.extent[i], b.off[i], b.ld[i]
                A = ot.root_view(stats_np, off, n, ld).astype(np.float64)
                X, _ = oroot.inverse_pth_root(A, b.p[i])
                roots[off:off + n * ld].reshape(n, ld)[:, :n] = X
    return roots


@pytest.mark.parametrize("block", [1024, 32])
def test_tensor_precondition_with_oracle_roots(shp, block):
    shapes = SHAPES + [(1, 1, 1, 9000)]  # a diagonal-only block at max_precond_dim 8192
    Gs, pl, po, Gd, Dd, Pd = _setup(shp, shapes, block, seed=5)
    stats = torch.zeros(pl.stats_elems, dtype=torch.float32, device=DEV)
    gn = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    table = shp.TTensorTable(Gd, Dd, Pd)
    shp.tensor_stats_update(table, pl, stats, 1.0, 1.0, -1, gn)
    torch.cuda.synchronize()
    so = stats.cpu().numpy()
    roots = _oracle_roots(po, so)
    sc = torch.zeros(pl.n_blocks, dtype=torch.float32, device=DEV)
    den = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    shp.tensor_precondition(table, pl, torch.from_numpy(roots).to(DEV), gn, sc, den)
    torch.cuda.synchronize()
    Ds = [D.cpu().numpy() for D in Dd]
    Po, sco, deno = ot.precondition_plan(Gs, Ds, po, roots.astype(np.float64), gn.cpu().numpy())
    for P, p in zip(Pd, Po):
        assert rel(P.cpu().numpy(), p) < 1e-5
    np.testing.assert_allclose(den.cpu().numpy(), deno, rtol=1e-5)
    np.testing.assert_allclose(sc.cpu().numpy(), sco, rtol=1e-5)


def test_tensor_end_to_end_gpu_roots(shp):
    """stats -> roots (batched coupled Newton over the tensor plan's groups,
    p = 2k') -> precondition, all on the GPU, vs the oracle chain (bar 1e-3)."""
    shapes = [(3, 3, 16, 24), (50,), (7, 7, 3, 64), (1, 1, 64, 48)]
    Gs, pl, po, Gd, Dd, Pd = _setup(shp, shapes, 1024, seed=9)
    stats = torch.zeros(pl.stats_elems, dtype=torch.float32, device=DEV)
    gn = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    table = shp.TTensorTable(Gd, Dd, Pd)
    shp.tensor_stats_update(table, pl, stats, 1.0, 1.0, -1, gn)
    roots = torch.zeros_like(stats)
    infos = shp.refresh_group_roots(pl, stats, roots, 0)
    sc = torch.zeros(pl.n_blocks, dtype=torch.float32, device=DEV)
    shp.tensor_precondition(table, pl, roots, gn, sc)
    torch.cuda.synchronize()
    assert sorted({int(g["p"]) for g in pl.groups}) == [2, 4, 8]
    so = np.zeros(po.stats_elems, np.float32)
    Do = [np.zeros(s, np.float32) for s in shapes]
    num_o, _ = ot.stats_update(Gs, Do, po, so, 1.0, 1.0)
    ro = _oracle_roots(po, so).astype(np.float64)
    rg = roots.cpu().numpy()
    for b in po.blocks:
        for i in range(b.order):
            if b.p[i]:
                n, off, ld = b.extent[i], b.off[i], b.ld[i]
                assert rel(ot.root_view(rg, off, n, ld), ot.root_view(ro, off, n, ld)) < 2e-6
    Po, sco, _ = ot.precondition_plan(Gs, Do, po, ro, num_o)
    for P, p in zip(Pd, Po):
        assert rel(P.cpu().numpy(), p) < 1e-3
    np.testing.assert_allclose(sc.cpu().numpy(), sco, rtol=1e-3)


def test_resnet50_full_plan_sampled_blocks(shp):
    """ResNet-50 at full size through one statistics call; the oracle
    recomputes a sample of blocks (the largest 3x3 and 1x1 convs, the stem, fc,
    BN vectors): bit-exact."""
    named = synth.resnet50_shapes()
    shapes = [s for _, s in named]
    Gs = [synth.conv_gradient(s, synth.BASE_SEED + 26 + i) for i, s in enumerate(shapes)]
    pl = shp.make_tensor_plan(shapes, 1024, 8192, 1)
    po = ot.plan(shapes, 1024, 8192, 1)
    Gd = [torch.from_numpy(G).to(DEV) for G in Gs]
    Dd = [torch.zeros(s, dtype=torch.float32, device=DEV) for s in shapes]
    stats = torch.zeros(pl.stats_elems, dtype=torch.float32, device=DEV)
    gn = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    shp.tensor_stats_update(shp.TTensorTable(Gd, Dd), pl, stats, 1.0, 1.0, -1, gn)
    torch.cuda.synchronize()
    names = [n for n, _ in named]
    want = {names.index("conv1"), names.index("layer4.2.conv2"), names.index("layer4.0.downsample"),
            names.index("fc"), names.index("layer3.5.conv3.bn.gamma"), names.index("layer1.0.conv2")}
    sample = [b.block_index for b in po.blocks if b.tensor_id in want]
    so = np.zeros(po.stats_elems, np.float32)
    Do = [np.zeros(s, np.float32) for s in shapes]
    num_o, _ = ot.stats_update(Gs, Do, po, so, 1.0, 1.0, blocks=sample)
    sg = stats.cpu().numpy()
    gnc = gn.cpu().numpy()
    for bi in sample:
        b = po.blocks[bi]
        for i in range(b.order):
            if b.p[i]:
                n, off, ld = b.extent[i], b.off[i], b.ld[i]
                assert np.array_equal(sg[off:off + n * ld].view(np.uint32), so[off:off + n * ld].view(np.uint32))
        assert gnc[bi] == pytest.approx(num_o[bi], rel=1e-12)


def test_resnet50_full_step_sampled_precondition(shp):
    """ResNet-50 at full size: statistics, every root on the GPU (tensor plan
    groups, p in {2, 4, 8}), preconditioning; the oracle recomputes P for a
    sample of blocks from the GPU's fp32 roots (kernel-isolated, bar 1e-5) and
    the roots of the sample from the GPU statistics (bar 2e-6)."""
    named = synth.resnet50_shapes()
    shapes = [s for _, s in named]
    Gs = [synth.conv_gradient(s, synth.BASE_SEED + 26 + i) for i, s in enumerate(shapes)]
    pl = shp.make_tensor_plan(shapes, 1024, 8192, 1)
    po = ot.plan(shapes, 1024, 8192, 1)
    Gd = [torch.from_numpy(G).to(DEV) for G in Gs]
    Dd = [torch.zeros(s, dtype=torch.float32, device=DEV) for s in shapes]
    Pd = [torch.zeros(s, dtype=torch.float32, device=DEV) for s in shapes]
    table = shp.TTensorTable(Gd, Dd, Pd)
    stats = torch.zeros(pl.stats_elems, dtype=torch.float32, device=DEV)
    gn = torch.zeros(pl.n_blocks, dtype=torch.float64, device=DEV)
    shp.tensor_stats_update(table, pl, stats, 1.0, 1.0, -1, gn)
    roots = torch.zeros_like(stats)
    infos = shp.refresh_group_roots(pl, stats, roots, 0)
    sc = torch.zeros(pl.n_blocks, dtype=torch.float32, device=DEV)
    shp.tensor_precondition(table, pl, roots, gn, sc)
    torch.cuda.synchronize()
    for _, info in infos:
        assert set(shp.info_to_numpy(info)["status"].tolist()) <= {0, 1}
    names = [n for n, _ in named]
    want = {names.index("conv1"), names.index("layer2.1.conv2"), names.index("layer1.0.conv3"),
            names.index("layer3.0.conv1.bn.beta")}
    sample = [b.block_index for b in po.blocks if b.tensor_id in want]
    sg, rg = stats.cpu().numpy(), roots.cpu().numpy()
    for bi in sample:
        b = po.blocks[bi]
        for i in range(b.order):
            if b.p[i]:
                n, off, ld = b.extent[i], b.off[i], b.ld[i]
                Xo, _ = oroot.inverse_pth_root(ot.root_view(sg, off, n, ld).astype(np.float64), b.p[i])
                assert rel(ot.root_view(rg, off, n, ld), Xo) < 2e-6
    Ds = [D.cpu().numpy() for D in Dd]
    Po, sco, _ = ot.precondition_plan(Gs, Ds, po, rg.astype(np.float64), gn.cpu().numpy(), blocks=sample)
    scg = sc.cpu().numpy()
    for bi in sample:
        b = po.blocks[bi]
        t = b.tensor_id
        sl = b.slices()
        assert rel(Pd[t].cpu().numpy()[sl], Po[t][sl]) < 1e-5
        assert scg[bi] == pytest.approx(sco[bi], rel=1e-5)
