"""f1: the delayed refresh adopts, at each kappa boundary, roots bit-identical to a
synchronous refresh of the statistics snapshot taken one kappa earlier (Alg. 1
P:603-606: the step uses L_(t-kappa)^{-1/4}); the work is spread over steps."""

import numpy as np
import pytest
import torch

import synth

DEV = "cuda:0"


def _setup(shp, shapes, block):
    plan = shp.make_plan(shapes, block, 8192, 1)
    Gs = [torch.zeros(s, dtype=torch.float32, device=DEV) for s in shapes]
    table = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs])
    stats = torch.zeros(plan.stats_elems, dtype=torch.float32, device=DEV)
    return plan, Gs, table, stats


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [None, "ozaki"])
def test_delayed_refresh_matches_synchronous_refresh_of_snapshot(precision):
    import paper_2002_09018_b200 as shp
    from paper_2002_09018_b200.schedule import DelayedRefresh
    shapes = [(256, 384), (128, 128), (300, 200)]
    plan, Gs, table, stats = _setup(shp, shapes, 128)
    roots = torch.zeros_like(stats)
    kappa = 4
    dr = DelayedRefresh(plan, stats, roots, kappa=kappa, spread=3, fp64_iters=precision)
    snapshots = {}
    adopted_at = []
    for t in range(0, 3 * kappa + 1):
        for i, (G, s) in enumerate(zip(Gs, shapes)):
            G.copy_(torch.from_numpy(synth.gaussian(s, 1000 * t + i)))
        shp.stats_update(table, plan, stats, 1.0, 1.0)
        if t % kappa == 0:
            snapshots[t] = stats.clone()
        if dr.step(t):
            adopted_at.append(t)
            ref = torch.zeros_like(stats)
            shp.refresh_group_roots(plan, snapshots[t - kappa], ref, 0, fp64_iters=precision)
            torch.cuda.synchronize()
            assert torch.equal(dr.current[:plan.stats_elems], ref[:plan.stats_elems]), t
    assert adopted_at == [kappa, 2 * kappa, 3 * kappa]
    assert dr.refreshes == 3


def test_schedule_covers_every_root_once_cpu():
    """Host-side chunking: every owned root is scheduled exactly once per refresh, at most `chunk` per step, and
    the number of chunk steps -- hence the step of the all-gather -- is the same on every rank even when the LPT
    owners hold unequal counts (a rank-dependent gather step would match collectives out of order)."""
    import paper_2002_09018_b200 as shp
    from paper_2002_09018_b200.schedule import chunking, schedule_units
    cases = [([s for _, s in synth.transformer_big_shapes()], 1024),
             ([(256, 384), (128, 128), (300, 200), (1000, 64), (640, 512)], 128)]
    for shapes, block in cases:
        for world in (1, 2, 3):
            plan = shp.make_plan(shapes, block, 8192, world)
            counts = [sum(int(g["count"]) for g in plan.groups_of(r)) for r in range(world)]
            for kappa, spread in ((500, None), (500, 7), (20, 1), (4, 3)):
                chunk, n_steps = chunking(plan, world, kappa, spread)
                assert n_steps <= min(kappa, spread or kappa)
                for rank in range(world):
                    units = [(g, 0, int(g["count"])) for g in plan.groups_of(rank)]
                    steps = schedule_units(units, chunk, n_steps)
                    assert len(steps) == n_steps  # identical on every rank
                    seen = []
                    for st in steps:
                        assert sum(n for _, _, n in st) <= chunk
                        for g, i, n in st:
                            seen += [(int(g["offset"]), i + k) for k in range(n)]
                    assert len(seen) == len(set(seen)) == counts[rank]
