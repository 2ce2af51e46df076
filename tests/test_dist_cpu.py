"""Multi-process host logic of row a7 on CPU (gloo, world_size 2 and 3): every
rank fills only the roots it owns (per the plan's segments), one all-gather of
the equal-size segments rebuilds the identical full buffer on every rank, and
the owner-only statistics are disjoint and cover every root exactly once."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import transformer_big_shapes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shapes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2002_09018_b200 as shp
        from paper_2002_09018_b200 import dist as sdist
        plan = shp.make_plan(shapes, 1024, 8192, world)
        roots = torch.full((plan.stats_elems,), float("nan"))
        # this rank "computes" its roots: value = 1000*block + side + 1 at every element
        for b_idx, b in enumerate(plan.blocks):
            for side, p, n, off, ld, own in ((0, b["p_left"], b["rows"], b["left_off"], b["left_ld"], b["owner_left"]),
                                             (1, b["p_right"], b["cols"], b["right_off"], b["right_ld"], b["owner_right"])):
                if p and own == rank:
                    roots[int(off):int(off) + int(n) * int(ld)] = 1000.0 * b_idx + side + 1
        sdist.all_gather_roots(plan, roots, rank, world)
        q.put((rank, roots.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_all_gather_rebuilds_every_root(world):
    shapes = [s for _, s in transformer_big_shapes()][:12] + [(32000, 1024)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shapes, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import paper_2002_09018_b200 as shp
    plan = shp.make_plan(shapes, 1024, 8192, world)
    ref = out[0]
    for r in range(1, world):
        assert np.array_equal(np.nan_to_num(out[r], nan=-1), np.nan_to_num(ref, nan=-1))
    for b_idx, b in enumerate(plan.blocks):
        for side, p, n, off, ld in ((0, b["p_left"], b["rows"], b["left_off"], b["left_ld"]),
                                    (1, b["p_right"], b["cols"], b["right_off"], b["right_ld"])):
            if p:
                seg = ref[int(off):int(off) + int(n) * int(ld)]
                assert np.all(seg == 1000.0 * b_idx + side + 1)


def test_owner_shards_cover_each_root_once():
    import paper_2002_09018_b200 as shp
    shapes = [s for _, s in transformer_big_shapes()]
    for world in (1, 2, 4, 8):
        plan = shp.make_plan(shapes, 1024, 8192, world)
        owned = [0] * world
        load = [0] * world
        for b in plan.blocks:
            for p, own, n in ((b["p_left"], b["owner_left"], b["rows"]), (b["p_right"], b["owner_right"], b["cols"])):
                if p:
                    owned[int(own)] += 1
                    load[int(own)] += int(n) ** 3 * {2: 3, 4: 4}[int(p)]
        assert sum(owned) == 624
        assert max(load) - min(load) <= 4 * 1024 ** 3  # LPT: within one root's cost
        # every rank's groups live inside its own segment
        for g in plan.groups:
            o = int(g["owner"])
            assert o * plan.segment_elems <= int(g["offset"])
            assert int(g["offset"]) + int(g["count"]) * int(g["stride"]) <= (o + 1) * plan.segment_elems


def _worker_overlapped(rank, world, port, shapes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2002_09018_b200 as shp
        from paper_2002_09018_b200 import dist as sdist
        plan = shp.make_plan(shapes, 1024, 8192, world)

        def fill(buf, g):  # the owner's "computed" roots of group g: a distinct value per element
            off, cnt, stride = int(g["offset"]), int(g["count"]), int(g["stride"])
            buf[off:off + cnt * stride] = torch.arange(cnt * stride, dtype=torch.float32) + 1e6 * (1 + int(g["owner"]))

        ref = torch.full((plan.stats_elems,), float("nan"))
        for g in plan.groups_of(rank):
            fill(ref, g)
        sdist.all_gather_roots(plan, ref, rank, world)
        roots = torch.full((plan.stats_elems,), float("nan"))
        sdist.refresh_gather_overlapped(plan, None, roots, rank, world, compute_group=lambda g: fill(roots, g))
        q.put((rank, ref.numpy().copy(), roots.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_overlapped_group_broadcasts_equal_the_all_gather(world):
    """refresh_gather_overlapped (per-group broadcasts from the owners, overlapping the next group's roots)
    rebuilds exactly the buffer all_gather_roots rebuilds, on every rank."""
    shapes = [s for _, s in transformer_big_shapes()][:12] + [(32000, 1024)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_overlapped, args=(r, world, port, shapes, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ref, got in out:
        assert np.array_equal(np.nan_to_num(ref, nan=-1), np.nan_to_num(got, nan=-1)), rank
    assert np.array_equal(np.nan_to_num(out[0][2], nan=-1), np.nan_to_num(out[-1][2], nan=-1))


def _layer_worker(rank, world, port, shapes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2002_09018_b200 as shp
        from paper_2002_09018_b200 import dist as sdist
        plan = shp.make_plan(shapes, 128, 8192, world, owners="tensor")
        ls = sdist.LayerShards(plan, world)
        flat = torch.full((ls.numel,), float("nan"))
        P = ls.p_views(flat)
        # this rank "preconditions" its own tensors: P[t] = t + 1 + (index in the tensor) * 1e-3
        for t, (m, n) in enumerate(shapes):
            if ls.owner[t] == rank:
                P[t].copy_(float(t + 1) + 1e-3 * torch.arange(m * n, dtype=torch.float32).view(m, n))
        sc = ls.scales_of(flat, rank)
        sc.copy_(torch.as_tensor(ls.block_idx[rank], dtype=torch.float32) + 0.5)
        ls.gather(flat, rank)
        full = torch.zeros(plan.n_blocks)
        ls.unpack_scales(flat, full)
        q.put((rank, [p.clone().numpy() for p in ls.p_views(flat)], full.numpy().copy(),
               [len(s.blocks) for s in ls.sub], ls.block_idx))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_layer_shards_gather_every_p_and_scale(world):
    """Layer-granular step (reading #30): each rank writes only its tensors' P and its blocks' graft scales into
    its segment of the flat buffer; one all-gather of the equal segments gives every rank every P and every
    scale; the per-rank sub-plans partition the blocks (no block twice, none missing)."""
    shapes = [(300, 200), (128, 128), (1000, 64), (64, 1), (50, 700), (256, 384)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_layer_worker, args=(r, world, port, shapes, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, Ps, sc, counts, idx = q.get(timeout=240)
        out[r] = (Ps, sc, counts, idx)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Ps0, sc0, counts, idx = out[0]
    allidx = np.sort(np.concatenate(idx))
    assert np.array_equal(allidx, np.arange(len(allidx)))  # sub-plans partition the blocks
    assert sum(counts) == len(allidx)
    for r in range(world):
        Ps, sc, _, _ = out[r]
        for t, (m, n) in enumerate(shapes):
            want = float(t + 1) + 1e-3 * np.arange(m * n, dtype=np.float32).reshape(m, n)
            assert np.array_equal(Ps[t], want), (r, t)
        assert np.array_equal(sc, np.arange(len(sc), dtype=np.float32) + 0.5)
