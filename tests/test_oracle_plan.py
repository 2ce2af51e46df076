"""Pins for oracle.plan (row a1): paper/SPEC worked plans, tiling, exponent-sum,
owner balance and packing invariants.  CPU only."""

import json
import os

import pytest

from oracle import plan as oplan
from synth import transformer_big_shapes
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden():
    with open(os.path.join(GOLDEN, "plan_cases.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _golden()["cases"], ids=lambda c: "x".join(map(str, c["shape"])) + f"_b{c['block_size']}")
def test_paper_plans(case):
    pl = oplan.plan([tuple(case["shape"])], case["block_size"], case["max_precond_dim"], 1)
    got = [[b.row0, b.col0, b.rows, b.cols] for b in pl.blocks]
    assert got == case["blocks"], case["cite"]
    for b in pl.blocks:
        assert (b.p_left, b.p_right) == (case["p_left"], case["p_right"]), case["cite"]


def test_exponents_sum_to_minus_half():
    # P:358-359 ("exponents sum up to -1/2"): -1/(2*)... each kept side contributes -1/p_side * 1/2... i.e.
    # two-sided: -1/4 - 1/4 = -1/2 ; one-sided: -1/2.
    for shape in [(7, 9), (1, 5), (5, 1), (9000, 7), (7, 9000), (300, 300)]:
        pl = oplan.plan([shape], 128, 8192, 1)
        for b in pl.blocks:
            s = (-1.0 / b.p_left if b.p_left else 0.0) + (-1.0 / b.p_right if b.p_right else 0.0)
            if b.p_left or b.p_right:
                assert s == -0.5
            else:
                assert shape[0] in (1,) or shape[0] > 8192


def test_tiling_invariant():
    # blocks tile each tensor exactly and disjointly; ragged last block.
    shapes = [(1000, 300), (1, 77), (4097, 4096), (33, 2049)]
    pl = oplan.plan(shapes, 512, 4096, 3)
    for t, (m, n) in enumerate(shapes):
        cover = [[0] * n for _ in range(m)] if m * n <= 40000 else None
        area = 0
        for b in pl.blocks:
            if b.tensor_id != t:
                continue
            assert 1 <= b.rows <= 512 and 1 <= b.cols <= 512
            assert b.row0 % 512 == 0 and b.col0 % 512 == 0
            area += b.rows * b.cols
            if cover is not None:
                for i in range(b.row0, b.row0 + b.rows):
                    for j in range(b.col0, b.col0 + b.cols):
                        cover[i][j] += 1
        assert area == m * n
        if cover is not None:
            assert all(c == 1 for row in cover for c in row)


def test_transformer_big_counts():
    g = _golden()["transformer_big"]
    shapes = [s for _, s in transformer_big_shapes()]
    assert len(shapes) == 99
    total = sum(m * n for m, n in shapes)
    assert total == g["matrix_params"]
    assert abs(total / 1e6 - g["paper_params_millions"]) / g["paper_params_millions"] < 0.001
    pl = oplan.plan(shapes, g["block_size"], g["max_precond_dim"], 1)
    assert len(pl.blocks) == g["n_blocks"]
    p4 = sum((b.p_left == 4) + (b.p_right == 4) for b in pl.blocks)
    p2 = sum((b.p_left == 2) + (b.p_right == 2) for b in pl.blocks)
    assert (p4, p2) == (g["n_roots_p4"], g["n_roots_p2"])


@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
def test_owner_balance_and_packing(W):
    shapes = [s for _, s in transformer_big_shapes()] + [(100, 37), (2048, 256)]
    pl = oplan.plan(shapes, 1024, 8192, W)
    costs = []
    intervals = []
    for b in pl.blocks:
        for side, p, n, off, ld, own in ((0, b.p_left, b.rows, b.left_off, b.left_ld, b.owner_left),
                                          (1, b.p_right, b.cols, b.right_off, b.right_ld, b.owner_right)):
            if not p:
                assert off == -1
                continue
            assert 0 <= own < W
            assert ld == -(-n // 4) * 4 and off % 64 == 0
            seg0 = own * pl.segment_elems
            assert seg0 <= off and off + n * ld <= seg0 + pl.segment_elems  # inside its owner's segment
            intervals.append((off, off + n * ld))
            costs.append(n ** 3 * oplan.products_per_iteration(p))
    intervals.sort()
    for a, b in zip(intervals, intervals[1:]):
        assert a[1] <= b[0]  # no overlap
    assert pl.stats_elems == W * pl.segment_elems
    # LPT bound: max load - min load <= largest single cost
    assert max(pl.loads) - min(pl.loads) <= max(costs)
    assert sum(pl.loads) == sum(costs)
    # groups are strided batches that cover exactly the owned roots
    assert sum(g.count for g in pl.groups) == len(intervals)
    for g in pl.groups:
        assert g.stride >= g.n * (-(-g.n // 4) * 4) and g.stride % 64 == 0


def test_round_robin_for_uniform_costs():
    pl = oplan.plan([(1024, 1024)] * 8, 1024, 8192, 4)
    owners = [(b.owner_left, b.owner_right) for b in pl.blocks]
    # sorted by (tensor, block, side) with equal costs -> L0 R0 L1 R1 ... dealt round-robin
    flat = [o for pair in owners for o in pair]
    assert flat == [i % 4 for i in range(16)]


def test_plan_is_deterministic():
    shapes = [s for _, s in transformer_big_shapes()]
    a = oplan.plan(shapes, 1024, 8192, 8)
    b = oplan.plan(shapes, 1024, 8192, 8)
    assert [vars(x) for x in a.blocks] == [vars(x) for x in b.blocks]


def test_layer_owners_hand_worked():
    """owners="tensor" (reading #30), worked by hand: costs are sum(n^3 x (products + 12)) + m*n per tensor.
    4 equal 1024^2 tensors at W=4 -> one tensor per rank (LPT deals them 0, 1, 2, 3); at W=3 the fourth goes
    back to rank 0 (all loads equal, lowest rank).  Sizes 256, 512, 512, 1024 (two-sided, 4 products each:
    costs 2*(4+12)*n^3 + n^2) at W=2: the 1024 tensor alone on rank 0, the rest on rank 1 (1024-cost 3.44e10 >
    2 x 4.3e9 + 5.4e8).  The +12 decides the order of a one-sided and a two-sided tensor: (24576, 1024)
    has 24 p=2 roots (24 x 15 = 360 units of 1024^3; products alone: 72), (2048, 5120) 20 p=4 roots (320; 80):
    the vocabulary-like tensor goes first (rank 0), then the two-sided one and the small (1024, 1024) (32) to
    rank 1 -- with products alone the order, and the owners, would flip."""
    pl = oplan.plan([(1024, 1024)] * 4, 1024, 8192, 4, owners="tensor")
    assert pl.tensor_owner == [0, 1, 2, 3]
    assert [(b.owner_left, b.owner_right) for b in pl.blocks] == [(r, r) for r in range(4)]
    pl3 = oplan.plan([(1024, 1024)] * 4, 1024, 8192, 3, owners="tensor")
    assert pl3.tensor_owner == [0, 1, 2, 0]
    pl2 = oplan.plan([(256, 256), (512, 512), (512, 512), (1024, 1024)], 1024, 8192, 2, owners="tensor")
    assert pl2.tensor_owner == [1, 1, 1, 0]
    assert pl2.loads == [2 * 4 * 1024 ** 3, 2 * 4 * (256 ** 3 + 2 * 512 ** 3)]
    pl3 = oplan.plan([(24576, 1024), (2048, 5120), (1024, 1024)], 1024, 8192, 2, owners="tensor")
    assert pl3.tensor_owner == [0, 1, 1]


def test_layer_owners_keep_tensors_whole():
    """Every root of a tensor has the tensor's owner; segments still rebuild the buffer (equal, padded)."""
    shapes = [s for _, s in transformer_big_shapes()]
    for W in (2, 3, 8):
        pl = oplan.plan(shapes, 1024, 8192, W, owners="tensor")
        for b in pl.blocks:
            for p, o in ((b.p_left, b.owner_left), (b.p_right, b.owner_right)):
                if p:
                    assert o == pl.tensor_owner[b.tensor_id]
        assert pl.stats_elems == W * pl.segment_elems
        # LPT over layers: the spread of the root loads is at most one tensor's cost
        tcost = {}
        for b in pl.blocks:
            c = (b.rows ** 3 * oplan.products_per_iteration(b.p_left) if b.p_left else 0) + \
                (b.cols ** 3 * oplan.products_per_iteration(b.p_right) if b.p_right else 0)
            tcost[b.tensor_id] = tcost.get(b.tensor_id, 0) + c
        assert max(pl.loads) - min(pl.loads) <= max(tcost.values()) + max(m * n for m, n in shapes)
