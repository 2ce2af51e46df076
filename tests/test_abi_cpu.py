"""C-ABI checks that need no GPU: the in-tree library loads, exports every
function declared in include/shampoo.h, its host-side plan is bit-exact with
the oracle plan, and host-checkable errors return status codes without
touching the device."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import plan as oplan
import synth
from synth import transformer_big_shapes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def shp():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_shampoo_build", os.path.join(ROOT, "paper_2002_09018_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()
    import paper_2002_09018_b200 as shp
    return shp


def test_library_exports_every_declared_symbol(shp):
    from paper_2002_09018_b200 import _lib
    header = open(os.path.join(ROOT, "include", "shampoo.h")).read()
    declared = sorted(set(re.findall(r"^(?:int|int64_t|size_t|const char\*)\s+(shampoo_[a-z_0-9]+)\(", header, re.M)))
    assert len(declared) >= 12
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTED) == declared
    assert L.shampoo_abi_version() == 4


def _fields_equal(lib_plan, o):
    assert lib_plan.n_blocks == len(o.blocks)
    for b, ob in zip(lib_plan.blocks, o.blocks):
        got = (int(b["tensor_id"]), int(b["row0"]), int(b["col0"]), int(b["rows"]), int(b["cols"]),
               int(b["p_left"]), int(b["p_right"]), int(b["r_left"]), int(b["r_right"]),
               int(b["owner_left"]), int(b["owner_right"]),
               int(b["left_off"]), int(b["right_off"]), int(b["left_ld"]), int(b["right_ld"]))
        want = (ob.tensor_id, ob.row0, ob.col0, ob.rows, ob.cols, ob.p_left, ob.p_right, ob.r_left, ob.r_right,
                ob.owner_left,
                ob.owner_right, ob.left_off, ob.right_off, ob.left_ld, ob.right_ld)
        assert got == want
    assert lib_plan.stats_elems == o.stats_elems and lib_plan.segment_elems == o.segment_elems
    got_g = [tuple(int(g[k]) for k in ("owner", "n", "p", "r", "offset", "count", "stride")) for g in lib_plan.groups]
    want_g = [(g.owner, g.n, g.p, g.r, g.offset, g.count, g.stride) for g in o.groups]
    assert got_g == want_g


CASES = [
    ([s for _, s in transformer_big_shapes()], 1024, 8192),
    ([s for _, s in transformer_big_shapes()], 1024, 4096),
    ([s for _, s in transformer_big_shapes()], 128, 8192),
    ([(32000, 1024)], 1024, 8192),
    ([(1, 10), (10, 1), (1, 1), (7, 9), (1000, 300), (9000, 7)], 64, 8192),
    ([(512, 2048)], 1024, 4096),
]


@pytest.mark.parametrize("W", [1, 2, 3, 8])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_plan_bit_exact_vs_oracle(shp, case, W):
    shapes, b, mpd = CASES[case]
    _fields_equal(shp.make_plan(shapes, b, mpd, W), oplan.plan(shapes, b, mpd, W))


@pytest.mark.parametrize("W", [1, 2, 3, 8])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_plan_layers_bit_exact_vs_oracle(shp, case, W):
    """Layer-granular owners (shampoo_plan_layers, reading #30): blocks, groups and the tensor owners."""
    shapes, b, mpd = CASES[case]
    lp = shp.make_plan(shapes, b, mpd, W, owners="tensor")
    op = oplan.plan(shapes, b, mpd, W, owners="tensor")
    _fields_equal(lp, op)
    assert list(map(int, lp.tensor_owner)) == op.tensor_owner


# f4 splits 1/p = a/d: (1,4) -> 1/8, 3/8; (3,4) -> 3/8, 1/8; (1,3) -> 1/6, 1/3; (2,5) -> 1/5, 3/10
@pytest.mark.parametrize("split", [(1, 4), (3, 4), (1, 3), (2, 5), (1, 8)])
@pytest.mark.parametrize("W", [1, 3])
def test_plan_split_bit_exact_vs_oracle(shp, split, W):
    shapes = [(1024, 1024), (512, 2048), (32000, 512), (300, 200), (1, 50)]
    _fields_equal(shp.make_plan(shapes, 512, 4096, W, split), oplan.plan(shapes, 512, 4096, W, split))


def test_plan_split_invalid(shp):
    from paper_2002_09018_b200 import ShampooError
    for split in [(0, 2), (2, 2), (3, 2), (1, 9)]:  # (1, 9): 1/18 needs a root order > 16
        with pytest.raises(ShampooError):
            shp.make_plan([(64, 64)], 64, 4096, 1, split)
        with pytest.raises(ValueError):
            oplan.plan([(64, 64)], 64, 4096, 1, split)


def test_plan_capacity_and_invalid(shp):
    from paper_2002_09018_b200 import _lib
    L = _lib.lib()
    sh = np.array([[4, 4]], np.int64)
    nb = np.zeros(1, np.int32)
    ng = np.zeros(1, np.int32)
    se = np.zeros(1, np.int64)
    sg = np.zeros(1, np.int64)
    blocks = np.zeros(1, _lib.BLOCK_DTYPE)
    rc = L.shampoo_plan(sh.ctypes.data, 1, 2, 8192, 1, 1, 2, blocks.ctypes.data, 1, nb.ctypes.data, None, 0,
                        ng.ctypes.data, se.ctypes.data, sg.ctypes.data)
    assert rc == 5 and nb[0] == 4  # CAPACITY, counts still written
    bad = np.array([[0, 4]], np.int64)
    assert L.shampoo_plan(bad.ctypes.data, 1, 2, 8192, 1, 1, 2, None, 0, nb.ctypes.data, None, 0, ng.ctypes.data,
                          se.ctypes.data, sg.ctypes.data) == 1
    assert b"zero dimension" in L.shampoo_last_error()


def test_host_checked_errors_need_no_device(shp):
    from paper_2002_09018_b200 import _lib
    L = _lib.lib()
    fake = 1 << 40  # never dereferenced: validation fails first
    # p not in [1, 16]
    assert L.shampoo_inverse_pth_root_batched(fake, 8, 64, fake, 8, 64, 1, 8, 17, 1e-6, 1e-7, 100, 100, fake, fake,
                                              1 << 30, None) == 1
    assert b"p = 17" in L.shampoo_last_error()
    assert L.shampoo_inverse_pth_root_batched(fake, 8, 64, fake, 8, 64, 1, 8, 0, 1e-6, 1e-7, 100, 100, fake, fake,
                                              1 << 30, None) == 1
    # rational exponent: r outside [1, p]
    for p, r in ((8, 0), (8, 9), (3, 4)):
        assert L.shampoo_inverse_root_rational_batched(fake, 8, 64, fake, 8, 64, 1, 8, p, r, 1e-6, 1e-7, 100, 100,
                                                       fake, fake, 1 << 30, None) == 1
        assert b"r = " in L.shampoo_last_error()
    # n out of range
    assert L.shampoo_inverse_pth_root_batched(fake, 8, 64, fake, 8, 64, 1, 0, 4, 1e-6, 1e-7, 100, 100, fake, fake,
                                              1 << 30, None) == 1
    # non-finite eps
    assert L.shampoo_inverse_pth_root_batched(fake, 8, 64, fake, 8, 64, 1, 8, 4, float("nan"), 1e-7, 100, 100, fake,
                                              fake, 1 << 30, None) == 1
    # workspace too small
    assert L.shampoo_inverse_pth_root_batched(fake, 8, 64, fake, 8, 64, 1, 8, 4, 1e-6, 1e-7, 100, 100, fake, fake,
                                              16, None) == 4
    # Ozaki slice count outside {6, 7} (checked before the workspace)
    for bad in (0, 5, 8):
        assert L.shampoo_inverse_pth_root_batched_ozaki(fake, 8, 64, fake, 8, 64, 1, 8, 4, 1e-6, 1e-7, 100, 100, bad,
                                                        0.0, fake, fake, 1 << 30, None) == 1
        assert b"slices" in L.shampoo_last_error()
    # slice budget (ABI v4, reading #29) outside [0, 1)
    for bad in (-1e-9, 1.0, float("nan")):
        assert L.shampoo_inverse_pth_root_batched_ozaki(fake, 8, 64, fake, 8, 64, 1, 8, 4, 1e-6, 1e-7, 100, 100, 7,
                                                        bad, fake, fake, 1 << 30, None) == 1
        assert b"slice_budget" in L.shampoo_last_error()
    # statistics: non-finite decay
    assert L.shampoo_stats_update(fake, 1, fake, fake, 1, -1, fake, float("inf"), 1.0, None, None, fake, 1 << 30,
                                  None) == 1
    # empty batch is a no-op
    assert L.shampoo_inverse_pth_root_batched(None, 0, 0, None, 0, 0, 0, 8, 4, 1e-6, 1e-7, 100, 100, None, None, 0,
                                              None) == 0
    # workspace sizes are pure host functions
    assert L.shampoo_root_workspace_bytes(2, 1024, 4, 100) >= 2 * 7 * 1024 * 1024 * 8
    blk = np.zeros(1, _lib.BLOCK_DTYPE)
    blk["rows"], blk["cols"], blk["p_left"], blk["p_right"] = 100, 70, 4, 4
    assert L.shampoo_stats_workspace_bytes(blk.ctypes.data, 1, -1) >= (128 * 96 + 128 * 128) * 8


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2002_09018_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "liboracle" not in src and "oracle_stats" not in re.sub(r"(#|//).*", "", src), f


# ------------------------------------------------------------------ f3 tensor plan
def _tplan_equal(lib_plan, o):
    assert lib_plan.n_blocks == len(o.blocks) and lib_plan.stats_elems == o.stats_elems
    assert lib_plan.segment_elems == o.segment_elems
    for b, ob in zip(lib_plan.blocks, o.blocks):
        got = (int(b["tensor_id"]), int(b["order"]), [int(x) for x in b["origin"]], [int(x) for x in b["extent"]],
               [int(x) for x in b["p"]], [int(x) for x in b["owner"]], [int(x) for x in b["ld"]],
               [int(x) for x in b["off"]])
        assert got == (ob.tensor_id, ob.order, ob.origin, ob.extent, ob.p, ob.owner, ob.ld, ob.off)
    got_g = [tuple(int(g[k]) for k in ("owner", "n", "p", "r", "offset", "count", "stride")) for g in lib_plan.groups]
    assert got_g == [(g.owner, g.n, g.p, g.r, g.offset, g.count, g.stride) for g in o.groups]


@pytest.mark.parametrize("W", [1, 2, 8])
@pytest.mark.parametrize("b", [1024, 128])
def test_tensor_plan_bit_exact_vs_oracle(shp, W, b):
    from oracle import tensor as ot
    shapes = [s for _, s in synth.resnet50_shapes()] + [(5, 3, 7), (1, 1, 1, 9000), (300, 70, 2)]
    _tplan_equal(shp.make_tensor_plan(shapes, b, 4096, W), ot.plan(shapes, b, 4096, W))


def test_tensor_entry_points_validate_host_tables(shp):
    from paper_2002_09018_b200 import ShampooError, _lib
    L = _lib.lib()
    with pytest.raises(ValueError):
        shp.make_tensor_plan([(2, 3, 4, 5, 6)])
    dims = np.ones((1, 4), np.int64)
    orders = np.array([5], np.int32)
    nb = np.zeros(1, np.int32)
    ng = np.zeros(1, np.int32)
    se = np.zeros(1, np.int64)
    assert L.shampoo_tensor_plan(dims.ctypes.data, orders.ctypes.data, 1, 64, 4096, 1, None, 0, nb.ctypes.data,
                                 None, 0, ng.ctypes.data, se.ctypes.data, se.ctypes.data) == 1
    pl = shp.make_tensor_plan([(3, 4, 5)], 64, 4096, 1)
    t = np.zeros(1, _lib.TTENSOR_DTYPE)
    t[0]["G"] = 1 << 40
    t[0]["dims"][:] = (3, 4, 5, 1)
    t[0]["order"] = 3
    # block extends beyond its tensor -> INVALID_ARG, nothing enqueued
    bad = pl.blocks.copy()
    bad[0]["extent"][0] = 4
    assert L.shampoo_tensor_stats_update(t.ctypes.data, 1, bad.ctypes.data, 1, -1, 1 << 40, 1.0, 1.0, None, None,
                                         1 << 40, 1 << 30, None) == 1
    assert b"outside" in L.shampoo_last_error()
    # precondition needs P
    assert L.shampoo_tensor_precondition(t.ctypes.data, 1, pl.blocks.ctypes.data, 1, 1 << 40, None, None, None,
                                         1 << 40, 1 << 30, None) == 1
    assert b"null G or P" in L.shampoo_last_error()
    with pytest.raises(ShampooError):
        shp.make_tensor_plan([(0, 3)])


def test_ozaki_slice_schedule_worked_values(shp):
    """Reading #29's schedule (host function of the library), worked by hand: S_k = the fewest slices in [5, s_max]
    with 2^-(7S-1) sqrt(n/1024) / (p m_k) <= budget, m_k = min(1, eps g^k), g = ((p+1)/p)^p.
    n = 1024, p = 4 (g = 2.4414): S = 6 needs m >= 2^-41 / 4e-9 = 1.14e-4 -> g^k >= 113.7 -> k >= 5.30; S = 5 needs
    m >= 2^-34 / 4e-9 = 0.01455 -> g^k >= 14552 -> k >= 10.74.  p = 2 (g = 2.25, amplification 1/(2m)): k >= 6.69
    and 12.67.  n = 2048 (x sqrt 2): k >= 5.69 and 11.13.  eps = 0 or budget = 0: s_max throughout."""
    from paper_2002_09018_b200 import _lib
    L = _lib.lib()

    def sched(p, n, eps=1e-6, budget=1e-9, smax=7, ks=range(16)):
        return [L.shampoo_ozaki_iteration_slices(k, p, n, eps, budget, smax) for k in ks]

    assert sched(4, 1024) == [7] * 6 + [6] * 5 + [5] * 5
    assert sched(2, 1024) == [7] * 7 + [6] * 6 + [5] * 3
    assert sched(4, 2048) == [7] * 6 + [6] * 6 + [5] * 4
    assert sched(4, 1024, eps=0.0) == [7] * 16
    assert sched(4, 1024, budget=0.0) == [7] * 16
    assert sched(4, 1024, smax=6) == [6] * 11 + [5] * 5
