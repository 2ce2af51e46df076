"""Oracle: statistics update over a whole plan (row a2), wrapping oracle_stats.c.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

``stats_update`` mirrors the semantics of the product's one-launch-per-step
call: for every block, a non-finite G leaves the block's L/R/D unchanged and
reports status 2; otherwise L (if p_left and owned) and R (if p_right
and owned) are updated under the sequential fp64 contract of
``oracle/csrc/oracle_stats.c`` and D / the graft numerator are updated for
every block (D is needed by every rank's grafting).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "oracle_stats.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_f32p = ctypes.POINTER(ctypes.c_float)
_i64 = ctypes.c_int64
_i32 = ctypes.c_int


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain C, fp64, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        for name in ("oracle_stats_left", "oracle_stats_right"):
            f = getattr(_lib, name)
            f.argtypes = [_f32p, _i64, _i64, _i64, _i32, _i32, _f32p, _i64, ctypes.c_double, ctypes.c_double]
            f.restype = None
        _lib.oracle_block_finite.argtypes = [_f32p, _i64, _i64, _i64, _i32, _i32]
        _lib.oracle_block_finite.restype = _i32
        _lib.oracle_diag_update.argtypes = [_f32p, _i64, _i64, _i64, _i32, _i32, _f32p, _i64]
        _lib.oracle_diag_update.restype = ctypes.c_double
        _lib.oracle_mode_stat.argtypes = [_f32p, _i32, _i64, _i64, _f32p, _i64, ctypes.c_double, ctypes.c_double]
        _lib.oracle_mode_stat.restype = None
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_f32p)


def block_finite(G: np.ndarray, row0: int, col0: int, rows: int, cols: int) -> bool:
    return bool(lib().oracle_block_finite(_ptr(G), G.shape[1], row0, col0, rows, cols))


def stats_left(G, row0, col0, rows, cols, L: np.ndarray, decay: float, weight: float):
    """L (rows x >=rows view with leading dim L.shape[1]) <- decay L + weight G_b G_b^T."""
    lib().oracle_stats_left(_ptr(G), G.shape[1], row0, col0, rows, cols, _ptr(L), L.shape[1], decay, weight)


def stats_right(G, row0, col0, rows, cols, R: np.ndarray, decay: float, weight: float):
    lib().oracle_stats_right(_ptr(G), G.shape[1], row0, col0, rows, cols, _ptr(R), R.shape[1], decay, weight)


def diag_update(G, row0, col0, rows, cols, D: np.ndarray) -> float:
    return float(lib().oracle_diag_update(_ptr(G), G.shape[1], row0, col0, rows, cols, _ptr(D), D.shape[1]))


def stat_view(stats: np.ndarray, off: int, n: int, ld: int) -> np.ndarray:
    """n x ld row-major view of a packed statistic (padding columns included)."""
    return stats[off:off + n * ld].reshape(n, ld)


def stats_update(Gs, D_list, pl, stats: np.ndarray, decay: float, weight: float,
                 only_owner: int = -1, blocks=None):
    """One statistics step over the plan ``pl`` (oracle.plan.Plan), in place.

    Returns (graft_num [n_blocks] float64, block_status [n_blocks] int32).
    ``blocks``: optional subset of block indices to process (sampled parity).
    """
    nb = len(pl.blocks)
    num = np.zeros(nb, np.float64)
    status = np.zeros(nb, np.int32)
    idx = range(nb) if blocks is None else blocks
    for bi in idx:
        b = pl.blocks[bi]
        G = Gs[b.tensor_id]
        if not block_finite(G, b.row0, b.col0, b.rows, b.cols):
            status[bi] = 2
            continue
        if b.p_left and (only_owner < 0 or b.owner_left == only_owner):
            stats_left(G, b.row0, b.col0, b.rows, b.cols,
                       stat_view(stats, b.left_off, b.rows, b.left_ld), decay, weight)
        if b.p_right and (only_owner < 0 or b.owner_right == only_owner):
            stats_right(G, b.row0, b.col0, b.rows, b.cols,
                        stat_view(stats, b.right_off, b.cols, b.right_ld), decay, weight)
        if D_list is not None:
            num[bi] = diag_update(G, b.row0, b.col0, b.rows, b.cols, D_list[b.tensor_id])
    return num, status


def mode_stat(U: np.ndarray, S: np.ndarray, chunk: int, decay: float, weight: float):
    """S (rows x >=rows view, leading dim S.shape[1]) <- decay S + weight U U^T under the
    chunked sequential contract (oracle_stats.c, f3)."""
    U = np.ascontiguousarray(U, np.float32)
    lib().oracle_mode_stat(_ptr(U), U.shape[0], U.shape[1], chunk, _ptr(S), S.shape[1], decay, weight)
