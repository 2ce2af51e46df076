"""Oracle: Shampoo for tensors of order 1..4 (row f3): blocking plan, per-mode
statistics, preconditioned gradient and grafting.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain Python integers for
the plan; the chunked sequential fp64 contract in plain C for the statistics
(``oracle/csrc/oracle_stats.c``); numpy fp64 (``tensordot``, a library
contraction) for the mode products.

The paper: "our design, analysis, and implementation holds for tensors of
arbitrary order" and "All of our modifications to Shampoo are
extended and implemented for tensors of arbitrary dimension"; the
blocking of P:396-398 and the large-dimension bypass with "exponents sum up to
-1/2" of P:356-359 apply per mode.  The tensor algebra is not printed; the
readings (DESIGN.md §3 #24-#26) are those of the original Shampoo for order-k
tensors:

* mode i of an order-k tensor is preconditioned iff 1 < d_i <= max_precond_dim;
  with k' kept modes each kept mode gets the exponent -1/(2k') (p = 2k'), so the
  exponents sum to -1/2; k' = 2 is the matrix rule (p = 4), k' = 1
  the one-sided rule (p = 2); k' = 0 -> grafted diagonal AdaGrad (reading #17).
* every mode is split into ceil(d_i / b) contiguous ranges (last ragged);
  blocks row-major over the block grid (mode 0 slowest), tensors in caller order.
* statistic of kept mode i of block B: H_i <- decay H_i + weight U_i U_i^T with
  U_i the mode-i unfolding of B (rows: mode-i index; columns: the remaining
  block indices in row-major order), under the chunked sequential contract
  (chunk C = 4096 columns; identical to the matrix contract when K <= C).
* preconditioned block: P_B = B x_0 X_0 x_1 X_1 ... (mode-i product with
  X_i = H_i^{-1/p} over the kept modes), (B x_i X)[.., a, ..] = sum_c X[a, c] B[.., c, ..].
* roots: sorted by (n^3 * products(p) desc, tensor, block, mode), LPT owners,
  packed exactly as the matrix plan (groups of equal (n, p), r = 1).
* D, the graft numerator and the graft scale as for matrices, per block.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .plan import RootGroup, _roundup, products_per_iteration
from . import stats as ostats

MAX_ORDER = 4
STAT_CHUNK = 4096


@dataclass
class TBlock:
    tensor_id: int
    block_index: int
    order: int
    origin: list
    extent: list
    p: list
    owner: list = field(default_factory=lambda: [-1] * MAX_ORDER)
    off: list = field(default_factory=lambda: [-1] * MAX_ORDER)
    ld: list = field(default_factory=lambda: [0] * MAX_ORDER)

    def slices(self):
        return tuple(slice(self.origin[i], self.origin[i] + self.extent[i]) for i in range(self.order))


@dataclass
class TPlan:
    blocks: list = field(default_factory=list)
    groups: list = field(default_factory=list)
    stats_elems: int = 0
    segment_elems: int = 0
    loads: list = field(default_factory=list)


def plan(shapes, block_size: int, max_precond_dim: int, world_size: int) -> TPlan:
    if block_size < 1 or max_precond_dim < 1 or world_size < 1:
        raise ValueError("block_size, max_precond_dim and world_size must be >= 1")
    out = TPlan()
    for t, shape in enumerate(shapes):
        shape = tuple(int(d) for d in shape)
        k = len(shape)
        if not (1 <= k <= MAX_ORDER) or min(shape) < 1:
            raise ValueError(f"tensor {t}: order 1..{MAX_ORDER} with dims >= 1")
        kept = [1 < d <= max_precond_dim for d in shape]
        pk = 2 * sum(kept)
        grid = [-(-d // block_size) for d in shape]
        for flat in range(int(np.prod(grid))):
            idx = []
            rem = flat
            for g in reversed(grid):
                idx.append(rem % g)
                rem //= g
            idx = idx[::-1]
            origin = [i * block_size for i in idx] + [0] * (MAX_ORDER - k)
            extent = [min(block_size, d - o) for d, o in zip(shape, origin)] + [1] * (MAX_ORDER - k)
            p = [pk if kp else 0 for kp in kept] + [0] * (MAX_ORDER - k)
            out.blocks.append(TBlock(t, len(out.blocks), k, origin, extent, p))
    roots = []
    for b in out.blocks:
        for i in range(b.order):
            if b.p[i]:
                n = b.extent[i]
                roots.append((n ** 3 * products_per_iteration(b.p[i]), b.tensor_id, b.block_index, i))
    roots.sort(key=lambda r: (-r[0], r[1], r[2], r[3]))
    loads = [0] * world_size
    owned = [[] for _ in range(world_size)]
    for pos, (cost, _t, bidx, mode) in enumerate(roots):
        r = min(range(world_size), key=lambda i: (loads[i], i))
        loads[r] += cost
        b = out.blocks[bidx]
        b.owner[mode] = r
        owned[r].append((b.extent[mode], b.p[mode], pos, bidx, mode))
    seg_used = []
    for r in range(world_size):
        items = sorted(owned[r], key=lambda x: (-x[0], -x[1], x[2]))
        off = 0
        i = 0
        while i < len(items):
            nn, pp = items[i][0], items[i][1]
            j = i
            while j < len(items) and items[j][:2] == (nn, pp):
                j += 1
            ld = _roundup(nn, 4)
            stride = _roundup(nn * ld, 64)
            out.groups.append(RootGroup(r, nn, pp, off, j - i, stride, 1))
            for q in range(i, j):
                _, _, _, bidx, mode = items[q]
                b = out.blocks[bidx]
                b.off[mode], b.ld[mode] = off + (q - i) * stride, ld
            off += (j - i) * stride
            i = j
        seg_used.append(off)
    seg = _roundup(max(seg_used) if seg_used else 0, 64)
    out.segment_elems = seg
    out.stats_elems = seg * world_size
    for g in out.groups:
        g.offset += g.owner * seg
    for b in out.blocks:
        for i in range(b.order):
            if b.off[i] >= 0:
                b.off[i] += b.owner[i] * seg
    out.loads = loads
    return out


def unfold(B: np.ndarray, mode: int) -> np.ndarray:
    """Mode-`mode` unfolding: rows = the mode's index, columns = the remaining
    indices in row-major order."""
    return np.moveaxis(B, mode, 0).reshape(B.shape[mode], -1)


def mode_product(B: np.ndarray, X: np.ndarray, mode: int) -> np.ndarray:
    """(B x_mode X)[.., a, ..] = sum_c X[a, c] B[.., c, ..] in fp64."""
    return np.moveaxis(np.tensordot(np.asarray(X, np.float64), np.asarray(B, np.float64), axes=([1], [mode])), 0,
                       mode)


def stats_update(Gs, Ds, pl: TPlan, stats: np.ndarray, decay: float, weight: float, only_owner: int = -1,
                 blocks=None):
    """One statistics step (in place).  Returns (graft_num, block_status) like
    oracle.stats.stats_update: a non-finite block leaves H/D untouched, status 2."""
    nb = len(pl.blocks)
    num = np.zeros(nb, np.float64)
    status = np.zeros(nb, np.int32)
    for bi in (range(nb) if blocks is None else blocks):
        b = pl.blocks[bi]
        G = Gs[b.tensor_id]
        Gb = np.ascontiguousarray(G[b.slices()], np.float32)
        if not np.all(np.isfinite(Gb)):
            status[bi] = 2
            continue
        for i in range(b.order):
            if b.p[i] and (only_owner < 0 or b.owner[i] == only_owner):
                n = b.extent[i]
                S = ostats.stat_view(stats, b.off[i], n, b.ld[i])
                ostats.mode_stat(unfold(Gb, i), S, STAT_CHUNK, decay, weight)
        if Ds is not None:
            Db = np.ascontiguousarray(Ds[b.tensor_id][b.slices()], np.float32)
            g1 = Gb.reshape(1, -1)
            d1 = Db.reshape(1, -1)
            num[bi] = ostats.diag_update(g1, 0, 0, 1, g1.shape[1], d1)
            Ds[b.tensor_id][b.slices()] = d1.reshape(Db.shape)
    return num, status


def root_view(roots: np.ndarray, off: int, n: int, ld: int) -> np.ndarray:
    return roots[off:off + n * ld].reshape(n, ld)[:, :n]


def precondition_plan(Gs, Ds, pl: TPlan, roots: np.ndarray, graft_num=None, blocks=None):
    """P (fp64, shaped like G) for every tensor, per-block graft scales and
    den_b = ||P_b||^2.  Blocks with no kept mode: P_b = D_b^{-1/2} o G_b."""
    Ps = [np.full(np.shape(G), np.nan) for G in Gs]
    scales = np.zeros(len(pl.blocks))
    dens = np.zeros(len(pl.blocks))
    for bi in (range(len(pl.blocks)) if blocks is None else blocks):
        b = pl.blocks[bi]
        Gb = np.asarray(Gs[b.tensor_id][b.slices()], np.float64)
        if not any(b.p[:b.order]):
            D = np.maximum(np.asarray(Ds[b.tensor_id][b.slices()], np.float64), 1e-30)
            P = Gb / np.sqrt(D)
        else:
            P = Gb
            for i in range(b.order):
                if b.p[i]:
                    P = mode_product(P, root_view(roots, b.off[i], b.extent[i], b.ld[i]), i)
        Ps[b.tensor_id][b.slices()] = P
        dens[bi] = float(np.sum(P * P))
        if graft_num is not None:
            scales[bi] = float(np.sqrt(graft_num[bi]) / np.sqrt(dens[bi])) if dens[bi] > 0 else 0.0
    return Ps, scales, dens
