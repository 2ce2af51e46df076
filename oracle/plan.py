"""Oracle: blocking plan, exponents, root owners and packed offsets (row a1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain Python integers.

Rule (DESIGN.md §3 readings #5, #12, #13, #17):
* A side of a tensor is preconditioned iff ``1 < dim <= max_precond_dim``
  ("we bypass preconditioning of excessively large dimensions").
* Exponents: both sides kept -> p_L = p_R = 4 (L^{-1/4} G R^{-1/4});
  one side kept -> p = 2 on that side ("G R^{-1/2} and L^{-1/2} G",
  P:388-390); none -> 0/0 (grafted diagonal AdaGrad direction).
  f4 ("L^{-1/2p} G R^{-1/2q}" for 1/p + 1/q = 1; reading #23):
  split = (a, d) sets 1/p = a/d, so a two-sided block uses the exponents
  e_L = a/(2d) and e_R = (d-a)/(2d); each is stored reduced as r/p_root
  (root = S^{-r/p_root}), p_root <= 16.  The default (1, 2) is (1/4, 1/4).
* Blocking: each axis is split into ceil(dim/b) contiguous ranges, the last
  one ragged ("divide the tensor into blocks ... treating individual block as
  a separate tensor").  Blocks are ordered tensor by tensor (caller
  order), row-major over the block grid.
* Roots: a block contributes a left root (n = rows) if p_L > 0 and a right
  root (n = cols) if p_R > 0.  Cost = n^3 * products_per_iteration(p).
  Owners: roots sorted by (-cost, tensor_id, block_index, side) and assigned
  longest-processing-time first to the least-loaded rank (lowest rank on
  ties) -- "we distribute the computation across all the CPUs".
  owners="tensor" (reading #30, "As preconditioners need to be computed for
  every layer of the network, we distribute the computation"):
  tensors sorted by (-cost_t, t) with cost_t = sum over the tensor's roots of
  n^3 (products_per_iteration(p) + 12) + m*n (the +12: a root's time on the
  Ozaki path hardly depends on p -- measured), each assigned to the
  least-loaded rank (lowest on ties); every root of tensor t is owned by t's
  owner.
* Packing: one fp32 buffer holds all statistics (and, at the same offsets,
  all roots).  Rank r's segment holds the roots it owns, grouped by (n desc,
  p desc, r desc), each matrix ``n x ld`` with ``ld = roundup(n, 4)`` and a group
  stride ``roundup(n*ld, 64)``.  Every segment is padded to the largest one
  (rounded up to 64 elements) so an all-gather of equal segments rebuilds the
  whole buffer.
"""

from __future__ import annotations

from dataclasses import dataclass, field


def products_per_iteration(p: int) -> int:
    """Matrix products per coupled-Newton iteration (the iteration of S:131):
    X*T, T^p by the left-to-right binary chain (bitlen(p)-1 squarings plus
    popcount(p)-1 multiplications by T), and T^p * M."""
    return 2 + (p.bit_length() - 1) + (bin(p).count("1") - 1)


def reduce_exponent(num: int, den: int):
    """num/den in lowest terms -> (r, p)."""
    from math import gcd
    g = gcd(num, den)
    return num // g, den // g


def _roundup(x: int, m: int) -> int:
    return (x + m - 1) // m * m


@dataclass
class Block:
    tensor_id: int
    block_index: int  # index inside the global block list
    row0: int
    col0: int
    rows: int
    cols: int
    p_left: int
    p_right: int
    r_left: int = 0
    r_right: int = 0
    owner_left: int = -1
    owner_right: int = -1
    left_off: int = -1
    right_off: int = -1
    left_ld: int = 0
    right_ld: int = 0


@dataclass
class RootGroup:
    owner: int
    n: int
    p: int
    offset: int
    count: int
    stride: int
    r: int = 1


@dataclass
class Plan:
    blocks: list = field(default_factory=list)
    groups: list = field(default_factory=list)
    stats_elems: int = 0
    segment_elems: int = 0
    loads: list = field(default_factory=list)
    tensor_owner: list | None = None


def plan(shapes, block_size: int, max_precond_dim: int, world_size: int, split=(1, 2), owners: str = "root") -> Plan:
    if block_size < 1 or max_precond_dim < 1 or world_size < 1:
        raise ValueError("block_size, max_precond_dim and world_size must be >= 1")
    sa, sd = split
    if not (1 <= sa < sd):
        raise ValueError("split (a, d) needs 1 <= a < d")
    rl2, pl2 = reduce_exponent(sa, 2 * sd)
    rr2, pr2 = reduce_exponent(sd - sa, 2 * sd)
    if max(pl2, pr2) > 16:
        raise ValueError("split exponents need a root order <= 16")
    out = Plan()
    for t, (m, n) in enumerate(shapes):
        if m < 1 or n < 1:
            raise ValueError("tensor dims must be >= 1")
        left = 1 < m <= max_precond_dim
        right = 1 < n <= max_precond_dim
        if left and right:
            (pl, rl), (pr, rr) = (pl2, rl2), (pr2, rr2)
        elif left:
            (pl, rl), (pr, rr) = (2, 1), (0, 0)
        elif right:
            (pl, rl), (pr, rr) = (0, 0), (2, 1)
        else:
            (pl, rl), (pr, rr) = (0, 0), (0, 0)
        nbr = -(-m // block_size)
        nbc = -(-n // block_size)
        for bi in range(nbr):
            for bj in range(nbc):
                r0, c0 = bi * block_size, bj * block_size
                out.blocks.append(Block(t, len(out.blocks), r0, c0,
                                        min(block_size, m - r0), min(block_size, n - c0), pl, pr, rl, rr))
    # roots: (cost, tensor, block, side)
    roots = []
    for b in out.blocks:
        if b.p_left:
            roots.append((b.rows ** 3 * products_per_iteration(b.p_left), b.tensor_id, b.block_index, 0))
        if b.p_right:
            roots.append((b.cols ** 3 * products_per_iteration(b.p_right), b.tensor_id, b.block_index, 1))
    roots.sort(key=lambda r: (-r[0], r[1], r[2], r[3]))
    tensor_owner = None
    if owners == "tensor":
        tcost = [m * n for (m, n) in shapes]
        for _cost, t, bidx, side in roots:
            b = out.blocks[bidx]
            nn, pp = (b.rows, b.p_left) if side == 0 else (b.cols, b.p_right)
            tcost[t] += nn ** 3 * (products_per_iteration(pp) + 12)
        tload = [0] * world_size
        tensor_owner = [0] * len(shapes)
        for t in sorted(range(len(shapes)), key=lambda t: (-tcost[t], t)):
            r = min(range(world_size), key=lambda i: (tload[i], i))
            tload[r] += tcost[t]
            tensor_owner[t] = r
    elif owners != "root":
        raise ValueError("owners must be 'root' or 'tensor'")
    loads = [0] * world_size
    owned = [[] for _ in range(world_size)]  # (n, p, r, sort position, block, side)
    for pos, (cost, t_, bidx, side) in enumerate(roots):
        if tensor_owner is not None:
            r = tensor_owner[t_]
        else:
            r = min(range(world_size), key=lambda i: (loads[i], i))
        loads[r] += cost
        b = out.blocks[bidx]
        nn = b.rows if side == 0 else b.cols
        pp = b.p_left if side == 0 else b.p_right
        rr_ = b.r_left if side == 0 else b.r_right
        if side == 0:
            b.owner_left = r
        else:
            b.owner_right = r
        owned[r].append((nn, pp, rr_, pos, bidx, side))
    # packing, segment by segment
    seg_used = []
    for r in range(world_size):
        items = sorted(owned[r], key=lambda x: (-x[0], -x[1], -x[2], x[3]))
        off = 0
        i = 0
        while i < len(items):
            nn, pp, rr_ = items[i][0], items[i][1], items[i][2]
            j = i
            while j < len(items) and items[j][:3] == (nn, pp, rr_):
                j += 1
            ld = _roundup(nn, 4)
            stride = _roundup(nn * ld, 64)
            out.groups.append(RootGroup(r, nn, pp, off, j - i, stride, rr_))  # offset relative to segment for now
            for k in range(i, j):
                _, _, _, _, bidx, side = items[k]
                b = out.blocks[bidx]
                if side == 0:
                    b.left_off, b.left_ld = off + (k - i) * stride, ld
                else:
                    b.right_off, b.right_ld = off + (k - i) * stride, ld
            off += (j - i) * stride
            i = j
        seg_used.append(off)
    seg = _roundup(max(seg_used) if seg_used else 0, 64)
    out.segment_elems = seg
    out.stats_elems = seg * world_size
    for g in out.groups:
        g.offset += g.owner * seg
    for b in out.blocks:
        if b.left_off >= 0:
            b.left_off += b.owner_left * seg
        if b.right_off >= 0:
            b.right_off += b.owner_right * seg
    out.loads = loads
    out.tensor_owner = tensor_owner
    return out
