"""Multi-GPU sharding of the root refresh (row a7 / SURVEY §8(e)).

Roots of different blocks are independent units, distributed over all
processors as the paper distributes per-layer root work "across all the CPUs
that are part of the training system".  One process per GPU:

  * the plan assigns every statistic an owner rank (LPT over n^3 cost) and packs
    rank r's statistics into segment r of the packed buffer;
  * owners update only their L/R statistics (``only_owner = rank``), D and the
    graft numerator are updated everywhere (every rank preconditions all blocks);
  * each rank computes the roots of its segment, then ONE
    ``all_gather_into_tensor`` (NCCL over NVLink/NVSwitch) of the equal-size
    segments rebuilds the full roots buffer on every rank (in place for NCCL);
  * or (``refresh_gather_overlapped``) per root group: once the owners have
    computed a group, its region of every segment is broadcast from its owner on
    NCCL's stream while the next group computes -- the same bytes, but only the
    last group's transfer stays on the critical path;
  * or (``LayerShards``, reading #30) whole tensors per rank: a layer-granular
    plan (``make_plan(..., owners="tensor")``) gives every root of a tensor to
    one rank, which also updates that tensor's statistics and computes its
    preconditioned gradient; ONE all-gather of P (+ the graft scales) per step
    replaces the roots' all-gather and the replicated preconditioning.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

import numpy as np

from . import Plan, inverse_pth_root_ptr, last_launch_count, new_info, refresh_group_roots, subplan


def segment(plan: Plan, buf: torch.Tensor, rank: int) -> torch.Tensor:
    s = plan.segment_elems
    return buf[rank * s:(rank + 1) * s]


def all_gather_roots(plan: Plan, roots: torch.Tensor, rank: int, world_size: int, group=None):
    """Rebuild the full packed roots buffer from every rank's segment."""
    if world_size == 1:
        return
    mine = segment(plan, roots, rank)
    backend = dist.get_backend(group)
    if backend == "nccl":
        dist.all_gather_into_tensor(roots[:plan.stats_elems], mine, group=group)  # in place
    else:  # gloo (CPU tests): out-of-place
        out = torch.empty_like(roots[:plan.stats_elems])
        dist.all_gather_into_tensor(out, mine.clone(), group=group)
        roots[:plan.stats_elems].copy_(out)


def refresh_roots(plan: Plan, stats: torch.Tensor, roots: torch.Tensor, rank: int = 0, world_size: int = 1,
                  group=None, eps_rel: float = 1e-6, tol: float = 1e-7, max_iter: int = 100,
                  power_iters: int = 100, stream=None, fp64_iters="auto"):
    """Owner-sharded inverse p-th roots + all-gather.  Returns [(group, info)].
    fp64_iters: root precision as in ``refresh_group_roots`` (default "auto", the bench's path: the INT8 Ozaki
    root for n >= 512, FP64 DMMA below; None forces FP64 DMMA)."""
    infos = refresh_group_roots(plan, stats, roots, rank, eps_rel, tol, max_iter, power_iters, stream=stream,
                                fp64_iters=fp64_iters)
    all_gather_roots(plan, roots, rank, world_size, group)
    return infos


def _group_keys(plan: Plan):
    """(n, p, r) root groups in the plan's order: every rank walks the same sequence."""
    keys = []
    for g in plan.groups:
        k = (int(g["n"]), int(g["p"]), int(g["r"]))
        if k not in keys:
            keys.append(k)
    return keys


def _region(g):
    off, cnt, stride = int(g["offset"]), int(g["count"]), int(g["stride"])
    return off, cnt * stride


def refresh_gather_overlapped(plan: Plan, stats: torch.Tensor, roots: torch.Tensor, rank: int, world_size: int,
                              group=None, eps_rel: float = 1e-6, tol: float = 1e-7, max_iter: int = 100,
                              power_iters: int = 100, fp64_iters=None, compute_group=None):
    """Owner-sharded refresh with the root exchange overlapped (rows a5-a7): for every (n, p, r) group in the
    plan's order this rank computes its own roots of the group (``compute_group(g)``, default: the batched root
    call), then the group's region of EVERY rank's segment is broadcast from its owner (async, NCCL's stream
    waits for the launches enqueued so far) -- so group k's transfer runs under group k+1's roots.  On return
    the current stream waits for all transfers: the full roots buffer, as after ``all_gather_roots``.
    Returns ([(group, info)], kernel launches)."""
    out, launches, works = [], 0, []
    for key in _group_keys(plan):
        mine = [g for g in plan.groups_of(rank) if (int(g["n"]), int(g["p"]), int(g["r"])) == key]
        for g in mine:
            if compute_group is not None:
                compute_group(g)
                continue
            cnt, n, p, r = int(g["count"]), int(g["n"]), int(g["p"]), int(g["r"])
            off, stride = int(g["offset"]), int(g["stride"])
            ld = (n + 3) // 4 * 4
            info = new_info(cnt, stats.device)
            inverse_pth_root_ptr(stats.data_ptr() + 4 * off, ld, stride, roots.data_ptr() + 4 * off, ld, stride,
                                 cnt, n, p, info, eps_rel, tol, max_iter, power_iters, stats.device, None, r,
                                 fp64_iters if r == 1 else None)
            launches += last_launch_count()
            out.append((g, info))
        if world_size > 1:
            for src in range(world_size):
                for g in plan.groups_of(src):
                    if (int(g["n"]), int(g["p"]), int(g["r"])) != key:
                        continue
                    off, length = _region(g)
                    works.append(dist.broadcast(roots[off:off + length], src=src, group=group, async_op=True))
    for w in works:
        w.wait()
    return out, launches


class LayerShards:
    """Layer-granular sharding of the whole step (reading #30; "As preconditioners need to be computed
    for every layer of the network, we distribute the computation across all the CPUs").

    ``plan`` comes from ``make_plan(..., owners="tensor")``.  Rank r owns the tensors with ``tensor_owner == r``:
    ``sub[r]`` is the plan restricted to their blocks (statistics, D, graft numerator, roots and P of those
    blocks only).  The preconditioned gradients live in ONE flat fp32 buffer laid out rank-major: segment r holds
    rank r's tensors (index order, offsets rounded up to 4 elements = 16 bytes), then the graft scales of its
    blocks (``sub[r]`` order); every segment is padded to the largest (rounded up to 64 elements), so one
    ``all_gather_into_tensor`` of equal segments rebuilds every P and every scale on every rank."""

    def __init__(self, plan: Plan, world_size: int):
        if plan.tensor_owner is None:
            raise ValueError("LayerShards needs a layer-granular plan (make_plan(..., owners='tensor'))")
        self.world = world_size
        self.shapes = [tuple(s) for s in plan.shapes]
        self.owner = np.asarray(plan.tensor_owner, dtype=np.int64)
        tid = plan.blocks["tensor_id"].astype(np.int64)
        self.block_idx = [np.nonzero(self.owner[tid] == r)[0] for r in range(world_size)]
        self.sub = [subplan(plan, self.block_idx[r]) for r in range(world_size)]
        self.offset = np.zeros(len(self.shapes), dtype=np.int64)   # absolute offset of tensor t's P
        self.scale_off = np.zeros(world_size, dtype=np.int64)      # absolute offset of rank r's scales
        used = []
        for r in range(world_size):
            off = 0
            for t in range(len(self.shapes)):
                if self.owner[t] == r:
                    self.offset[t] = off
                    m, n = self.shapes[t]
                    off += (m * n + 3) // 4 * 4
            self.scale_off[r] = off
            used.append(off + len(self.block_idx[r]))
        self.segment = (max(used) + 63) // 64 * 64
        for t in range(len(self.shapes)):
            self.offset[t] += self.owner[t] * self.segment
        self.scale_off += np.arange(world_size, dtype=np.int64) * self.segment
        self.numel = self.segment * world_size

    def p_views(self, flat):
        """Row-major (m, n) views of every tensor's P inside the flat buffer."""
        out = []
        for t, (m, n) in enumerate(self.shapes):
            o = int(self.offset[t])
            out.append(flat[o:o + m * n].view(m, n))
        return out

    def scales_of(self, flat, rank: int):
        o = int(self.scale_off[rank])
        return flat[o:o + len(self.block_idx[rank])]

    def gather(self, flat, rank: int, group=None):
        """All-gather of the equal segments (in place for NCCL)."""
        if self.world == 1:
            return
        mine = flat[rank * self.segment:(rank + 1) * self.segment]
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(flat[:self.numel], mine, group=group)
        else:  # gloo (CPU tests): out-of-place
            out = torch.empty_like(flat[:self.numel])
            dist.all_gather_into_tensor(out, mine.clone(), group=group)
            flat[:self.numel].copy_(out)

    def unpack_scales(self, flat, scales_full):
        """Graft scales of every block (full-plan order) from the gathered segments."""
        for r in range(self.world):
            idx = torch.as_tensor(self.block_idx[r], device=scales_full.device)
            if idx.numel():
                scales_full.index_copy_(0, idx, self.scales_of(flat, r).to(scales_full.dtype))
