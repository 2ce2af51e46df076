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
    segments rebuilds the full roots buffer on every rank (in place for NCCL).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import Plan, refresh_group_roots


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
                  power_iters: int = 100, stream=None):
    """Owner-sharded inverse p-th roots + all-gather.  Returns [(group, info)]."""
    infos = refresh_group_roots(plan, stats, roots, rank, eps_rel, tol, max_iter, power_iters, stream=stream)
    all_gather_roots(plan, roots, rank, world_size, group)
    return infos
