"""f1 -- delayed, pipelined preconditioner refresh on the GPU.

The paper's central systems idea: inverse p-th roots are recomputed only every
kappa steps, from a snapshot of the statistics, off the critical path, and the
training step keeps using the previous ("stale") roots meanwhile
(Alg. 1: "Gather preconditioners
L_(t-kappa)^{-1/4} ... Send L_t, R_t to CPU host").  The paper runs the roots
on otherwise idle host CPUs ("pipelined and runs asynchronously without
blocking the training loop").  Here the idle processor is the part of
the GPU the training step leaves unused: the refresh runs on its own
LOWEST-priority CUDA stream, concurrently with the step, in chunks small enough
that each of its launches holds the SMs only briefly (the block scheduler
serves the step's pending CTAs first).

Schedule of one kappa window starting at a boundary t0 (t0 % kappa == 0):
  * t0: adopt the roots gathered during the last window (if any) -- swap the
    buffers, TF32 remainder of the new current roots on the training stream;
    snapshot this rank's owned statistics (one device copy on the training
    stream, an event the refresh stream waits on);
  * t0 + j, j = 0 .. n_steps-1: enqueue chunk j of this rank's owned roots on
    the refresh stream (the host does not wait);
  * t0 + n_steps - 1: the training stream waits for the refresh stream and ONE
    all-gather rebuilds the new roots on every rank; they are adopted at the
    next boundary.
The roots used at step t therefore come from the statistics of step <= t - kappa
and are at most 2*kappa steps old, exactly as in Alg. 1.

n_steps (and so the step of the collective) is the same on every rank: it is
derived on the host from the whole plan -- the largest owned root count over the
ranks -- never from this rank's own count, so the all-gather is issued at the
same step everywhere and cannot be matched out of order with another collective
(a rank with fewer roots has empty chunk steps).

Every chunk runs the same deterministic kernels as a one-shot refresh, so the
adopted roots are bit-identical to a synchronous refresh of the same snapshot
(tests/test_gpu_schedule.py).
"""

from __future__ import annotations

import math

import torch

from . import Plan, inverse_pth_root_ptr, new_info, tf32_split
from .dist import all_gather_roots


def _owned_counts(plan: Plan, world_size: int):
    return [sum(int(g["count"]) for g in plan.groups_of(r)) for r in range(world_size)]


def chunking(plan: Plan, world_size: int, kappa: int, spread: int | None = None, chunk: int | None = None):
    """-> (chunk, n_steps): roots per step on the busiest rank and the number of chunk steps of a refresh.
    Rank-uniform: derived from the busiest rank's owned count (host-side, no collective)."""
    busiest = max(_owned_counts(plan, world_size) + [1])
    if chunk is None:
        sp = max(1, min(int(spread if spread is not None else kappa), kappa))
        chunk = math.ceil(busiest / sp)
    chunk = max(1, int(chunk))
    n_steps = math.ceil(busiest / chunk)
    if n_steps > kappa:
        raise ValueError(f"chunk {chunk} spreads the busiest rank's {busiest} roots over {n_steps} > kappa steps")
    return chunk, n_steps


def schedule_units(units, chunk: int, n_steps: int):
    """A rank's owned roots [(group, first, count)] cut into exactly n_steps per-step lists of (group, first,
    count) units, at most `chunk` roots per step in total (trailing lists may be empty)."""
    steps = [[] for _ in range(n_steps)]
    s, room = 0, chunk
    for g, first, count in units:
        i = first
        while i < first + count:
            if room == 0:
                s, room = s + 1, chunk
            n = min(room, first + count - i)
            steps[s].append((g, i, n))
            i += n
            room -= n
    return steps


class DelayedRefresh:
    def __init__(self, plan: Plan, stats: torch.Tensor, roots: torch.Tensor, rank: int = 0, world_size: int = 1,
                 kappa: int = 500, spread: int | None = None, eps_rel: float = 1e-6, tol: float = 1e-7,
                 max_iter: int = 100, power_iters: int = 100, group=None, fp64_iters="auto",
                 chunk: int | None = None, stream: torch.cuda.Stream | None = None, gather_roots: bool = True):
        """spread: the number of steps a refresh is spread over (<= kappa; default: as many as the chunk size
        needs, at most kappa).  chunk: roots per step on the busiest rank (default: ceil(max owned / spread)).
        stream: the refresh stream (default: a new lowest-priority stream on the statistics' device).
        gather_roots: all-gather the new roots at the end of the window (root shards); False for layer shards
        (``make_plan(..., owners="tensor")``), whose roots stay with their owner -- the step then exchanges P."""
        self.plan, self.stats, self.rank, self.world = plan, stats, rank, world_size
        self.kappa = int(kappa)
        self.kw = dict(eps_rel=eps_rel, tol=tol, max_iter=max_iter, power_iters=power_iters)
        self.fp64_iters = fp64_iters  # root precision: "auto" (Ozaki for n >= 512), None (FP64 DMMA), "ozaki"...
        self.group = group
        self.gather_roots = gather_roots
        self.current = roots                       # roots the step uses (stale by <= 2 kappa)
        self.next = torch.zeros_like(roots)        # roots being built from the last snapshot
        # TF32 remainder of the current roots for shampoo_precondition_split,
        # recomputed only when roots are adopted (once per kappa steps)
        self.current_lo = tf32_split(self.current)
        seg = plan.segment_elems
        self.seg0 = rank * seg
        self.snapshot = torch.empty(seg, dtype=stats.dtype, device=stats.device)
        self.chunk, self.n_steps = chunking(plan, world_size, self.kappa, spread, chunk)
        self.units = [(g, 0, int(g["count"])) for g in plan.groups_of(rank)]
        if stream is None:
            lo, _hi = torch.cuda.Stream.priority_range()  # (lowest, highest); lowest = least urgent
            stream = torch.cuda.Stream(device=stats.device, priority=lo)
        self.stream = stream
        self.ev_snap = torch.cuda.Event()
        self.ev_done = torch.cuda.Event()
        self.pending: list = []
        self.ready = False       # self.next holds a complete, gathered refresh
        self.refreshes = 0
        self.infos: list = []

    def _schedule(self):
        return schedule_units(self.units, self.chunk, self.n_steps)

    def _run(self, units):
        """Enqueue one chunk on the refresh stream (all allocations made on that stream)."""
        with torch.cuda.stream(self.stream):
            for g, i, n in units:
                nn, p, r = int(g["n"]), int(g["p"]), int(g["r"])
                ld = (nn + 3) // 4 * 4
                off, stride = int(g["offset"]) + i * int(g["stride"]), int(g["stride"])
                info = new_info(n, self.stats.device)
                src = self.snapshot.data_ptr() + 4 * (off - self.seg0)
                dst = self.next.data_ptr() + 4 * off
                inverse_pth_root_ptr(src, ld, stride, dst, ld, stride, n, nn, p, info, device=self.stats.device,
                                     stream=self.stream, r=r, fp64_iters=self.fp64_iters if r == 1 else None,
                                     ws_tag="delayed_refresh", **self.kw)
                self.infos.append((g, i, n, info))

    def step(self, t: int) -> bool:
        """Call once per training step t, on the training stream, after the statistics update.  Returns True
        when new roots were adopted at this step (use ``current`` / ``current_lo`` for the preconditioning)."""
        adopted = False
        cur = torch.cuda.current_stream(self.stats.device)
        if t % self.kappa == 0:
            if self.ready:
                self.current, self.next = self.next, self.current
                tf32_split(self.current, self.current_lo)
                self.ready = False
                adopted = True
            seg = self.plan.segment_elems
            # the snapshot's previous readers and `next`'s previous readers (the preconditioning of the steps
            # before this boundary) are ordered before this point of the training stream
            self.snapshot.copy_(self.stats[self.seg0:self.seg0 + seg])
            self.ev_snap.record(cur)
            self.stream.wait_event(self.ev_snap)
            self.pending = self._schedule()
            self.infos = []
        if self.pending:
            self._run(self.pending.pop(0))
            if not self.pending:
                self.ev_done.record(self.stream)
                cur.wait_event(self.ev_done)  # the gather (on the training stream / NCCL's) sees finished roots
                if self.gather_roots:
                    all_gather_roots(self.plan, self.next, self.rank, self.world, self.group)
                self.ready = True
                self.refreshes += 1
        return adopted
