"""f1 -- delayed, pipelined preconditioner refresh on the GPU.

The paper's central systems idea: inverse p-th roots are recomputed only every
kappa steps, from a snapshot of the statistics, off the critical path, and the
training step keeps using the previous ("stale") roots meanwhile
(Alg. 1: "Gather preconditioners
L_(t-kappa)^{-1/4} ... Send L_t, R_t to CPU host").  The paper runs the roots
on otherwise idle host CPUs.  On a GPU that is busy with the training step
there is no idle processor to hide behind, so this scheduler amortises the
refresh instead: at a kappa boundary it snapshots the rank's owned statistics
(one device copy), then every step runs the next chunk of the owned roots
(a few matrices, one batched root call per group slice) on the caller's
stream; when the last chunk is done it all-gathers the new roots into a
second buffer, which is adopted at the next kappa boundary.  The roots used
at step t therefore come from the statistics of step <= t - kappa and are at
most 2*kappa steps old, exactly as in Alg. 1.

Every chunk runs the same deterministic kernels as a one-shot refresh, so the
adopted roots are bit-identical to a synchronous refresh of the same snapshot
(tests/test_gpu_schedule.py).
"""

from __future__ import annotations

import math

import torch

from . import Plan, inverse_pth_root_ptr, new_info, tf32_split
from .dist import all_gather_roots


class DelayedRefresh:
    def __init__(self, plan: Plan, stats: torch.Tensor, roots: torch.Tensor, rank: int = 0, world_size: int = 1,
                 kappa: int = 500, spread: int | None = None, eps_rel: float = 1e-6, tol: float = 1e-7,
                 max_iter: int = 100, power_iters: int = 100, group=None, fp64_iters=None):
        self.plan, self.stats, self.rank, self.world = plan, stats, rank, world_size
        self.kappa = int(kappa)
        self.spread = max(1, min(int(spread if spread is not None else kappa), self.kappa))
        self.kw = dict(eps_rel=eps_rel, tol=tol, max_iter=max_iter, power_iters=power_iters)
        self.fp64_iters = fp64_iters  # root precision: None (FP64 DMMA), "ozaki", or a hybrid switch
        self.group = group
        self.current = roots                       # roots the step uses (stale by <= 2 kappa)
        self.next = torch.zeros_like(roots)        # roots being built from the last snapshot
        # TF32 remainder of the current roots for shampoo_precondition_split,
        # recomputed only when roots are adopted (once per kappa steps)
        self.current_lo = tf32_split(self.current)
        seg = plan.segment_elems
        self.seg0 = rank * seg
        self.snapshot = torch.empty(seg, dtype=stats.dtype, device=stats.device)
        # (group, first index, count) work units of this rank, and the chunking
        self.units = []
        for g in plan.groups_of(rank):
            self.units.append((g, 0, int(g["count"])))
        total = sum(u[2] for u in self.units)
        self.chunk = max(1, math.ceil(total / self.spread))
        self.pending: list = []
        self.ready = False       # self.next holds a complete, gathered refresh
        self.refreshes = 0
        self.infos: list = []

    def _schedule(self):
        work = []
        for g, first, count in self.units:
            i = first
            while i < first + count:
                n = min(self.chunk, first + count - i)
                work.append((g, i, n))
                i += n
        # pack units into per-step chunks of ~self.chunk matrices
        steps, cur, cur_n = [], [], 0
        for u in work:
            cur.append(u)
            cur_n += u[2]
            if cur_n >= self.chunk:
                steps.append(cur)
                cur, cur_n = [], 0
        if cur:
            steps.append(cur)
        return steps

    def _run(self, units, stream=None):
        for g, i, n in units:
            nn, p, r = int(g["n"]), int(g["p"]), int(g["r"])
            ld = (nn + 3) // 4 * 4
            off, stride = int(g["offset"]) + i * int(g["stride"]), int(g["stride"])
            info = new_info(n, self.stats.device)
            src = self.snapshot.data_ptr() + 4 * (off - self.seg0)
            dst = self.next.data_ptr() + 4 * off
            inverse_pth_root_ptr(src, ld, stride, dst, ld, stride, n, nn, p, info, device=self.stats.device,
                                 stream=stream, r=r, fp64_iters=self.fp64_iters if r == 1 else None, **self.kw)
            self.infos.append((g, i, n, info))

    def step(self, t: int, stream=None) -> bool:
        """Call once per training step t (after the statistics update).  Returns
        True when new roots were adopted at this step."""
        adopted = False
        if t % self.kappa == 0:
            if self.ready:
                self.current, self.next = self.next, self.current
                tf32_split(self.current, self.current_lo, stream)
                self.ready = False
                adopted = True
            seg = self.plan.segment_elems
            self.snapshot.copy_(self.stats[self.seg0:self.seg0 + seg])
            self.pending = self._schedule()
            self.infos = []
        if self.pending:
            self._run(self.pending.pop(0), stream)
            if not self.pending:
                all_gather_roots(self.plan, self.next, self.rank, self.world, self.group)
                self.ready = True
                self.refreshes += 1
        return adopted
