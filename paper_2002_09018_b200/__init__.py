"""paper_2002_09018_b200 -- B200-native data-parallel hot path of distributed Shampoo
(Anil et al., "Second Order Optimization Made Practical", arXiv 2002.09018).

Thin Python binding over the C ABI of ``libshampoo.so`` (include/shampoo.h).
PyTorch supplies device memory, streams and process groups only; every step of
the hot path (statistics, power iteration, coupled-Newton roots, residual,
preconditioning, grafting) runs in the library's sm_100a kernels.  There is no
CPU fallback: importing the package raises if the library is not built.

Rows of the hot path:
  a1  make_plan                     blocking plan, exponents, owners, packing
  a2  stats_update                  L/R statistics, D, graft numerator (bit-exact)
  a3-a6 inverse_pth_root_batched    power iteration + ridge + coupled Newton
        root_residual_batched       ||X^p A_hat - I||_F check
  a7  dist.refresh_roots            owner-sharded roots + NCCL all-gather
  a8-a9 precondition                L^{-1/p} G R^{-1/p} and the graft scale
  f2  momentum_step                 Alg. 1 tail (momentum, grafted step, update)
  f3  make_tensor_plan, tensor_stats_update, tensor_precondition
                                    order-1..4 tensors (per-mode statistics, mode products)
  f4  make_plan(split=(a, d)), inverse_root_rational_batched
                                    L^{-a/2d} G R^{-(d-a)/2d}, roots S^{-r/p}
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import (BLOCK_DTYPE, GROUP_DTYPE, ROOT_INFO_DTYPE, STATE_DTYPE, TBLOCK_DTYPE, TENSOR_DTYPE,
                   TTENSOR_DTYPE, ShampooError, check, last_launch_count)

_lib.lib()  # fail loudly at import if the CUDA library is missing

__all__ = [
    "Plan", "make_plan", "TensorTable", "stats_update", "inverse_pth_root_batched", "root_residual_batched",
    "precondition", "root_workspace_bytes", "inverse_root_rational_batched", "ShampooError", "last_launch_count", "ROOT_INFO_DTYPE",
]


def _stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


_WS: dict = {}


def workspace(nbytes: int, device, tag: str = "default", stream=None) -> torch.Tensor:
    """Cached device workspace (torch allocations are >= 512-B aligned), one per (device, tag, stream) and
    allocated ON the stream the library call runs on: the caching allocator then reuses a replaced (smaller)
    workspace's memory only in that stream's order, never under a launch still running on it."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    key = (str(device), tag, int(s.cuda_stream))
    w = _WS.get(key)
    if w is None or w.numel() < nbytes:
        _WS.pop(key, None)
        with torch.cuda.stream(s):
            w = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _WS[key] = w
    return w


def free_workspaces():
    _WS.clear()


# ----------------------------------------------------------------------- a1
@dataclass
class Plan:
    shapes: list
    block_size: int
    max_precond_dim: int
    world_size: int
    blocks: np.ndarray
    groups: np.ndarray
    stats_elems: int
    segment_elems: int
    _dev: dict = field(default_factory=dict, repr=False)
    tensor_owner: np.ndarray | None = None   # layer-granular plans (owners="tensor"): owner rank of every tensor

    @property
    def n_blocks(self) -> int:
        return int(self.blocks.shape[0])

    def device_blocks(self, device) -> torch.Tensor:
        key = str(device)
        if key not in self._dev:
            self._dev[key] = torch.from_numpy(self.blocks.view(np.uint8).copy()).to(device)
        return self._dev[key]

    def groups_of(self, owner: int):
        return [g for g in self.groups if int(g["owner"]) == owner]


def make_plan(shapes, block_size: int = 1024, max_precond_dim: int = 8192, world_size: int = 1,
              split=(1, 2), owners: str = "root") -> Plan:
    """split = (a, d): the Lemma's 1/p = a/d (f4); (1, 2) -> L^{-1/4} G R^{-1/4}.
    owners: "root" -- every root assigned LPT on its own (shampoo_plan); "tensor" -- whole tensors (layers)
    assigned LPT, every root of a tensor on its owner (shampoo_plan_layers, reading #30)."""
    if owners not in ("root", "tensor"):
        raise ValueError("owners must be 'root' or 'tensor'")
    L = _lib.lib()
    fn = L.shampoo_plan if owners == "root" else L.shampoo_plan_layers
    sa, sd = int(split[0]), int(split[1])
    sh = np.ascontiguousarray(np.asarray(shapes, dtype=np.int64).reshape(-1, 2))
    nb = np.zeros(1, np.int32)
    ng = np.zeros(1, np.int32)
    se = np.zeros(1, np.int64)
    sg = np.zeros(1, np.int64)
    towner = np.zeros(max(1, sh.shape[0]), np.int32)
    extra = (towner.ctypes.data,) if owners == "tensor" else ()
    check(fn(sh.ctypes.data, sh.shape[0], block_size, max_precond_dim, world_size, sa, sd, None, 0,
             nb.ctypes.data, None, 0, ng.ctypes.data, se.ctypes.data, sg.ctypes.data, *extra))
    blocks = np.zeros(int(nb[0]), BLOCK_DTYPE)
    groups = np.zeros(int(ng[0]), GROUP_DTYPE)
    check(fn(sh.ctypes.data, sh.shape[0], block_size, max_precond_dim, world_size, sa, sd,
             blocks.ctypes.data, blocks.shape[0], nb.ctypes.data, groups.ctypes.data, groups.shape[0],
             ng.ctypes.data, se.ctypes.data, sg.ctypes.data, *extra))
    return Plan([tuple(map(int, s)) for s in sh], block_size, max_precond_dim, world_size, blocks, groups,
                int(se[0]), int(sg[0]), tensor_owner=towner[:sh.shape[0]].copy() if owners == "tensor" else None)


def subplan(plan: Plan, block_indices) -> Plan:
    """The plan restricted to some of its blocks (same packed offsets and groups): e.g. the blocks of one
    rank's tensors in a layer-granular plan.  Per-block outputs (graft numerator / scale) of calls made with it
    are indexed by position in ``block_indices``."""
    idx = np.asarray(block_indices, dtype=np.int64)
    return Plan(plan.shapes, plan.block_size, plan.max_precond_dim, plan.world_size,
                np.ascontiguousarray(plan.blocks[idx]), plan.groups, plan.stats_elems, plan.segment_elems,
                tensor_owner=plan.tensor_owner)


# ------------------------------------------------------------- tensor table
class TensorTable:
    """Device table of shampoo_tensor_t for lists of G (grad), D and P tensors.
    Tensors must stay alive (and keep their storage) while the table is used."""

    def __init__(self, Gs, Ds=None, Ps=None):
        n = len(Gs)
        Ds = Ds if Ds is not None else [None] * n
        Ps = Ps if Ps is not None else [None] * n
        host = np.zeros(n, TENSOR_DTYPE)
        self.device = Gs[0].device
        for i, (G, D, P) in enumerate(zip(Gs, Ds, Ps)):
            for name, T in (("G", G), ("D", D), ("P", P)):
                if T is None:
                    continue
                if T.dtype != torch.float32 or T.dim() != 2 or T.stride(1) != 1 or T.device != self.device:
                    raise ValueError(f"tensor {i} {name}: need a row-major 2-D float32 tensor on {self.device}")
                if tuple(T.shape) != tuple(G.shape):
                    raise ValueError(f"tensor {i} {name}: shape {tuple(T.shape)} != G {tuple(G.shape)}")
            host[i]["G"] = G.data_ptr()
            host[i]["ldg"] = G.stride(0)
            host[i]["m"], host[i]["n"] = G.shape
            if D is not None:
                host[i]["D"], host[i]["ldd"] = D.data_ptr(), D.stride(0)
            if P is not None:
                host[i]["P"], host[i]["ldp"] = P.data_ptr(), P.stride(0)
        self.host = host
        self.n = n
        self.dev = torch.from_numpy(host.view(np.uint8).copy()).to(self.device)
        self._keep = (list(Gs), list(Ds), list(Ps))


# ----------------------------------------------------------------------- a2
def stats_update(table: TensorTable, plan: Plan, stats: torch.Tensor, decay: float = 1.0, weight: float = 1.0,
                 only_owner: int = -1, graft_num: torch.Tensor | None = None,
                 block_status: torch.Tensor | None = None, stream=None):
    """One statistics step over every block (one call, one launch sequence)."""
    assert stats.dtype == torch.float32 and stats.is_contiguous() and stats.numel() >= plan.stats_elems
    L = _lib.lib()
    nb = plan.n_blocks
    wsb = L.shampoo_stats_workspace_bytes(plan.blocks.ctypes.data, nb, only_owner)
    ws = workspace(wsb, stats.device, "stats", stream)
    check(L.shampoo_stats_update(table.dev.data_ptr(), table.n, plan.device_blocks(stats.device).data_ptr(),
                                 plan.blocks.ctypes.data, nb, only_owner, stats.data_ptr(), float(decay), float(weight),
                                 graft_num.data_ptr() if graft_num is not None else None,
                                 block_status.data_ptr() if block_status is not None else None,
                                 ws.data_ptr(), ws.numel(), _stream_ptr(stream)))


# -------------------------------------------------------------------- a3-a6
def root_workspace_bytes(batch: int, n: int, p: int, max_iter: int = 100) -> int:
    return int(_lib.lib().shampoo_root_workspace_bytes(batch, n, p, max_iter))


def inverse_pth_root_ptr(A_ptr: int, lda: int, stride_a: int, X_ptr: int, ldx: int, stride_x: int, batch: int,
                         n: int, p: int, info: torch.Tensor, eps_rel: float = 1e-6, tol: float = 1e-7,
                         max_iter: int = 100, power_iters: int = 100, device=None, stream=None, r: int = 1,
                         fp64_iters: int | None = None, ws_tag: str = "root"):
    """X = A_hat^{-r/p} (r = 1: shampoo_inverse_pth_root_batched, else the rational entry).
    fp64_iters (r = 1 only): hybrid FP64 -> 3xTF32 tensor-core root (-1 = automatic switch);
    fp64_iters="ozaki": every product on the INT8 tensor cores with the per-iteration slice schedule
    (reading #29: 7 slices while the ridge-bounded amplification is large, down to 5; SLICE_BUDGET);
    fp64_iters="ozaki7" / "ozaki6": 7 / 6 slices for every product;
    fp64_iters="auto" / "auto7" / "auto6": "ozaki" / "ozaki7" / "ozaki6" for n >= OZAKI_MIN_N, FP64 DMMA below.
    ws_tag: workspace cache key -- calls that may run concurrently on different streams need different tags."""
    L = _lib.lib()
    if fp64_iters in ("auto", "auto6", "auto7") and r == 1:  # the library picks Ozaki (n >= 512) or FP64 DMMA
        slices = int(fp64_iters[4:] or 7)
        budget = SLICE_BUDGET if fp64_iters == "auto" else 0.0
        wsb = L.shampoo_root_auto_workspace_bytes(batch, n, p, max_iter)
        ws = workspace(wsb, device if device is not None else info.device, ws_tag, stream)
        check(L.shampoo_inverse_pth_root_batched_auto(A_ptr, lda, stride_a, X_ptr, ldx, stride_x, batch, n, p, eps_rel,
                                                      tol, max_iter, power_iters, slices, budget, info.data_ptr(),
                                                      ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
        return
    if fp64_iters in ("auto", "auto6", "auto7"):  # rational roots (r > 1): the FP64 path
        fp64_iters = None
    if isinstance(fp64_iters, str) and fp64_iters.startswith("ozaki"):
        slices = int(fp64_iters[5:] or 7)
        budget = SLICE_BUDGET if fp64_iters == "ozaki" else 0.0
        if r != 1:
            raise ValueError("the ozaki root serves r = 1 only")
        wsb = L.shampoo_root_ozaki_workspace_bytes(batch, n, p, max_iter)
        ws = workspace(wsb, device if device is not None else info.device, ws_tag, stream)
        check(L.shampoo_inverse_pth_root_batched_ozaki(A_ptr, lda, stride_a, X_ptr, ldx, stride_x, batch, n, p, eps_rel,
                                                       tol, max_iter, power_iters, slices, budget, info.data_ptr(),
                                                       ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
        return
    wsb = L.shampoo_root_workspace_bytes(batch, n, p, max_iter)
    ws = workspace(wsb, device if device is not None else info.device, ws_tag, stream)
    if fp64_iters is not None:
        if r != 1:
            raise ValueError("the hybrid root serves r = 1 only")
        check(L.shampoo_inverse_pth_root_batched_hybrid(A_ptr, lda, stride_a, X_ptr, ldx, stride_x, batch, n, p,
                                                        eps_rel, tol, max_iter, power_iters, fp64_iters,
                                                        info.data_ptr(), ws.data_ptr(), ws.numel(),
                                                        _stream_ptr(stream)))
    elif r == 1:
        check(L.shampoo_inverse_pth_root_batched(A_ptr, lda, stride_a, X_ptr, ldx, stride_x, batch, n, p, eps_rel, tol,
                                                 max_iter, power_iters, info.data_ptr(), ws.data_ptr(), ws.numel(),
                                                 _stream_ptr(stream)))
    else:
        check(L.shampoo_inverse_root_rational_batched(A_ptr, lda, stride_a, X_ptr, ldx, stride_x, batch, n, p, r,
                                                      eps_rel, tol, max_iter, power_iters, info.data_ptr(),
                                                      ws.data_ptr(), ws.numel(), _stream_ptr(stream)))


def new_info(batch: int, device) -> torch.Tensor:
    return torch.zeros(batch * ROOT_INFO_DTYPE.itemsize, dtype=torch.uint8, device=device)


def info_to_numpy(info: torch.Tensor) -> np.ndarray:
    return info.cpu().numpy().view(ROOT_INFO_DTYPE)


def inverse_pth_root_batched(A: torch.Tensor, p: int, X: torch.Tensor | None = None, eps_rel: float = 1e-6,
                             tol: float = 1e-7, max_iter: int = 100, power_iters: int = 100,
                             info: torch.Tensor | None = None, stream=None, r: int = 1,
                             fp64_iters: int | None = None):
    """A: (batch, n, n) or (n, n) float32 CUDA tensor (row stride >= n, unit column stride).
    Returns (X, info) with X like A and info a uint8 tensor of shampoo_root_info_t."""
    squeeze = A.dim() == 2
    A3 = A.unsqueeze(0) if squeeze else A
    assert A3.dtype == torch.float32 and A3.is_cuda and A3.stride(2) == 1
    batch, n, n2 = A3.shape
    assert n == n2
    if X is None:
        X = torch.empty_like(A3)
    X3 = X.unsqueeze(0) if X.dim() == 2 else X
    if info is None:
        info = new_info(batch, A3.device)
    inverse_pth_root_ptr(A3.data_ptr(), A3.stride(1), A3.stride(0), X3.data_ptr(), X3.stride(1), X3.stride(0), batch,
                         n, p, info, eps_rel, tol, max_iter, power_iters, A3.device, stream, r, fp64_iters)
    return (X3[0] if squeeze else X3), info


def inverse_root_rational_batched(A: torch.Tensor, p: int, r: int, **kw):
    """X = A_hat^{-r/p} (f4): the p-th root raised to the power r."""
    return inverse_pth_root_batched(A, p, r=r, **kw)


def root_residual_batched(A: torch.Tensor, X: torch.Tensor, p: int, info: torch.Tensor, eps_rel: float = 1e-6,
                          stream=None) -> torch.Tensor:
    A3 = A.unsqueeze(0) if A.dim() == 2 else A
    X3 = X.unsqueeze(0) if X.dim() == 2 else X
    batch, n, _ = A3.shape
    L = _lib.lib()
    out = torch.empty(batch, dtype=torch.float64, device=A3.device)
    wsb = L.shampoo_root_residual_workspace_bytes(batch, n, p)
    ws = workspace(wsb, A3.device, "residual", stream)
    check(L.shampoo_root_residual_batched(A3.data_ptr(), A3.stride(1), A3.stride(0), X3.data_ptr(), X3.stride(1),
                                          X3.stride(0), batch, n, p, eps_rel, info.data_ptr(), out.data_ptr(),
                                          ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
    return out


_refresh_launches = 0
# smallest n for which precision "auto" picks the Ozaki root (measured on B200: n = 128 ozaki 19k roots/s vs
# FP64 DMMA 72k; n = 512 2.7k vs 2.5k; n = 1024 580 vs 354 -- profiles/r01t_*)
OZAKI_MIN_N = 512  # = SHAMPOO_OZAKI_MIN_N of include/shampoo.h (the library's "auto" switch; for reporting)
# per-iteration slice schedule of the Ozaki root (reading #29, shampoo.h slice_budget): iteration k takes the fewest
# slices S in [5, 7] with 2^-(7S-1) sqrt(n/1024) / (p min(1, eps_rel g^k)) <= SLICE_BUDGET (host emulation at n = 1024, p = 4,
# kappa 1e6: 0.68 of the fixed-7 slice products, root error 2.9e-7 vs 1.2e-7; tools/ozaki_schedule.py)
SLICE_BUDGET = 1e-9


def last_refresh_launch_count() -> int:
    """Kernel launches enqueued by the last refresh_group_roots call (all groups)."""
    return _refresh_launches


def refresh_group_roots(plan: Plan, stats: torch.Tensor, roots: torch.Tensor, owner: int, eps_rel: float = 1e-6,
                        tol: float = 1e-7, max_iter: int = 100, power_iters: int = 100, infos=None, stream=None,
                        fp64_iters: int | None = None):
    """Inverse p-th roots of every statistic owned by `owner` (one batched call per
    (n, p) group); roots land at the statistics' offsets."""
    global _refresh_launches
    _refresh_launches = 0
    out = []
    for g in plan.groups_of(owner):
        cnt, n, p, r = int(g["count"]), int(g["n"]), int(g["p"]), int(g["r"])
        off, stride = int(g["offset"]), int(g["stride"])
        ld = (n + 3) // 4 * 4
        info = new_info(cnt, stats.device)
        inverse_pth_root_ptr(stats.data_ptr() + 4 * off, ld, stride, roots.data_ptr() + 4 * off, ld, stride, cnt, n,
                             p, info, eps_rel, tol, max_iter, power_iters, stats.device, stream, r,
                             fp64_iters if r == 1 else None)
        _refresh_launches += last_launch_count()
        out.append((g, info))
    if infos is not None:
        infos.extend(out)
    return out


# -------------------------------------------------------------------- a8-a9
def tf32_split(x: torch.Tensor, lo: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """lo = x - trunc_tf32(x) (the remainder of the tensor cores' TF32 split), e.g. of
    the packed roots once per refresh; pass it to precondition(..., roots_lo=lo)."""
    assert x.dtype == torch.float32 and x.is_contiguous()
    if lo is None:
        lo = torch.empty_like(x)
    n = x.numel() // 4 * 4
    check(_lib.lib().shampoo_tf32_split(x.data_ptr(), lo.data_ptr(), n, _stream_ptr(stream)))
    return lo


def precondition(table: TensorTable, plan: Plan, roots: torch.Tensor, graft_num: torch.Tensor | None = None,
                 graft_scale: torch.Tensor | None = None, den: torch.Tensor | None = None, stream=None,
                 roots_lo: torch.Tensor | None = None):
    """P for every block (3xTF32 tcgen05 / FP64 DMMA) and the per-block graft scale.
    roots_lo: optional precomputed tf32_split(roots) (once per refresh)."""
    L = _lib.lib()
    nb = plan.n_blocks
    th, bh = table.host, plan.blocks
    wsb = L.shampoo_precondition_workspace_bytes(th.ctypes.data, table.n, bh.ctypes.data, nb)
    ws = workspace(wsb, roots.device, "precondition", stream)
    check(L.shampoo_precondition_split(th.ctypes.data, table.n, bh.ctypes.data, nb, roots.data_ptr(),
                                 roots_lo.data_ptr() if roots_lo is not None else None,
                                 graft_num.data_ptr() if graft_num is not None else None,
                                 graft_scale.data_ptr() if graft_scale is not None else None,
                                 den.data_ptr() if den is not None else None, ws.data_ptr(), ws.numel(),
                                 _stream_ptr(stream)))


# ----------------------------------------------------------------------- f2
class StateTable:
    """Device table of shampoo_state_t (W, M, Pm per tensor), parallel to a TensorTable."""

    def __init__(self, Ws, Ms, Pms):
        host = np.zeros(len(Ws), STATE_DTYPE)
        for i, (W, M, Pm) in enumerate(zip(Ws, Ms, Pms)):
            for T in (W, M, Pm):
                if T.dtype != torch.float32 or T.dim() != 2 or T.stride(1) != 1:
                    raise ValueError(f"state {i}: need row-major 2-D float32 tensors")
            host[i] = (W.data_ptr(), M.data_ptr(), Pm.data_ptr(), W.stride(0), M.stride(0), Pm.stride(0))
        self.host = host
        self.n = len(Ws)
        self.dev = torch.from_numpy(host.view(np.uint8).copy()).to(Ws[0].device)
        self._keep = (list(Ws), list(Ms), list(Pms))


def momentum_step(table: TensorTable, states: StateTable, plan: Plan, beta1: float, eta0: float,
                  shampoo_branch: bool, eta_out: torch.Tensor | None = None, stream=None):
    """Alg. 1 lines 12, 17-23 per block: momentum of both directions, grafted step
    size and the parameter update (f2)."""
    L = _lib.lib()
    nb = plan.n_blocks
    ws = workspace(L.shampoo_momentum_workspace_bytes(nb), table.device, "momentum", stream)
    check(L.shampoo_momentum_step(table.dev.data_ptr(), states.dev.data_ptr(), table.n,
                                  plan.device_blocks(table.device).data_ptr(), nb, float(beta1), float(eta0),
                                  1 if shampoo_branch else 0, eta_out.data_ptr() if eta_out is not None else None,
                                  ws.data_ptr(), ws.numel(), _stream_ptr(stream)))


# ----------------------------------------------------------------------- f3
def make_tensor_plan(shapes, block_size: int = 1024, max_precond_dim: int = 8192, world_size: int = 1) -> Plan:
    """Plan for tensors of order 1..4 (shampoo_tensor_plan); ``blocks`` holds TBLOCK_DTYPE."""
    L = _lib.lib()
    n = len(shapes)
    dims = np.ones((max(n, 1), 4), np.int64)
    orders = np.zeros(max(n, 1), np.int32)
    for i, s in enumerate(shapes):
        s = tuple(int(d) for d in s)
        if not 1 <= len(s) <= 4:
            raise ValueError(f"tensor {i}: order must be 1..4")
        dims[i, :len(s)] = s
        orders[i] = len(s)
    nb = np.zeros(1, np.int32)
    ng = np.zeros(1, np.int32)
    se = np.zeros(1, np.int64)
    sg = np.zeros(1, np.int64)
    check(L.shampoo_tensor_plan(dims.ctypes.data, orders.ctypes.data, n, block_size, max_precond_dim, world_size,
                                None, 0, nb.ctypes.data, None, 0, ng.ctypes.data, se.ctypes.data, sg.ctypes.data))
    blocks = np.zeros(int(nb[0]), TBLOCK_DTYPE)
    groups = np.zeros(int(ng[0]), GROUP_DTYPE)
    check(L.shampoo_tensor_plan(dims.ctypes.data, orders.ctypes.data, n, block_size, max_precond_dim, world_size,
                                blocks.ctypes.data, blocks.shape[0], nb.ctypes.data, groups.ctypes.data,
                                groups.shape[0], ng.ctypes.data, se.ctypes.data, sg.ctypes.data))
    return Plan([tuple(int(d) for d in s) for s in shapes], block_size, max_precond_dim, world_size, blocks, groups,
                int(se[0]), int(sg[0]))


class TTensorTable:
    """HOST table of shampoo_ttensor_t for lists of contiguous G / D / P tensors (order 1..4)."""

    def __init__(self, Gs, Ds=None, Ps=None):
        n = len(Gs)
        Ds = Ds if Ds is not None else [None] * n
        Ps = Ps if Ps is not None else [None] * n
        host = np.zeros(n, TTENSOR_DTYPE)
        self.device = Gs[0].device
        for i, (G, D, P) in enumerate(zip(Gs, Ds, Ps)):
            if not 1 <= G.dim() <= 4:
                raise ValueError(f"tensor {i}: order must be 1..4")
            for name, T in (("G", G), ("D", D), ("P", P)):
                if T is None:
                    continue
                if T.dtype != torch.float32 or not T.is_contiguous() or T.device != self.device:
                    raise ValueError(f"tensor {i} {name}: need a contiguous float32 tensor on {self.device}")
                if tuple(T.shape) != tuple(G.shape):
                    raise ValueError(f"tensor {i} {name}: shape {tuple(T.shape)} != G {tuple(G.shape)}")
            host[i]["G"] = G.data_ptr()
            host[i]["D"] = D.data_ptr() if D is not None else 0
            host[i]["P"] = P.data_ptr() if P is not None else 0
            host[i]["dims"][:] = 1
            host[i]["dims"][:G.dim()] = G.shape
            host[i]["order"] = G.dim()
        self.host = host
        self.n = n
        self._keep = (list(Gs), list(Ds), list(Ps))


def tensor_stats_update(table: TTensorTable, plan: Plan, stats: torch.Tensor, decay: float = 1.0,
                        weight: float = 1.0, only_owner: int = -1, graft_num: torch.Tensor | None = None,
                        block_status: torch.Tensor | None = None, stream=None):
    """Per-mode statistics, D and graft numerator for every tensor block (f3)."""
    L = _lib.lib()
    nb = plan.n_blocks
    th, bh = table.host, plan.blocks
    wsb = L.shampoo_tensor_stats_workspace_bytes(th.ctypes.data, table.n, bh.ctypes.data, nb, only_owner)
    ws = workspace(wsb, stats.device, "tstats", stream)
    check(L.shampoo_tensor_stats_update(th.ctypes.data, table.n, bh.ctypes.data, nb, only_owner, stats.data_ptr(),
                                        float(decay), float(weight),
                                        graft_num.data_ptr() if graft_num is not None else None,
                                        block_status.data_ptr() if block_status is not None else None,
                                        ws.data_ptr(), ws.numel(), _stream_ptr(stream)))


def tensor_precondition(table: TTensorTable, plan: Plan, roots: torch.Tensor, graft_num: torch.Tensor | None = None,
                        graft_scale: torch.Tensor | None = None, den: torch.Tensor | None = None, stream=None):
    """P_B = B x_0 X_0 x_1 X_1 ... for every tensor block and the graft scale (f3)."""
    L = _lib.lib()
    nb = plan.n_blocks
    th, bh = table.host, plan.blocks
    wsb = L.shampoo_tensor_precondition_workspace_bytes(th.ctypes.data, table.n, bh.ctypes.data, nb)
    ws = workspace(wsb, roots.device, "tprecondition", stream)
    check(L.shampoo_tensor_precondition(th.ctypes.data, table.n, bh.ctypes.data, nb, roots.data_ptr(),
                                        graft_num.data_ptr() if graft_num is not None else None,
                                        graft_scale.data_ptr() if graft_scale is not None else None,
                                        den.data_ptr() if den is not None else None, ws.data_ptr(), ws.numel(),
                                        _stream_ptr(stream)))


# ----------------------------------------------------------------- profiling
def profile_begin():
    """Bracket the library's dominant kernels with CUDA events (bench roofline)."""
    check(_lib.lib().shampoo_profile_begin())


def profile_end(kernel: str | None = None):
    """-> (summed ms, launches) of `kernel` ("root_kernel", "ozaki_gemm") since profile_begin()."""
    ms = np.zeros(1, np.float64)
    n = np.zeros(1, np.int64)
    check(_lib.lib().shampoo_profile_end(kernel.encode() if kernel else None, ms.ctypes.data, n.ctypes.data))
    return float(ms[0]), int(n[0])


def ozaki_iteration_slices(k: int, p: int, n: int = 1024, eps_rel: float = 1e-6, budget: float | None = None,
                           slices: int = 7) -> int:
    """Slices of the M-chain products of Ozaki iteration k (reading #29; the library's schedule)."""
    b = SLICE_BUDGET if budget is None else budget
    return int(_lib.lib().shampoo_ozaki_iteration_slices(k, p, n, eps_rel, b, slices))


def ozaki_int8_ops(iters, n: int, p: int, eps_rel: float = 1e-6, budget: float | None = None,
                   slices: int = 7) -> float:
    """Algorithmic int8 ops of an Ozaki root call: per matrix and iteration, each symmetric product takes
    S(S+1)/2 slice products of n^2 (n+1) ops (upper triangle incl. the diagonal, 2 ops per multiply-add);
    the X-update at min(S, 5) under a schedule.  `iters`: iterations per matrix (root info)."""
    b = SLICE_BUDGET if budget is None else budget
    prods = (p.bit_length() - 1) + bin(p).count("1")  # T^p chain (squarings + multiplications) + T^p M
    per_k = []
    for k in range(int(max(iters)) if len(iters) else 0):
        S = ozaki_iteration_slices(k, p, n, 1e-6 if eps_rel is None else eps_rel, b, slices)
        Sx = min(S, 5) if b > 0 else S
        per_k.append(Sx * (Sx + 1) // 2 + prods * S * (S + 1) // 2)
    cum = np.concatenate([[0], np.cumsum(per_k)])
    return float(sum(cum[int(i)] for i in iters)) * n * n * (n + 1)


def profile_launch_ms(kernel: str | None = None) -> np.ndarray:
    """After profile_end(): per-launch milliseconds of `kernel`, in launch order."""
    L = _lib.lib()
    n = np.zeros(1, np.int64)
    key = kernel.encode() if kernel else None
    check(L.shampoo_profile_launch_ms(key, None, 0, n.ctypes.data))
    out = np.zeros(max(1, int(n[0])), np.float32)
    check(L.shampoo_profile_launch_ms(key, out.ctypes.data, out.shape[0], n.ctypes.data))
    return out[:int(n[0])]
