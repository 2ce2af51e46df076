"""Oracle: preconditioned gradient and grafting (rows a8, a9).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy, fp64.

* Two-sided block:   P_b = L_b^{-1/4} G_b R_b^{-1/4}
* One-sided block:   P_b = G_b R_b^{-1/2}  or  L_b^{-1/2} G_b
* No side kept:      P_b = D_b^{-1/2} o G_b (grafted diagonal AdaGrad; the
                     plan "degenerates to grafted diagonal AdaGrad", S:261 --
                     DESIGN.md reading #17; D clamped at 1e-30, reading #11)
* Grafting per block (blocks are "treated as a separate tensor", P:398;
  reading #9), instantaneous ratio of §5.1 (reading #10):
      num_b = ||D^{-1/2} o G_b||_F^2 = sum g^2 / max(D, 1e-30)   (from the stats step)
      den_b = ||P_b||_F^2
      scale_b = sqrt(num_b) / sqrt(den_b)    (0 when den_b == 0)
  so that ||scale_b P_b||_F = ||D^{-1/2} o G_b||_F (the grafting identity).
"""

from __future__ import annotations

import numpy as np


def precondition_block(G_b, XL=None, XR=None, D_b=None) -> np.ndarray:
    G_b = np.asarray(G_b, np.float64)
    if XL is None and XR is None:
        D = np.maximum(np.asarray(D_b, np.float64), 1e-30)
        return G_b / np.sqrt(D)
    P = G_b
    if XL is not None:
        P = np.asarray(XL, np.float64) @ P
    if XR is not None:
        P = P @ np.asarray(XR, np.float64)
    return P


def graft_numerator(G_b, D_b) -> float:
    G_b = np.asarray(G_b, np.float64)
    return float(np.sum(G_b * G_b / np.maximum(np.asarray(D_b, np.float64), 1e-30)))


def graft_scale(num: float, den: float) -> float:
    if den == 0.0:
        return 0.0
    return float(np.sqrt(num) / np.sqrt(den))


def precondition_plan(Gs, Ds, pl, roots: np.ndarray, graft_num=None, blocks=None):
    """P for every tensor of the plan (fp64 arrays shaped like G) and the per-block
    graft scale.  ``roots``: packed buffer (same offsets as the statistics).
    ``blocks``: optional subset of block indices (sampled parity); other
    entries of P are left NaN."""
    Ps = [np.full(G.shape, np.nan) for G in Gs]
    scales = np.zeros(len(pl.blocks))
    dens = np.zeros(len(pl.blocks))
    idx = range(len(pl.blocks)) if blocks is None else blocks
    for bi in idx:
        b = pl.blocks[bi]
        G = Gs[b.tensor_id]
        Gb = G[b.row0:b.row0 + b.rows, b.col0:b.col0 + b.cols]
        XL = XR = Db = None
        if b.p_left:
            XL = roots[b.left_off:b.left_off + b.rows * b.left_ld].reshape(b.rows, b.left_ld)[:, :b.rows]
        if b.p_right:
            XR = roots[b.right_off:b.right_off + b.cols * b.right_ld].reshape(b.cols, b.right_ld)[:, :b.cols]
        if XL is None and XR is None:
            Db = Ds[b.tensor_id][b.row0:b.row0 + b.rows, b.col0:b.col0 + b.cols]
        P = precondition_block(Gb, XL, XR, Db)
        Ps[b.tensor_id][b.row0:b.row0 + b.rows, b.col0:b.col0 + b.cols] = P
        dens[bi] = float(np.sum(P * P))
        if graft_num is not None:
            scales[bi] = graft_scale(float(graft_num[bi]), dens[bi])
    return Ps, scales, dens


def momentum_step_block(W, M, Pm, G, D, P, beta1: float, eta0: float, shampoo_branch: bool):
    """f2: the tail of Alg. 1 for one block (reading #9), in
    place on fp32 state arrays W, M, Pm (views of the block); arithmetic in fp64,
    every stored value rounded to fp32; norms over the stored fp32 values.
        M  <- beta1 M + (1-beta1) D^{-1/2} o G                 (line 12)
        t > tau: Pm <- beta1 Pm + (1-beta1) P                  (line 18)
                 eta = eta0 ||M||_F / ||Pm||_F  (0 if ||Pm|| = 0)  (line 19)
                 W <- W - eta Pm                               (line 20)
        else:    eta = eta0;  W <- W - eta0 M                  (lines 22-23)
    Returns eta."""
    g = np.asarray(G, np.float64)
    d = np.maximum(np.asarray(D, np.float64), 1e-30)
    M[...] = (beta1 * M.astype(np.float64) + (1.0 - beta1) * (g / np.sqrt(d))).astype(np.float32)
    if shampoo_branch:
        Pm[...] = (beta1 * Pm.astype(np.float64) + (1.0 - beta1) * np.asarray(P, np.float64)).astype(np.float32)
        nm = float(np.sum(M.astype(np.float64) ** 2))
        npm = float(np.sum(Pm.astype(np.float64) ** 2))
        eta = eta0 * np.sqrt(nm) / np.sqrt(npm) if npm > 0 else 0.0
        W[...] = (W.astype(np.float64) - eta * Pm.astype(np.float64)).astype(np.float32)
    else:
        eta = eta0
        W[...] = (W.astype(np.float64) - eta0 * M.astype(np.float64)).astype(np.float32)
    return float(eta)
