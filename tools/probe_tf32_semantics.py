"""Does tcgen05.mma.kind::tf32 truncate or round fp32 inputs with non-zero low
mantissa bits?  (Ran against commit 'tcgen05 ... 3xTF32 GEMM engine' + the
SHAMPOO_PROBE_RAW_TF32 knob of its split kernel; result recorded in
profiles/r01_tf32_probe.txt: P == trunc_tf32(G) for 100% of elements.  The
current split kernel has no knob: it relies on that result.)  Feeds raw fp32 G (SHAMPOO_PROBE_RAW_TF32=1: hi = x, lo = 0) and
identity roots through the precondition GEMMs: P = X_L G X_R = G exactly in
exact arithmetic; compare with trunc_tf32(G) and rna_tf32(G)."""
import os, sys
os.environ["SHAMPOO_PROBE_RAW_TF32"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_09018_b200 as shp
from synth import gaussian
G = gaussian((128, 128), 1)
pl = shp.make_plan([G.shape], 128, 8192, 1)
b = pl.blocks[0]
roots = np.zeros(pl.stats_elems, np.float32)
for off, ld in ((int(b["left_off"]), int(b["left_ld"])), (int(b["right_off"]), int(b["right_ld"]))):
    roots[off:off + 128 * ld].reshape(128, ld)[:, :128] = np.eye(128)
Gd = torch.from_numpy(G).cuda(); Pd = torch.zeros_like(Gd)
shp.precondition(shp.TensorTable([Gd], [torch.ones_like(Gd)], [Pd]), pl, torch.from_numpy(roots).cuda())
P = Pd.cpu().numpy()
u = G.view(np.uint32)
trunc = (u & np.uint32(0xFFFFE000)).view(np.float32)
# round-to-nearest (ties away) to 10 mantissa bits
rna = ((u + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)
print("P == G      :", np.mean(P == G))
print("P == trunc  :", np.mean(P == trunc))
print("P == rna    :", np.mean(P == rna))
