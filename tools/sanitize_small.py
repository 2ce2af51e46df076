"""Small invocations of every kernel family for compute-sanitizer (memcheck)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_09018_b200 as shp, synth
dev = "cuda:0"
for n in (40, 130):
    A = torch.from_numpy(synth.psd_batch(n, 3, 5, "mixed")).to(dev)
    for mode in (None, "ozaki", -1):
        shp.inverse_pth_root_batched(A, 4, fp64_iters=mode)
    shp.inverse_pth_root_batched(A, 8, r=3)
    X, info = shp.inverse_pth_root_batched(A, 6)
    shp.root_residual_batched(A, X, 6, info)
shapes = [(200, 130), (64, 1), (300, 2048)]
pl = shp.make_plan(shapes, 128, 1024, 1)
Gs = [torch.randn(s, device=dev) for s in shapes]
Ds = [torch.zeros_like(G) for G in Gs]
Ps = [torch.zeros_like(G) for G in Gs]
t = shp.TensorTable(Gs, Ds, Ps)
st = torch.zeros(pl.stats_elems, device=dev)
gn = torch.zeros(pl.n_blocks, dtype=torch.float64, device=dev)
shp.stats_update(t, pl, st, 1.0, 1.0, -1, gn)
roots = torch.zeros_like(st)
shp.refresh_group_roots(pl, st, roots, 0, fp64_iters="ozaki")
shp.precondition(t, pl, roots, gn, torch.zeros(pl.n_blocks, device=dev), roots_lo=shp.tf32_split(roots))
tshapes = [(3, 3, 8, 40), (50,), (5, 70, 3)]
tp = shp.make_tensor_plan(tshapes, 32, 4096, 1)
TG = [torch.randn(s, device=dev) for s in tshapes]
TD = [torch.zeros_like(g) for g in TG]
TP = [torch.zeros_like(g) for g in TG]
tt = shp.TTensorTable(TG, TD, TP)
ts = torch.zeros(tp.stats_elems, device=dev)
tg = torch.zeros(tp.n_blocks, dtype=torch.float64, device=dev)
shp.tensor_stats_update(tt, tp, ts, 1.0, 1.0, -1, tg)
tr = torch.zeros_like(ts)
shp.refresh_group_roots(tp, ts, tr, 0)
shp.tensor_precondition(tt, tp, tr, tg, torch.zeros(tp.n_blocks, device=dev))
torch.cuda.synchronize()
print("sanitize run ok")
