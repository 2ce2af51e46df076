import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_09018_b200 as shp, synth
from oracle import root as oroot
dev = "cuda:0"
n = 1024
As = synth.psd_batch(n, 1, synth.BASE_SEED + 2, "wishart")
A = torch.from_numpy(As).to(dev)
for k in range(9, 22):
    X, info = shp.inverse_pth_root_batched(A, 4, fp64_iters=8, max_iter=k, tol=0.0)
    torch.cuda.synchronize()
    Xo, io = oroot.inverse_pth_root(As[0].astype(np.float64), 4, max_iter=k, tol=0.0)
    inf = shp.info_to_numpy(info)
    e = np.linalg.norm(X[0].cpu().numpy() - Xo) / np.linalg.norm(Xo)
    print(f"max_iter {k}: gpu iters {inf[0]['iters']} err {inf[0]['err']:.2e} | oracle iters {io.iters} err {io.err:.2e} | rel diff {e:.2e}")
