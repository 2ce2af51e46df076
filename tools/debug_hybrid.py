import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_09018_b200 as shp, synth
from oracle import root as oroot
dev = "cuda:0"
for n in (128, 1024):
    As = synth.psd_batch(n, 2, synth.BASE_SEED + 70 + n, "mixed")
    A = torch.from_numpy(As).to(dev)
    for k_sw in (-1, 100):
        X, info = shp.inverse_pth_root_batched(A, 4, fp64_iters=k_sw)
        torch.cuda.synchronize()
        inf = shp.info_to_numpy(info)
        for i in range(2):
            Xo, io = oroot.inverse_pth_root(As[i].astype(np.float64), 4)
            e = np.linalg.norm(X[i].cpu().numpy() - Xo) / np.linalg.norm(Xo)
            print(n, k_sw, i, "iters", inf[i]["iters"], "status", inf[i]["status"], "err", inf[i]["err"], "rel", e, "oracle iters", io.iters)
