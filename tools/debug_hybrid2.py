import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_09018_b200 as shp, synth
from oracle import root as oroot
dev = "cuda:0"

def al(x): return (x + 255) // 256 * 256

def errh_of(batch, n, max_iter=100):
    np_ = (n + 63) // 64 * 64
    ws = shp._WS[(str(torch.device(dev)), "root")]
    off = al(batch * 7 * np_ * np_ * 8) + al(batch * 8)
    e = ws[off:off + batch * (max_iter + 1) * 8].view(torch.float64).reshape(batch, max_iter + 1)
    return e.cpu().numpy()

for n, eps in ((128, 1e-6), (128, 1e-3), (1024, 1e-6)):
    As = synth.psd_batch(n, 2, synth.BASE_SEED + 70 + n, "wishart")
    A = torch.from_numpy(As).to(dev)
    for k_sw in (8, 2, 100):
        X, info = shp.inverse_pth_root_batched(A, 4, fp64_iters=k_sw, eps_rel=eps)
        torch.cuda.synchronize()
        inf = shp.info_to_numpy(info)
        eh = errh_of(2, n)
        Xo, io = oroot.inverse_pth_root(As[0].astype(np.float64), 4, eps_rel=eps)
        e = np.linalg.norm(X[0].cpu().numpy() - Xo) / np.linalg.norm(Xo)
        print(f"n {n} eps {eps} k_sw {k_sw}: iters {inf[0]['iters']} status {inf[0]['status']} rel {e:.2e}")
        print("   err:", " ".join(f"{x:.1e}" for x in eh[0][:26]))
