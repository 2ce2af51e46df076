"""Ozaki root vs the fp64 oracle and the FP64-DMMA path; timing of a 148/296-root batch."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_09018_b200 as shp, synth
from oracle import root as oroot
dev = "cuda:0"
for n in (128, 200, 1024):
    As = synth.psd_batch(n, 2, synth.BASE_SEED + 70 + n, "mixed")
    A = torch.from_numpy(As).to(dev)
    X, info = shp.inverse_pth_root_batched(A, 4, fp64_iters="ozaki")
    torch.cuda.synchronize()
    inf = shp.info_to_numpy(info)
    for i in range(2):
        Xo, io = oroot.inverse_pth_root(As[i].astype(np.float64), 4)
        e = np.linalg.norm(X[i].cpu().numpy() - Xo) / np.linalg.norm(Xo)
        print(f"n {n} mat {i}: ozaki iters {inf[i]['iters']} status {inf[i]['status']} err {inf[i]['err']:.2e} | oracle iters {io.iters} | rel {e:.2e}", flush=True)
Ab = synth.wishart_batch_device(1024, 296, synth.BASE_SEED + 2, torch.device(dev))
for mode in (None, "ozaki", None, "ozaki"):
    Xb = torch.empty_like(Ab)
    shp.inverse_pth_root_batched(Ab, 4, X=Xb, fp64_iters=mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); _, info = shp.inverse_pth_root_batched(Ab, 4, X=Xb, fp64_iters=mode); e1.record(); torch.cuda.synchronize()
    inf = shp.info_to_numpy(info)
    ms = e0.elapsed_time(e1)
    print(f"{mode or 'fp64'}: 296 roots {ms:.1f} ms = {296 / ms * 1e3:.1f} roots/s, iters {inf['iters'].mean():.2f}, status {set(inf['status'].tolist())}", flush=True)
