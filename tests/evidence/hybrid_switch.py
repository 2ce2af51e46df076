import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2002_09018_b200 as shp, synth
from oracle import root as oroot
dev = "cuda:0"
n = 1024
As = synth.psd_batch(n, 4, synth.BASE_SEED + 2, "mixed")
ref = [oroot.inverse_pth_root(a.astype(np.float64), 4)[0] for a in As]
Ab = synth.wishart_batch_device(n, 148, synth.BASE_SEED + 2, torch.device(dev))
A = torch.from_numpy(As).to(dev)
for k_sw in (8, 10, 11, 12, -1, 100):
    X, info = shp.inverse_pth_root_batched(A, 4, fp64_iters=k_sw)
    torch.cuda.synchronize()
    errs = [np.linalg.norm(X[i].cpu().numpy() - ref[i]) / np.linalg.norm(ref[i]) for i in range(4)]
    inf = shp.info_to_numpy(info)
    Xb = torch.empty_like(Ab)
    shp.inverse_pth_root_batched(Ab, 4, X=Xb, fp64_iters=k_sw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); shp.inverse_pth_root_batched(Ab, 4, X=Xb, fp64_iters=k_sw); e1.record(); torch.cuda.synchronize()
    print(f"k_sw {k_sw}: max rel err {max(errs):.2e}  status {set(inf['status'].tolist())} iters {inf['iters'].tolist()} err {[f'{x:.1e}' for x in inf['err']]}  148 roots {e0.elapsed_time(e1):.1f} ms")
