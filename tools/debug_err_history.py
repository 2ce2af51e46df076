"""err_k = max|M_k - I| history of the Ozaki root (one 1024^2 Wishart matrix): runs with max_iter = k, tol = 0
for k = 1..K and prints info.err (the last check) -- compares SHAMPOO_OZAKI_DUAL=1/0 when run twice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_09018_b200 as shp  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
A = synth.wishart_batch_device(1024, 2, synth.BASE_SEED + 2, dev)
out = []
for k in range(1, int(sys.argv[1]) if len(sys.argv) > 1 else 24):
    X, info = shp.inverse_pth_root_batched(A, 4, max_iter=k, tol=0.0, fp64_iters="ozaki")
    torch.cuda.synchronize()
    inf = shp.info_to_numpy(info)
    out.append(f"{k}:{inf['err'][0]:.3e}/{inf['status'][0]}")
print(f"DUAL={os.environ.get('SHAMPOO_OZAKI_DUAL', '1')}", " ".join(out), flush=True)
