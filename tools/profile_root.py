"""Launch the batched root kernel on a synthetic 1024^2 Wishart batch (for ncu).

    python tools/profile_root.py [--batch 148] [--n 1024] [--p 4] [--reps 2]
Prints the CUDA-event time of the last launch and the algorithmic FP64 rate.
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_09018_b200 as shp  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=148)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--max-iter", type=int, default=100)
ap.add_argument("--power-iters", type=int, default=100)
ap.add_argument("--slices", type=int, default=0, help="Ozaki slices with --hybrid -9 (0: the slice schedule)")
ap.add_argument("--digest", action="store_true", help="print a sha256 of the roots and lambda_max (bit-identity checks)")
ap.add_argument("--hybrid", type=int, default=None,
                help="fp64 iterations before the 3xTF32 tail (-1 = auto); -9 = the Ozaki INT8 root")
args = ap.parse_args()

dev = torch.device("cuda", 0)
A = synth.wishart_batch_device(args.n, args.batch, synth.BASE_SEED + 2, dev)
X = torch.empty_like(A)
for r in range(args.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    X, info = shp.inverse_pth_root_batched(A, args.p, X=X, max_iter=args.max_iter, power_iters=args.power_iters,
                                           fp64_iters=f"ozaki{args.slices or ''}" if args.hybrid == -9 else args.hybrid)
    e1.record()
    torch.cuda.synchronize()
inf = shp.info_to_numpy(info)
ms = e0.elapsed_time(e1)
n = args.n
prods = 2 + (args.p.bit_length() - 1) + (bin(args.p).count("1") - 1)
flops = float(inf["iters"].sum()) * prods * n * n * (n + 1)
print(f"{'fp64' if args.hybrid is None else (f"ozaki{args.slices or ''}" if args.hybrid == -9 else 'hybrid')} batch {args.batch} n {n} p {args.p}: {ms:.2f} ms, iters mean {inf['iters'].mean():.2f}, "
      f"status {set(inf['status'].tolist())}, {flops / ms / 1e9:.2f} TFLOP/s (sym-minimal), "
      f"{args.batch / ms * 1e3:.1f} roots/s")
if args.digest:
    import hashlib
    h = hashlib.sha256(X.cpu().numpy().tobytes() + inf["lambda_max"].tobytes()).hexdigest()
    print(f"digest {h} SHAMPOO_PI_GROUP={os.environ.get('SHAMPOO_PI_GROUP', '(default)')}")
