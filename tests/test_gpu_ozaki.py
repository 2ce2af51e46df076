"""GPU parity of the Ozaki root (every coupled-Newton product on the INT8
tensor cores, exact int32 accumulation of S-slice splits)
against the fp64 oracle.  Bars: roots <= 1e-3 (north star), held to 1e-6 for
S = 7 (fp64-level products: measured 2e-7 at n = 1024, kappa 1e6) and to 1e-4
for S = 6 (host emulation tools/ozaki_precision.py: 3.8e-6 at n = 256);
iterations +-1; statuses equal; lambda_hat 1e-12 (the power iteration is the
FP64 kernel's)."""

import numpy as np
import pytest
import torch

import synth
from oracle import root as oroot

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def shp():
    import paper_2002_09018_b200 as shp
    return shp


def rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b)


# (precision mode, root bar): "ozaki" = the per-iteration slice schedule (reading #29, the bench's default),
# "ozaki7" / "ozaki6" = a fixed slice count for every product
MODES = [("ozaki", 1e-6), ("ozaki7", 1e-6), ("ozaki6", 1e-4)]


def _both(shp, As, p, tol=1e-7, max_iter=100, eps=1e-6, mode="ozaki"):
    A = torch.from_numpy(np.ascontiguousarray(As)).to(DEV)
    X, info = shp.inverse_pth_root_batched(A, p, fp64_iters=mode, tol=tol, max_iter=max_iter, eps_rel=eps)
    torch.cuda.synchronize()
    outs = [oroot.inverse_pth_root(a.astype(np.float64), p, eps, tol, max_iter) for a in As]
    return X.cpu().numpy(), shp.info_to_numpy(info), outs


@pytest.mark.parametrize("mode,bar", MODES)
@pytest.mark.parametrize("n", [64, 130, 200, 512])
def test_ozaki_p4_mixed(shp, n, mode, bar):
    As = synth.psd_batch(n, 4, synth.BASE_SEED + 170 + n, "mixed")
    Xg, inf, outs = _both(shp, As, 4, mode=mode)
    for i, (Xo, io) in enumerate(outs):
        assert rel(Xg[i], Xo) < bar, (i, rel(Xg[i], Xo))
        assert inf[i]["status"] == io.status == 0
        assert abs(int(inf[i]["iters"]) - io.iters) <= 1
        assert abs(inf[i]["lambda_max"] - io.lambda_max) <= 1e-12 * io.lambda_max


@pytest.mark.parametrize("mode,bar", MODES)
def test_ozaki_1024(shp, mode, bar):
    As = synth.psd_batch(1024, 2, synth.BASE_SEED + 2, "mixed")
    Xg, inf, outs = _both(shp, As, 4, mode=mode)
    for i, (Xo, io) in enumerate(outs):
        print(f"{mode} n=1024 matrix {i}: root rel err {rel(Xg[i], Xo):.3e}")
        assert rel(Xg[i], Xo) < bar
        assert inf[i]["status"] == 0 and abs(int(inf[i]["iters"]) - io.iters) <= 1


@pytest.mark.parametrize("mode,bar", MODES)
def test_ozaki_1024_p2(shp, mode, bar):
    """The bench's one-sided vocabulary roots: p = 2 at n = 1024 (3 products per iteration, T^2 sliced in the
    squaring's epilogue with the a-priori scale of reading #28)."""
    As = synth.psd_batch(1024, 2, synth.BASE_SEED + 12, "mixed")
    Xg, inf, outs = _both(shp, As, 2, mode=mode)
    for i, (Xo, io) in enumerate(outs):
        print(f"{mode} n=1024 p=2 matrix {i}: root rel err {rel(Xg[i], Xo):.3e}")
        assert rel(Xg[i], Xo) < bar
        assert inf[i]["status"] == io.status == 0 and abs(int(inf[i]["iters"]) - io.iters) <= 1


def test_ozaki_940_tiled_padding(shp):
    """The vocabulary remainder block (33708 = 32 x 1024 + 940): np = 960 and the tiled planes' row padding to 1024
    (the last A tile's second row block is padding), k padding 940 .. 959 zeroed by every writer."""
    As = synth.psd_batch(940, 2, synth.BASE_SEED + 940, "mixed")
    for p in (4, 2):
        Xg, inf, outs = _both(shp, As, p, mode="ozaki")
        for i, (Xo, io) in enumerate(outs):
            print(f"n=940 p={p} matrix {i}: root rel err {rel(Xg[i], Xo):.3e}")
            assert rel(Xg[i], Xo) < 2e-6
            assert inf[i]["status"] == io.status == 0 and abs(int(inf[i]["iters"]) - io.iters) <= 1


@pytest.mark.parametrize("mode,bar", [("ozaki7", 1e-6), ("ozaki", 2e-6)])
def test_ozaki_2048(shp, mode, bar):
    """n > 1024: the two-pass slicing path and 32 k-chunks per tile (config 5's b = 2048 blocks).  The slice
    schedule's products sum 2048 terms: measured 1.14e-6 on B200 (r02c, before the sqrt(n/1024) factor), so its
    bar here is 2e-6 (north star 1e-3)."""
    As = synth.psd_batch(2048, 1, synth.BASE_SEED + 5, "wishart")
    Xg, inf, outs = _both(shp, As, 4, mode=mode)
    Xo, io = outs[0]
    print(f"{mode} n=2048: root rel err {rel(Xg[0], Xo):.3e}, iters {inf[0]['iters']} vs {io.iters}")
    assert rel(Xg[0], Xo) < bar
    assert inf[0]["status"] == 0 and abs(int(inf[0]["iters"]) - io.iters) <= 1


@pytest.mark.parametrize("mode,bar", MODES)
@pytest.mark.parametrize("p", [1, 2, 3, 6, 8])
def test_ozaki_root_orders(shp, p, mode, bar):
    As = synth.psd_batch(130, 2, synth.BASE_SEED + 190 + p, "mixed")
    Xg, inf, outs = _both(shp, As, p, mode=mode)
    for i, (Xo, io) in enumerate(outs):
        assert rel(Xg[i], Xo) < bar * max(1, 4 // p) * (4 if p == 1 else 1), (p, i, rel(Xg[i], Xo))
        assert inf[i]["status"] == io.status


@pytest.mark.parametrize("mode,bar", MODES)
def test_ozaki_edge_cases(shp, mode, bar):
    n = 40
    As = np.zeros((5, n, n), np.float32)
    As[0] = np.eye(n)                                    # converges at k = 0 (never reaches the INT8 loop)
    As[1] = synth.wishart(n, 3)
    As[2] = 0.0                                          # degenerate -> I, status 3
    As[3] = synth.wishart(n, 4)
    As[3][5, 7] = As[3][7, 5] = np.nan                   # non-finite -> untouched, status 2
    As[4] = synth.spectrum(n, 6)
    A = torch.from_numpy(As).to(DEV)
    X = torch.full_like(A, 7.0)
    X, info = shp.inverse_pth_root_batched(A, 4, X=X, fp64_iters=mode)
    torch.cuda.synchronize()
    Xg, inf = X.cpu().numpy(), shp.info_to_numpy(info)
    assert inf[0]["status"] == 0 and inf[0]["iters"] == 0
    np.testing.assert_allclose(Xg[0], (1 + 1e-6) ** -0.25 * np.eye(n), rtol=1e-7, atol=0)
    assert inf[2]["status"] == 3 and np.array_equal(Xg[2], np.eye(n, dtype=np.float32))
    assert inf[3]["status"] == 2 and np.all(Xg[3] == 7.0)
    for i in (1, 4):
        Xo, io = oroot.inverse_pth_root(As[i].astype(np.float64), 4)
        assert rel(Xg[i], Xo) < bar and inf[i]["status"] == io.status


@pytest.mark.parametrize("mode,bar", MODES)
def test_ozaki_max_iter_and_stagnation(shp, mode, bar):
    As = synth.psd_batch(64, 2, 77, "wishart")
    Xg, inf, outs = _both(shp, As, 4, max_iter=3, mode=mode)
    for i, (Xo, io) in enumerate(outs):
        assert inf[i]["status"] == io.status == 1 and inf[i]["iters"] == io.iters == 3
        assert rel(Xg[i], Xo) < bar
    Xg, inf, outs = _both(shp, As, 4, tol=0.0, max_iter=200, mode=mode)
    for i, (Xo, io) in enumerate(outs):
        assert inf[i]["status"] == 1 and inf[i]["iters"] < 60
        assert rel(Xg[i], Xo) < bar


@pytest.mark.parametrize("mode", ["ozaki", "ozaki7", "ozaki6"])
def test_ozaki_determinism_and_batch_independence(shp, mode):
    As = synth.psd_batch(128, 40, 31, "mixed")
    X1, _ = shp.inverse_pth_root_batched(torch.from_numpy(As[:3]).to(DEV), 4, fp64_iters=mode)
    X2, _ = shp.inverse_pth_root_batched(torch.from_numpy(As).to(DEV), 4, fp64_iters=mode)
    X3, _ = shp.inverse_pth_root_batched(torch.from_numpy(As).to(DEV), 4, fp64_iters=mode)
    torch.cuda.synchronize()
    assert torch.equal(X2, X3)
    assert torch.equal(X1, X2[:3])



@pytest.mark.parametrize("mode", ["ozaki", "ozaki7", "ozaki6"])
def test_ozaki_power_bound_violation_is_flagged(shp, mode):
    """Reading #28: the squarings' a-priori row scale assumes eig(M_0) <= 2(p+1), i.e. a power-iteration
    lambda_hat within (p+1)x of lambda_max.  One power step on a matrix with one dominant eigenvalue gives
    lambda_hat ~ lambda_max / n, so T_0 has eigenvalues far below -1 and T^2 exceeds the bound: the root must
    report status 2 and leave X untouched (never a silently wrong root); a well-estimated batch mate is
    unaffected."""
    n = 256
    As = np.zeros((2, n, n), np.float32)
    As[0] = np.eye(n, dtype=np.float32)
    As[0][7, 7] = 1e6
    As[1] = synth.wishart(n, 11)
    A = torch.from_numpy(As).to(DEV)
    X = torch.full_like(A, 7.0)
    X, info = shp.inverse_pth_root_batched(A, 4, X=X, fp64_iters=mode, power_iters=1)
    torch.cuda.synchronize()
    inf = shp.info_to_numpy(info)
    assert inf[0]["lambda_max"] < 1e6 / 20  # the premise: lambda_max / lambda_hat > 2(p + 1)
    assert inf[0]["status"] == 2 and np.all(X[0].cpu().numpy() == 7.0)
    Xo, io = oroot.inverse_pth_root(As[1].astype(np.float64), 4, power_iters=1)
    assert inf[1]["status"] == io.status and rel(X[1].cpu().numpy(), Xo) < 1e-4


def test_ozaki_tail_graph_launches_and_bits():
    """The convergence-driven tail (a CUDA graph with a conditional WHILE node after the a-priori iteration
    estimate) replaces round 1's fixed max_iter launch loop.  In fresh processes: the default call launches ~7 x the
    estimate instead of ~7 x max_iter kernels with the roots, iteration counts and statuses of launching every
    iteration directly (SHAMPOO_OZAKI_DIRECT=all); and with the graph taking over at iteration 6
    (SHAMPOO_OZAKI_DIRECT=6, fixed 7 slices) the matrices iterate ~14 more times INSIDE the graph, still bit-identical
    to the direct launches."""
    import json
    import os
    import subprocess
    import sys
    code = r"""
import hashlib, json, sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2002_09018_b200 as shp, synth
out = {}
for name, mode in (("sched", "ozaki"), ("fixed7", "ozaki7")):
    A = torch.from_numpy(synth.psd_batch(512, 6, 41, "mixed")).to("cuda:0")
    X, info = shp.inverse_pth_root_batched(A, 4, fp64_iters=mode, max_iter=100)
    n_launch = shp.last_launch_count()
    torch.cuda.synchronize()
    inf = shp.info_to_numpy(info)
    out[name] = {"X": hashlib.sha256(X.cpu().numpy().tobytes()).hexdigest(),
                 "iters": inf["iters"].tolist(), "status": inf["status"].tolist(), "launches": n_launch}
print(json.dumps(out))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for env_val in (None, "all", "6"):
        env = dict(os.environ)
        env.pop("SHAMPOO_OZAKI_DIRECT", None)
        if env_val:
            env["SHAMPOO_OZAKI_DIRECT"] = env_val
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[env_val] = json.loads(r.stdout.strip().splitlines()[-1])
    for name in ("sched", "fixed7"):
        g, d = res[None][name], res["all"][name]
        print(name, "launches graph", g["launches"], "direct", d["launches"], "iters", g["iters"])
        assert g["X"] == d["X"] and g["iters"] == d["iters"] and g["status"] == d["status"]
        assert g["launches"] < 0.35 * d["launches"]
    early, d = res["6"]["fixed7"], res["all"]["fixed7"]
    print("graph from k = 6: launches", early["launches"], "iters", early["iters"])
    assert early["X"] == d["X"] and early["iters"] == d["iters"] and early["status"] == d["status"]
    assert min(early["iters"]) > 6 and early["launches"] < res[None]["fixed7"]["launches"]
