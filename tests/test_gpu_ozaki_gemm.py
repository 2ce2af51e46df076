"""The Ozaki INT8 GEMM itself, bit-exact: tools/microbench/ozaki_test.cu slices random operands on the GPU into the
tiled planes (ozaki.cuh), runs gemm_kernel<S, 64> for S = 5, 6, 7 (symmetric and general products, n = 200 ... 1024,
ragged and row-padded plane layouts) and compares EVERY checked output with the exact integer pair sums recomputed
on the host from the same slices, rounded once to fp64 -- 0 mismatches is the bar.  The binary is
built here when it is missing (nvcc, sm_100a)."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "microbench", "ozaki_test.cu")
BIN = os.path.join(ROOT, "tools", "microbench", "bin", "ozaki_test")


def _binary():
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(ROOT, "paper_2002_09018_b200", "csrc", "ozaki.cuh"))):
        os.makedirs(os.path.dirname(BIN), exist_ok=True)
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I",
                               os.path.join(ROOT, "paper_2002_09018_b200", "csrc"), SRC, "-lcuda", "-o", BIN],
                              timeout=600)
    return BIN


def test_ozaki_gemm_bitexact_vs_host_integer_sums():
    out = subprocess.run([_binary()], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = [ln for ln in out.stdout.splitlines() if "mismatches vs exact host" in ln]
    assert len(lines) >= 14
    for ln in lines:
        assert ln.split(":")[1].strip().startswith("0/"), ln
    assert out.stdout.strip().endswith("PASS")
