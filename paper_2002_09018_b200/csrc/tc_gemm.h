// tc_gemm.h -- host/device interface of the tcgen05 3xTF32 GEMM engine (tc_gemm.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace shp {

// One operand of a block-level GEMM, loaded by TMA as an exact (hi, lo) TF32 split.
// Element (k, r) of the operand lives at tensor coordinates (x + k, y + r[, z]).
struct TcOperand {
  int32_t map_hi, map_lo;  // indices into the CUtensorMap table
  int32_t x, y, z;
  int32_t dims;            // 2 or 3
};

// C[M x N] = A[M x K] . B[N x K]^T over 128x256 tiles (tiles_n = ceil(N/256)).
// A maps use a 128-row TMA box, B maps a kTcGemmBN-row box.
// out_mode 0: out_hi[i*ld + j] = C;  1: out_hi[j*ld + i] = C, out_lo[j*ld + i] = C - trunc_tf32(C).
struct TcJob {
  TcOperand a, b;
  int32_t M, N, K;
  int32_t out_mode;
  float* out_hi;
  float* out_lo;
  int64_t ld_out;
  int32_t tiles_n, pad;
  int64_t tile_begin;  // first global tile index of this job (jobs sorted)
};

// lo[i] = x - trunc_tf32(x) for x = src[i], i < n (n % 4 == 0, 16-B aligned).
// The tensor core truncates fp32 inputs to TF32 (measured:
// tools/probe_tf32_semantics.py), so the raw fp32 buffer serves as "hi" and
// only the exact remainder lo needs storing.
struct SplitSeg {
  const float* src;
  float* lo;
  int64_t n;
};

constexpr int kTcGemmBN = 256;  // output tile columns (= B box rows)
size_t tc_gemm_smem_bytes();
int make_map_f32(CUtensorMap* out, const void* base, int dims, const uint64_t* size, const uint64_t* stride_bytes,
                 int box_rows);
int tc_gemm_launch(const TcJob* jobs_dev, int n_jobs, int64_t total_tiles, const CUtensorMap* maps_dev,
                   cudaStream_t stream, int64_t* launches);
int tf32_split_launch(const SplitSeg* segs_dev, int n_segs, cudaStream_t stream, int64_t* launches);
int split_flat_launch(const float* x, float* lo, int64_t n, cudaStream_t stream, int64_t* launches);

}  // namespace shp
