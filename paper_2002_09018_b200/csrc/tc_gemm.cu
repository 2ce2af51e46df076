// tc_gemm.cu -- 3xTF32 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   C[M x N] = A[M x K] . B[N x K]^T   (both operands K-major, fp32 in HBM)
//
// fp32-accurate products from TF32 tensor-core passes: every operand is an
// exact split x = hi + lo, hi = trunc_tf32(x) -- which is what the tensor core
// reads from the raw fp32 x -- and lo = x - hi (stored separately); the three
// passes lo.hi + hi.lo + hi.hi accumulate into one fp32 TMEM accumulator (the
// dropped lo.lo term and lo's own truncation are ~2^-20 relative; measured P
// error ~2e-6, bar 1e-3).  Used by the
// preconditioned gradient (row a8), whose error bar is 1e-3.
//
// Kernel structure (one CTA per SM, persistent over 128x128 output tiles):
//   warp 0      TMA producer: per 32-wide k-tile loads A_hi, A_lo, B_hi, B_lo
//               (4 x 16 KB, SWIZZLE_128B) into a 3-stage ring (full/empty mbarriers)
//   warp 1      TMEM allocator + single-thread MMA issuer: 4 k-steps x 3 passes of
//               tcgen05.mma.cta_group::1.kind::tf32 M=128 N=128 K=8 per k-tile,
//               tcgen05.commit -> empty[stage]; after the last k-tile -> tmem_full
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x16 from the (double-buffered) TMEM
//               accumulator, masked stores (row-major, or transposed + hi/lo split)
// Work items are (job, tile) pairs; a job is one block-level GEMM (see TcJob).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.h"
#include "tc_common.cuh"
#include "tc_gemm.h"

namespace shp {

// 128 x 256 output tiles: per 32-deep k-tile the MMAs read 4 KB of A and 8 KB
// of B per 128x256x8 step (180 cycles) and TMA writes 96 KB per 2160 MMA
// cycles -- ~112 B/clk of shared-memory traffic, under the 128 B/clk port
// (128 x 128 tiles needed ~150 B/clk and were shared-memory bound at 64%).
constexpr int kTcBM = 128, kTcBN = 256, kTcBK = 32;  // BK in fp32 elements (128 bytes)
constexpr int kTcStages = 2;
constexpr int kTcTileBytes = kTcBM * kTcBK * 4;      // 16 KB (A)
constexpr int kTcBTileBytes = kTcBN * kTcBK * 4;     // 32 KB (B)
constexpr int kTcStageBytes = 2 * kTcTileBytes + 2 * kTcBTileBytes;  // A_hi, A_lo, B_hi, B_lo
constexpr int kTcThreads = 192;
constexpr uint32_t kTcTmemCols = 2 * kTcBN;          // two fp32 accumulators

size_t tc_gemm_smem_bytes() { return 1024 + (size_t)kTcStages * kTcStageBytes + 256; }

TC_DEV int tc_find_job(const TcJob* jobs, int n_jobs, int64_t tile) {
  int lo = 0, hi = n_jobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile_begin <= tile) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

TC_DEV void tc_load_operand(const TcOperand& op, const CUtensorMap* maps, void* dst_hi, void* dst_lo, uint64_t* bar,
                            int k, int row) {
  const CUtensorMap* mh = maps + op.map_hi;
  const CUtensorMap* ml = maps + op.map_lo;
  if (op.dims == 3) {
    tc::tma_load_3d(dst_hi, mh, bar, op.x + k, op.y + row, op.z);
    tc::tma_load_3d(dst_lo, ml, bar, op.x + k, op.y + row, op.z);
  } else {
    tc::tma_load_2d(dst_hi, mh, bar, op.x + k, op.y + row);
    tc::tma_load_2d(dst_lo, ml, bar, op.x + k, op.y + row);
  }
}

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_3xtf32_kernel(const TcJob* __restrict__ jobs, int n_jobs, int64_t total_tiles,
                          const CUtensorMap* __restrict__ maps) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTcStages * kTcStageBytes);
  uint64_t* empty = full + kTcStages;
  uint64_t* tmem_full = empty + kTcStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(tmem_full + a, 1);
      tc::mbar_init(tmem_empty + a, 128);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kTcTmemCols>(tmem_base_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (tc::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int last_job = -1;
      for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int j = tc_find_job(jobs, n_jobs, tile);
        const TcJob& job = jobs[j];
        if (j != last_job) {
          tc::tma_acquire(maps + job.a.map_hi);
          tc::tma_acquire(maps + job.a.map_lo);
          tc::tma_acquire(maps + job.b.map_hi);
          tc::tma_acquire(maps + job.b.map_lo);
          last_job = j;
        }
        const int64_t local = tile - job.tile_begin;
        const int ti = (int)(local / job.tiles_n), tj = (int)(local % job.tiles_n);
        const int k_tiles = (job.K + kTcBK - 1) / kTcBK;
        for (int kt = 0; kt < k_tiles; ++kt) {
          tc::mbar_wait(empty + stage, phase ^ 1);
          uint8_t* st = smem + stage * kTcStageBytes;
          tc::mbar_arrive_expect_tx(full + stage, kTcStageBytes);
          tc_load_operand(job.a, maps, st, st + kTcTileBytes, full + stage, kt * kTcBK, ti * kTcBM);
          tc_load_operand(job.b, maps, st + 2 * kTcTileBytes, st + 2 * kTcTileBytes + kTcBTileBytes, full + stage,
                          kt * kTcBK, tj * kTcBN);
          if (++stage == kTcStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = tc::idesc_tf32(kTcBM, kTcBN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const TcJob& job = jobs[tc_find_job(jobs, n_jobs, tile)];
      const int k_tiles = (job.K + kTcBK - 1) / kTcBK;
      tc::mbar_wait(tmem_empty + acc, acc_phase ^ 1);
      tc::tc_fence_after();
      const uint32_t tmem_c = tmem_base + (uint32_t)(acc * kTcBN);
      for (int kt = 0; kt < k_tiles; ++kt) {
        tc::mbar_wait(full + stage, phase);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t s0 = tc::smem_u32(smem + stage * kTcStageBytes);
          const uint64_t a_hi = tc::umma_desc_sw128(s0), a_lo = tc::umma_desc_sw128(s0 + kTcTileBytes);
          const uint64_t b_hi = tc::umma_desc_sw128(s0 + 2 * kTcTileBytes);
          const uint64_t b_lo = tc::umma_desc_sw128(s0 + 2 * kTcTileBytes + kTcBTileBytes);
#pragma unroll
          for (int k = 0; k < kTcBK / 8; ++k) {
            const uint64_t adv = (uint64_t)((k * 8 * 4) >> 4);  // 32 bytes per K=8 step
            const uint32_t first = (kt == 0 && k == 0) ? 0u : 1u;
            tc::umma_tf32(tmem_c, a_lo + adv, b_hi + adv, idesc, first);
            tc::umma_tf32(tmem_c, a_hi + adv, b_lo + adv, idesc, 1u);
            tc::umma_tf32(tmem_c, a_hi + adv, b_hi + adv, idesc, 1u);
          }
          tc::umma_commit(empty + stage);  // smem slot free once these MMAs complete
        }
        __syncwarp();
        if (++stage == kTcStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (tc::elect_one()) tc::umma_commit(tmem_full + acc);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;  // TMEM lanes 32*quad .. 32*quad+31
    const int row_in_tile = quad * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const TcJob& job = jobs[tc_find_job(jobs, n_jobs, tile)];
      const int64_t local = tile - job.tile_begin;
      const int ti = (int)(local / job.tiles_n), tj = (int)(local % job.tiles_n);
      tc::mbar_wait(tmem_full + acc, acc_phase);
      tc::tc_fence_after();
      const int i = ti * kTcBM + row_in_tile;
      const bool row_ok = i < job.M;
#pragma unroll 1
      for (int c0 = 0; c0 < kTcBN; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * kTcBN + c0), r);
        tc::tmem_wait_ld();
        const int j0 = tj * kTcBN + c0;
        if (row_ok) {
          if (job.out_mode == 0) {
            float* o = job.out_hi + (int64_t)i * job.ld_out + j0;
            if (j0 + 16 <= job.N && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
              // 16-byte stores: lanes hold different rows, so this quarters the
              // number of scattered store transactions
#pragma unroll
              for (int q = 0; q < 4; ++q)
                reinterpret_cast<float4*>(o)[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                              __uint_as_float(r[4 * q + 2]),
                                                              __uint_as_float(r[4 * q + 3]));
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (j0 + e < job.N) o[e] = __uint_as_float(r[e]);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (j0 + e < job.N) {
                const float v = __uint_as_float(r[e]);
                job.out_hi[(int64_t)(j0 + e) * job.ld_out + i] = v;
                job.out_lo[(int64_t)(j0 + e) * job.ld_out + i] = tc::tf32_lo(v);
              }
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(tmem_empty + acc);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<kTcTmemCols>(tmem_base);
  }
}

// -------------------------------------------------------------- split kernel
// lo = x - trunc_tf32(x) over flat segments, float4 vectorised, 4 loads in flight.
__global__ void __launch_bounds__(256) tf32_split_kernel(const SplitSeg* __restrict__ segs, int n_segs) {
  const SplitSeg s = segs[blockIdx.y];
  const float4* src = reinterpret_cast<const float4*>(s.src);
  float4* lo = reinterpret_cast<float4*>(s.lo);
  const int64_t n4 = s.n >> 2, step = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * step < n4; i += 4 * step) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(src + i + u * step);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      lo[i + u * step] = make_float4(tc::tf32_lo(v[u].x), tc::tf32_lo(v[u].y), tc::tf32_lo(v[u].z), tc::tf32_lo(v[u].w));
  }
  for (; i < n4; i += step) {
    const float4 v = __ldg(src + i);
    lo[i] = make_float4(tc::tf32_lo(v.x), tc::tf32_lo(v.y), tc::tf32_lo(v.z), tc::tf32_lo(v.w));
  }
}

// one flat range (the caller-facing shampoo_tf32_split): no table, arguments by value
__global__ void __launch_bounds__(256) tf32_split_flat_kernel(const float* __restrict__ x, float* __restrict__ lo,
                                                              int64_t n) {
  const float4* src = reinterpret_cast<const float4*>(x);
  float4* dst = reinterpret_cast<float4*>(lo);
  const int64_t n4 = n >> 2, step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += step) {
    const float4 v = __ldg(src + i);
    dst[i] = make_float4(tc::tf32_lo(v.x), tc::tf32_lo(v.y), tc::tf32_lo(v.z), tc::tf32_lo(v.w));
  }
}

int split_flat_launch(const float* x, float* lo, int64_t n, cudaStream_t stream, int64_t* launches) {
  if (n == 0) return SHAMPOO_OK;
  tf32_split_flat_kernel<<<8 * num_sms(), 256, 0, stream>>>(x, lo, n);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("tf32_split_flat_kernel", e);
  return SHAMPOO_OK;
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_map_f32(CUtensorMap* out, const void* base, int dims, const uint64_t* size, const uint64_t* stride_bytes,
                 int box_rows) {
  auto enc = get_encode();
  if (!enc) return set_error(SHAMPOO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[3] = {size[0], size[1], dims == 3 ? size[2] : 1};
  cuuint64_t gstride[2] = {stride_bytes[0], dims == 3 ? stride_bytes[1] : 0};
  cuuint32_t box[3] = {(cuuint32_t)kTcBK, (cuuint32_t)box_rows, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)dims, const_cast<void*>(base), gdim, gstride, box,
                   estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SHAMPOO_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SHAMPOO_OK;
}

int tc_gemm_launch(const TcJob* jobs_dev, int n_jobs, int64_t total_tiles, const CUtensorMap* maps_dev,
                   cudaStream_t stream, int64_t* launches) {
  if (total_tiles == 0) return SHAMPOO_OK;
  const size_t smem = tc_gemm_smem_bytes();
  if (ensure_smem((const void*)tc_gemm_3xtf32_kernel, smem) !=
      cudaSuccess)
    return set_cuda_error("cudaFuncSetAttribute(tc_gemm_3xtf32_kernel)");
  const int64_t g = total_tiles < num_sms() ? total_tiles : num_sms();
  tc_gemm_3xtf32_kernel<<<(unsigned)g, kTcThreads, smem, stream>>>(jobs_dev, n_jobs, total_tiles, maps_dev);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("tc_gemm_3xtf32_kernel", e);
  return SHAMPOO_OK;
}

int tf32_split_launch(const SplitSeg* segs_dev, int n_segs, cudaStream_t stream, int64_t* launches) {
  if (n_segs == 0) return SHAMPOO_OK;
  tf32_split_kernel<<<dim3(2 * num_sms(), n_segs), 256, 0, stream>>>(segs_dev, n_segs);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("tf32_split_kernel", e);
  return SHAMPOO_OK;
}

}  // namespace shp
