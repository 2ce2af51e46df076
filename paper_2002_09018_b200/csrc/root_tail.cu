// root_tail.cu -- the 3xTF32 tail of the hybrid coupled-Newton root (rows a5-a6,
// DESIGN.md §6.3b; north star: "3xTF32 error-compensated splits or FP64 DMMA").
//
// root_kernel runs the first k_sw iterations in fp64 on the DMMA pipe and hands
// every still-iterating matrix over as fp32 pairs (hi, lo = hi - trunc_tf32(hi))
// of X_k, M_k, T_k.  Here the remaining iterations run on the tcgen05 tensor
// cores, one persistent kernel per product stage:
//   P1  X_{k+1} = X_k T , S0 = T T          (dual stage; p = 1: X T only)
//   ..  the rest of the left-to-right binary chain for T^p (S0/S1 ping-pong)
//   P3  M_{k+1} = T^p M_k ; epilogue: T_{k+1} = ((p+1)I - M_{k+1})/p and
//       max|M_{k+1} - I| (warp max + one 64-bit atomicMax per warp)
//   decide: the stopping rule of reading #20 with tol_tail = max(tol, 1e-5)
//           (the fp32 tail's noise floor of max|M - I|), ordered compaction.
// All iterates are symmetric polynomials of A_hat: only the upper 128x128 tiles
// are computed and each is stored twice (row-major and mirrored).
// Each product: 3 tcgen05.mma.kind::tf32 passes (lo.hi + hi.lo + hi.hi) into
// one fp32 TMEM accumulator, TMA (SWIZZLE_128B, 3-D maps over the batch) into a
// 3-stage ring, warp-specialised like tc_gemm.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "ozaki.cuh"

#include <cmath>
#include "tc_common.cuh"
#include "tc_gemm.h"

namespace shp {

constexpr int kRBM = 128, kRBK = 32;
constexpr int kRStages = 3;
constexpr int kRTileBytes = kRBM * kRBK * 4;  // 16 KB
constexpr int kRStageBytes = 4 * kRTileBytes;
constexpr int kRThreads = 192;
constexpr uint32_t kRTmemCols = 2 * kRBM;
constexpr double kTailTol = 1e-5;
constexpr int kTailRegions = 7;  // fp64 buffer regions per matrix (root.cu kBufs)
constexpr int kTailMaxBatch = 2048;

// tail pair q -> fp64 region of root.cu (X0, X1, M0, M1, T, S0, S1 = 0..6),
// given xs = k_sw & 1 (see tail_handoff)
enum { TX0 = 0, TX1 = 1, TM0 = 2, TM1 = 3, TT = 4, TS0 = 5, TS1 = 6 };
static int tail_region(int q, int xs) {
  switch (q) {
    case TX0: return 0 + (xs ^ 1);
    case TX1: return 0 + xs;
    case TM0: return 2 + (xs ^ 1);
    case TM1: return 2 + xs;
    case TT: return 6;  // BS1
    case TS0: return 4;  // BT
    default: return 5;  // BS0
  }
}

struct TailStage {
  int jobs;           // 1 or 2
  int a[2], b[2], d[2];  // fp64 regions of A, B and the output per job
  int mupdate;        // 1: M-update epilogue for job 0 (T -> region t_reg, err -> errh[kcheck])
  int t_reg;
  int kcheck;
};

struct TailArgs {
  double* bufs;
  const int* act;
  const int* nact;
  int n, np, p, tiles_n;
  double* errh;
  int max_iter;
  TailStage st;
};

TC_DEV float* region_f(const TailArgs& a, int mat, int reg) {
  return reinterpret_cast<float*>(a.bufs + ((int64_t)mat * kTailRegions + reg) * (int64_t)a.np * a.np);
}

// k-tile order of a tile: every k-tile outside the 128-row blocks ti and tj
// first, then block ti, then block tj.  The near-identity factors have their
// O(1) entries in those blocks, so the accumulator stays small until the last
// k-tiles and the tensor core's fp32 accumulation (biased: measured ~1e-5 on
// near-identity products in natural order) rounds far fewer O(1) partial sums.
TC_DEV int tail_ktile(int l, int k_tiles, int ti, int tj) {
  const int per = kRBM / kRBK;  // k-tiles per 128-row block
  const int bi0 = ti * per, bj0 = tj * per;
  const int ni = min(per, k_tiles - bi0);
  const int nj = (tj == ti) ? 0 : min(per, k_tiles - bj0);
  const int rest = k_tiles - ni - nj;
  if (l < rest) {  // l-th k-tile outside both blocks, ascending
    int k = l;
    const int lo = min(bi0, ti == tj ? bi0 : bj0), hi = max(bi0, ti == tj ? bi0 : bj0);
    const int nlo = lo == bi0 ? ni : nj, nhi = hi == bi0 ? ni : nj;
    if (k >= lo) k += nlo;
    if (ti != tj && k >= hi) k += nhi;
    return k;
  }
  l -= rest;
  return l < ni ? bi0 + l : bj0 + (l - ni);
}

TC_DEV void tail_decode(const TailArgs& a, int64_t tile, int& mat, int& ti, int& tj, int& job) {
  const int tiles = a.tiles_n * (a.tiles_n + 1) / 2;
  const int64_t per = (int64_t)tiles * a.st.jobs;
  const int pos = (int)(tile / per);
  int rem = (int)(tile - (int64_t)pos * per);
  job = rem % a.st.jobs;
  int t = rem / a.st.jobs;
  int i = 0;
  while (t >= a.tiles_n - i) {
    t -= a.tiles_n - i;
    ++i;
  }
  ti = i;
  tj = i + t;
  mat = a.act[pos];
}

__global__ void __launch_bounds__(kRThreads, 1)
    root_tail_gemm_kernel(const __grid_constant__ TailArgs a, const CUtensorMap* __restrict__ maps) {
  const int nact = *a.nact;
  if (nact == 0) return;
  const int64_t total = (int64_t)nact * (a.tiles_n * (a.tiles_n + 1) / 2) * a.st.jobs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRStages * kRStageBytes);
  uint64_t* empty = full + kRStages;
  uint64_t* tmem_full = empty + kRStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kRStages; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    for (int q = 0; q < 2; ++q) {
      tc::mbar_init(tmem_full + q, 1);
      tc::mbar_init(tmem_empty + q, 128);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kRTmemCols>(tmem_base_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  const int k_tiles = (a.n + kRBK - 1) / kRBK;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (tc::elect_one()) {
      for (int q = 0; q < kTailRegions * 2; ++q) tc::tma_acquire(maps + q);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        int mat, ti, tj, job;
        tail_decode(a, tile, mat, ti, tj, job);
        const CUtensorMap* ah = maps + 2 * a.st.a[job];
        const CUtensorMap* bh = maps + 2 * a.st.b[job];
        for (int kt = 0; kt < k_tiles; ++kt) {
          tc::mbar_wait(empty + stage, phase ^ 1);
          uint8_t* st = smem + stage * kRStageBytes;
          tc::mbar_arrive_expect_tx(full + stage, kRStageBytes);
          const int kk = tail_ktile(kt, k_tiles, ti, tj) * kRBK;
          tc::tma_load_3d(st, ah, full + stage, kk, ti * kRBM, mat);
          tc::tma_load_3d(st + kRTileBytes, ah + 1, full + stage, kk, ti * kRBM, mat);
          tc::tma_load_3d(st + 2 * kRTileBytes, bh, full + stage, kk, tj * kRBM, mat);
          tc::tma_load_3d(st + 3 * kRTileBytes, bh + 1, full + stage, kk, tj * kRBM, mat);
          if (++stage == kRStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = tc::idesc_tf32(kRBM, kRBM);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      tc::mbar_wait(tmem_empty + acc, acc_phase ^ 1);
      tc::tc_fence_after();
      const uint32_t tmem_c = tmem_base + (uint32_t)(acc * kRBM);
      for (int kt = 0; kt < k_tiles; ++kt) {
        tc::mbar_wait(full + stage, phase);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t s0 = tc::smem_u32(smem + stage * kRStageBytes);
          const uint64_t a_hi = tc::umma_desc_sw128(s0), a_lo = tc::umma_desc_sw128(s0 + kRTileBytes);
          const uint64_t b_hi = tc::umma_desc_sw128(s0 + 2 * kRTileBytes);
          const uint64_t b_lo = tc::umma_desc_sw128(s0 + 3 * kRTileBytes);
#pragma unroll
          for (int k = 0; k < kRBK / 8; ++k) {
            const uint64_t adv = (uint64_t)((k * 8 * 4) >> 4);
            const uint32_t first = (kt == 0 && k == 0) ? 0u : 1u;
            tc::umma_tf32(tmem_c, a_lo + adv, b_hi + adv, idesc, first);
            tc::umma_tf32(tmem_c, a_hi + adv, b_lo + adv, idesc, 1u);
            tc::umma_tf32(tmem_c, a_hi + adv, b_hi + adv, idesc, 1u);
          }
          tc::umma_commit(empty + stage);
        }
        __syncwarp();
        if (++stage == kRStages) {
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
    const int quad = warp & 3;
    const int row_in_tile = quad * 32 + lane;
    const int64_t half = (int64_t)a.np * a.np;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      int mat, ti, tj, job;
      tail_decode(a, tile, mat, ti, tj, job);
      tc::mbar_wait(tmem_full + acc, acc_phase);
      tc::tc_fence_after();
      const int i = ti * kRBM + row_in_tile;
      const bool row_ok = i < a.n, mirror = ti != tj;
      const bool mup = a.st.mupdate && job == 0;
      float* D = region_f(a, mat, a.st.d[job]);
      float* Tn = mup ? region_f(a, mat, a.st.t_reg) : nullptr;
      double emax = 0.0;
#pragma unroll 1
      for (int c0 = 0; c0 < kRBM; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * kRBM + c0), r);
        tc::tmem_wait_ld();
        const int j0 = tj * kRBM + c0;
        if (!row_ok) continue;
        float v[16], lo[16], t[16], tlo[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int j = j0 + e;
          v[e] = __uint_as_float(r[e]);
          lo[e] = tc::tf32_lo(v[e]);
          if (mup) {
            const double dlt = (i == j) ? 1.0 : 0.0;
            t[e] = (float)(((double)(a.p + 1) * dlt - (double)v[e]) / (double)a.p);
            tlo[e] = tc::tf32_lo(t[e]);
            if (j < a.n) emax = fmax_nan(emax, fabs((double)v[e] - dlt));
          }
        }
        // row-major part: 16-byte vector stores (4 per lane per array) when the
        // 16 columns are in range; the mirrored part: lanes = consecutive rows,
        // one coalesced 128-byte store per column
        float* drow = D + (int64_t)i * a.np + j0;
        float* trow = mup ? Tn + (int64_t)i * a.np + j0 : nullptr;
        if (j0 + 16 <= a.n) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            reinterpret_cast<float4*>(drow)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            reinterpret_cast<float4*>(drow + half)[q] =
                make_float4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
            if (mup) {
              reinterpret_cast<float4*>(trow)[q] = make_float4(t[4 * q], t[4 * q + 1], t[4 * q + 2], t[4 * q + 3]);
              reinterpret_cast<float4*>(trow + half)[q] =
                  make_float4(tlo[4 * q], tlo[4 * q + 1], tlo[4 * q + 2], tlo[4 * q + 3]);
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (j0 + e < a.n) {
              drow[e] = v[e];
              drow[half + e] = lo[e];
              if (mup) {
                trow[e] = t[e];
                trow[half + e] = tlo[e];
              }
            }
        }
        if (mirror) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int j = j0 + e;
            if (j >= a.n) continue;
            D[(int64_t)j * a.np + i] = v[e];
            D[half + (int64_t)j * a.np + i] = lo[e];
            if (mup) {
              Tn[(int64_t)j * a.np + i] = t[e];
              Tn[half + (int64_t)j * a.np + i] = tlo[e];
            }
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(tmem_empty + acc);
      if (mup) {
        emax = warp_max(emax);
        if (lane == 0) atomic_max_nonneg(a.errh + (int64_t)mat * (a.max_iter + 1) + a.st.kcheck, emax);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<kRTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------- decide / compact
// One CTA: the stopping rule (reading #20) at check k for every active matrix;
// the active list shrinks in order.  d[mat] records the decision check.
enum { TD_CONTINUE = 0, TD_CONVERGED = 1, TD_STAGNATED = 2, TD_MAXITER = 3, TD_NONFINITE = 4 };

TC_DEV int tail_decide(const double* errh, int max_iter, double tol, double stag, int mat, int k) {
  const double* e = errh + (int64_t)mat * (max_iter + 1);
  const double ek = e[k];
  if (!isfinite(ek)) return TD_NONFINITE;
  if (ek <= tol) return TD_CONVERGED;
  const double ep = e[k - 1];
  // reading #20, tail variant: fp32 iterates reach a noise floor where err may
  // keep creeping down; no quadratic progress (err_k >= 0.5 err_{k-1}) below
  // 1e-2 counts as stagnation
  if (ek >= stag * ep && ep < 1e-2) return TD_STAGNATED;
  if (k == max_iter) return TD_MAXITER;
  return TD_CONTINUE;
}

// Ordered compaction of the active list after check k (one CTA of 1024 threads); returns the new count.
__device__ int tail_decide_block(int* act, int* nact, const double* errh, int max_iter, double tol, double stag,
                                 int k) {
  __shared__ int cnt[1025];
  __shared__ int s_act[kTailMaxBatch];
  const int n = *nact;
  for (int q = threadIdx.x; q < n; q += 1024) s_act[q] = act[q];
  __syncthreads();
  const int per = (n + 1023) / 1024, b0 = threadIdx.x * per;
  int mine[kTailMaxBatch / 1024];
  int nm = 0;
  for (int q = 0; q < per; ++q)
    if (b0 + q < n) {
      const int mat = s_act[b0 + q];
      if (tail_decide(errh, max_iter, tol, stag, mat, k) == TD_CONTINUE) mine[nm++] = mat;
    }
  cnt[threadIdx.x] = nm;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < 1024; ++i) {
      const int c = cnt[i];
      cnt[i] = acc;
      acc += c;
    }
    cnt[1024] = acc;
  }
  __syncthreads();
  for (int q = 0; q < nm; ++q) act[cnt[threadIdx.x] + q] = mine[q];
  if (threadIdx.x == 0) *nact = cnt[1024];
  return cnt[1024];
}

__global__ void __launch_bounds__(1024) root_tail_decide_kernel(int* act, int* nact, const double* errh, int max_iter,
                                                                double tol, double stag, int k) {
  tail_decide_block(act, nact, errh, max_iter, tol, stag, k);
}

// The convergence-driven tail (CUDA graph with a conditional WHILE node): the iteration index lives in *kdev
// (the products of iteration *kdev wrote err_{*kdev + 1}); after the decision *kdev advances, and the last decide
// of the loop body sets the loop condition: another body only while matrices remain active.
__global__ void __launch_bounds__(1024) root_tail_decide_graph_kernel(int* act, int* nact, const double* errh,
                                                                      int max_iter, double tol, double stag,
                                                                      int* kdev, cudaGraphConditionalHandle h,
                                                                      int set_cond) {
  const int k = *kdev + 1;
  __syncthreads();  // every thread has read *kdev before thread 0 advances it
  const int left = tail_decide_block(act, nact, errh, max_iter, tol, stag, k);
  if (threadIdx.x == 0) {
    *kdev = k;
    if (set_cond) cudaGraphSetConditional(h, (left > 0 && k < max_iter) ? 1u : 0u);
  }
}

// Final decisions of the handed-off matrices (res.x == -3) and the fp32 output:
// X_k lives in pair TX[(k - k_sw) & 1]; the stored hi IS the fp32 iterate.
__global__ void __launch_bounds__(256) root_tail_finish_kernel(double* bufs, const int4* res, const double* errh,
                                                               shampoo_root_info_t* info, float* X, int64_t ldx,
                                                               int64_t stride_x, int batch, int n, int np,
                                                               int max_iter, int k_sw, double tol, double stag,
                                                               int reg_x0, int reg_x1, int fp64) {
  const int mat = blockIdx.x;
  if (mat >= batch || res[mat].x != -3) return;
  __shared__ int s_buf;
  if (threadIdx.x == 0) {
    int k = k_sw + 1, d = TD_CONTINUE;
    for (; k <= max_iter; ++k) {
      d = tail_decide(errh, max_iter, tol, stag, mat, k);
      if (d != TD_CONTINUE) break;
    }
    if (k > max_iter) k = max_iter;  // k_sw == max_iter: decided at the handoff check
    const double* e = errh + (int64_t)mat * (max_iter + 1);
    int status, iters, kx;
    double err;
    if (d == TD_CONVERGED) { status = 0; iters = k; kx = k; err = e[k]; }
    else if (d == TD_STAGNATED) { status = 1; iters = k - 1; kx = k - 1; err = e[k - 1]; }
    else if (d == TD_MAXITER) { status = 1; iters = k; kx = k; err = e[k]; }
    else { status = 2; iters = k; kx = -1; err = e[k]; }
    info[mat].iters = iters;
    info[mat].status = status;
    info[mat].err = err;
    s_buf = kx < 0 ? -1 : (((kx - k_sw) & 1) ? reg_x1 : reg_x0);
  }
  __syncthreads();
  if (s_buf < 0) return;
  const double* src64 = bufs + ((int64_t)mat * kTailRegions + s_buf) * (int64_t)np * np;
  const float* src = reinterpret_cast<const float*>(src64);
  float* out = X + (int64_t)mat * stride_x;
  // one warp per row; fp64 rows of 4 elements per lane (32-byte loads, 16-byte stores) when the output rows are
  // 16-byte aligned (round 2: one element per thread of a 128-thread CTA ran at ~1.3 TB/s)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const bool vec = fp64 && (ldx & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (int i = warp; i < n; i += nwarps) {
    const double* r64 = src64 + (int64_t)i * np;
    float* o = out + (int64_t)i * ldx;
    if (vec) {
      int j = 4 * lane;
      for (; j + 4 <= n; j += 128) {
        const double4 d = *reinterpret_cast<const double4*>(r64 + j);
        *reinterpret_cast<float4*>(o + j) =
            make_float4(__double2float_rn(d.x), __double2float_rn(d.y), __double2float_rn(d.z), __double2float_rn(d.w));
      }
      for (int jj = j; jj < n && jj < j + 4; ++jj) o[jj] = __double2float_rn(r64[jj]);  // the row tail
    } else {
      for (int j = lane; j < n; j += 32) o[j] = fp64 ? __double2float_rn(r64[j]) : src[(int64_t)i * np + j];
    }
  }
}

// ------------------------------------------------------------------ host side
size_t root_tail_smem_bytes() { return 1024 + (size_t)kRStages * kRStageBytes + 256; }

size_t root_tail_ws_bytes(int batch) {
  return ((size_t)2 * kTailRegions * sizeof(CUtensorMap) + 255) / 256 * 256 + ((size_t)(batch + 64) * 4 + 255) / 256 * 256;
}

int root_tail_launch(double* bufs, int batch, int n, int np, int p, int max_iter, int k_sw, double tol, double* errh,
                     const int4* res, shampoo_root_info_t* info, float* X, int64_t ldx, int64_t stride_x, int* act,
                     int* nact, void* maps_ws, cudaStream_t stream, int64_t* launches) {
  const size_t smem = root_tail_smem_bytes();
  if (ensure_smem((const void*)root_tail_gemm_kernel, smem) !=
      cudaSuccess)
    return set_cuda_error("cudaFuncSetAttribute(root_tail_gemm_kernel)");
  if (batch > kTailMaxBatch) return set_error(SHAMPOO_ERR_UNSUPPORTED, "hybrid root: batch chunk > %d", kTailMaxBatch);
  // 3-D TMA maps (hi, lo) of every region over the batch: (n cols, n rows, batch), OOB -> 0
  CUtensorMap maps[2 * kTailRegions];
  for (int r = 0; r < kTailRegions; ++r)
    for (int h = 0; h < 2; ++h) {
      const float* base = reinterpret_cast<const float*>(bufs + (int64_t)r * np * np) + (int64_t)h * np * np;
      uint64_t size[3] = {(uint64_t)n, (uint64_t)n, (uint64_t)batch};
      uint64_t st[2] = {(uint64_t)np * 4, (uint64_t)kTailRegions * np * np * 8};
      int rc = make_map_f32(&maps[2 * r + h], base, 3, size, st, kRBM);
      if (rc) return rc;
    }
  if (cudaMemcpyAsync(maps_ws, maps, sizeof maps, cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return set_cuda_error("cudaMemcpyAsync(tail maps)");
  const CUtensorMap* maps_dev = static_cast<const CUtensorMap*>(maps_ws);
  const double ttol = tol > kTailTol ? tol : kTailTol;
  TailArgs a;
  std::memset(&a, 0, sizeof a);
  a.bufs = bufs;
  a.act = act;
  a.nact = nact;
  a.n = n;
  a.np = np;
  a.p = p;
  a.tiles_n = (n + kRBM - 1) / kRBM;
  a.errh = errh;
  a.max_iter = max_iter;
  auto R = [&](int q) { return tail_region(q, k_sw & 1); };
  const int grid = num_sms();
  auto run = [&](const TailStage& st) -> int {
    a.st = st;
    root_tail_gemm_kernel<<<grid, kRThreads, smem, stream>>>(a, maps_dev);
    ++*launches;
    return SHAMPOO_OK;
  };
  const int lead = 31 - __builtin_clz((unsigned)p);
  int tcur = TT;  // pair holding T_k (p = 1 alternates TT / TS1: T_k is an operand of its own M-update)
  for (int k = k_sw; k < max_iter; ++k) {
    const int t = k - k_sw;
    const int xc = (t & 1) ? TX1 : TX0, xn = (t & 1) ? TX0 : TX1;
    const int mc = (t & 1) ? TM1 : TM0, mn = (t & 1) ? TM0 : TM1;
    // P1: X_{k+1} = X_k T ; S0 = T T (p >= 2)
    TailStage s1;
    std::memset(&s1, 0, sizeof s1);
    s1.jobs = p >= 2 ? 2 : 1;
    s1.a[0] = R(xc); s1.b[0] = R(tcur); s1.d[0] = R(xn);
    s1.a[1] = R(tcur); s1.b[1] = R(tcur); s1.d[1] = R(TS0);
    run(s1);
    // rest of the binary chain for T^p (S0 = T^2)
    int rb = TS0;
    for (int bit = lead - 1; bit >= 0; --bit) {
      if (bit != lead - 1) {
        TailStage q;
        std::memset(&q, 0, sizeof q);
        const int d = rb == TS0 ? TS1 : TS0;
        q.jobs = 1; q.a[0] = R(rb); q.b[0] = R(rb); q.d[0] = R(d);
        run(q);
        rb = d;
      }
      if ((p >> bit) & 1) {
        TailStage q;
        std::memset(&q, 0, sizeof q);
        const int d = rb == TS0 ? TS1 : TS0;
        q.jobs = 1; q.a[0] = R(rb); q.b[0] = R(tcur); q.d[0] = R(d);
        run(q);
        rb = d;
      }
    }
    // P3: M_{k+1} = T^p M_k ; T_{k+1} ; err_{k+1}
    const int tnext = (p == 1) ? (tcur == TT ? TS1 : TT) : TT;  // p >= 2: T_k is dead after the chain
    TailStage s3;
    std::memset(&s3, 0, sizeof s3);
    s3.jobs = 1;
    s3.a[0] = R(p == 1 ? tcur : rb); s3.b[0] = R(mc); s3.d[0] = R(mn);
    s3.mupdate = 1;
    s3.t_reg = R(tnext);
    s3.kcheck = k + 1;
    run(s3);
    tcur = tnext;
    root_tail_decide_kernel<<<1, 1024, 0, stream>>>(act, nact, errh, max_iter, ttol, 0.5, k + 1);
    ++*launches;
  }
  root_tail_finish_kernel<<<batch, 256, 0, stream>>>(bufs, res, errh, info, X, ldx, stride_x, batch, n, np, max_iter,
                                                     k_sw, ttol, 0.5, R(TX0), R(TX1), 0);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("root tail kernels", e);
  return SHAMPOO_OK;
}

// ======================================================= Ozaki (INT8) root
// All coupled-Newton iterations on the INT8 tensor cores (ozaki.cuh): fp64
// iterates in root.cu's regions, every operand sliced into S int8 planes right
// before its product (S = 6 or 7).  Slots (planes + row scales) for X_k, T, S0, S1, M_k.
enum { OZ_SX = 0, OZ_ST = 1, OZ_SS0 = 2, OZ_SS1 = 3, OZ_SM = 4, OZ_SLOTS = 5 };

size_t root_ozaki_ws_bytes(int batch, int n) {
  const int np = (n + 63) / 64 * 64;
  const size_t planes = (size_t)OZ_SLOTS * batch * oz::kSMax * oz::plane_pitch(np);
  const size_t scales = (size_t)OZ_SLOTS * batch * np * sizeof(double);
  return ((planes + 255) / 256 * 256) + ((scales + 255) / 256 * 256) + 256;
}

// Iterations enqueued one launch at a time before the convergence-driven tail graph takes over: the scalar
// recurrence m <- m ((p+1-m)/p)^p of the smallest eigenvalue of M from m_0 = eps_rel/(1+eps_rel) until |1 - m| <=
// tol (the iteration count of the worst-conditioned matrix the ridge allows), + 2; then up to where the slice
// schedule has settled (the tail graph runs one slice count) and even (its two-iteration body keeps the X / M
// ping-pong parity static).  No ridge: everything direct.
static int ozaki_direct_iterations(int p, int n, double eps_rel, double tol, int max_iter, double budget,
                                   int s_max) {
  if (!(eps_rel > 0.0)) return max_iter;
  double m = eps_rel / (1.0 + eps_rel);
  int k = 0;
  while (k < max_iter && std::fabs(1.0 - m) > tol) {
    m = m * std::pow(((double)(p + 1) - m) / (double)p, (double)p);
    ++k;
  }
  k += 2;
  const int s_floor = ozaki_iteration_slices(1000, p, n, eps_rel, budget, s_max);
  while (k < max_iter && ozaki_iteration_slices(k, p, n, eps_rel, budget, s_max) != s_floor) ++k;
  if (k & 1) ++k;
  return std::min(k, max_iter);
}

// Slice count of iteration k (reading #29): an error made in M_k reaches the
// root amplified by ~1/(p lambda_min(M_k)), lambda_min(M_0) >= eps_rel / (1 +
// eps_rel) (the ridge) and the scalar recurrence grows it by g = ((p+1)/p)^p per
// iteration while it is small -- so m_k = min(1, eps_rel g^k) bounds it a priori
// and S_k = the smallest S in [kOzSMin, s_max] with 2^-(7S-1) sqrt(n/1024) / (p m_k) <= budget
// (a product's rounding errors add up over its n-term sums like a random walk).
// budget <= 0 (or no ridge): S_k = s_max for every k (the fixed-slice root).
constexpr int kOzSMin = 5;  // S = 4 (2^-27) was measured (host emulation) to leave a 4e-6 floor in the root
constexpr int kOzSX = 5;    // the X-update X_k T_k: X only accumulates T's (no amplification)
int ozaki_iteration_slices(int k, int p, int n, double eps_rel, double budget, int s_max) {
  if (!(budget > 0.0) || !(eps_rel > 0.0)) return s_max;
  const double g = std::pow((double)(p + 1) / (double)p, (double)p);
  const double m = std::min(1.0, eps_rel * std::pow(g, (double)k));
  const double growth = std::sqrt((double)n / 1024.0);
  for (int S = kOzSMin; S < s_max; ++S)
    if (std::ldexp(1.0, -(7 * S - 1)) * growth / ((double)p * m) <= budget) return S;
  return s_max;
}

template <int S>
static cudaError_t oz_gemm_s(const oz::OzArgs& a, cudaStream_t stream) {
  const size_t smem = oz::gemm_smem_bytes<S, 64>();
  cudaError_t e = ensure_smem((const void*)oz::gemm_kernel<S, 64>, smem);
  if (e != cudaSuccess) return e;
  oz::gemm_kernel<S, 64><<<num_sms(), oz::kThreads, smem, stream>>>(a);
  return cudaSuccess;
}

static cudaError_t oz_gemm(int S, const oz::OzArgs& a, cudaStream_t stream) {
  switch (S) {
    case 5: return oz_gemm_s<5>(a, stream);
    case 6: return oz_gemm_s<6>(a, stream);
    default: return oz_gemm_s<7>(a, stream);
  }
}

// M_k and T_k (n <= 1024): the row-pair slicer (whole-line stores: 2.47 vs 3.42 ms for the one-row-per-warp slicer at
// S = 7, 528 matrices); X_k and the rest: slice_kernel (one register-resident row per warp, 16 warps per SM: its
// write share is half the M/T slicer's, and the pair slicer's 12 warps per SM lose there -- 1.51 vs 1.11 ms, r02zf)
template <int S, int MODE>
static void oz_slice_pair(const double* src, int64_t mstride, int n, int np, int batch, const int* act,
                          const int* nact, int8_t* pa, double* sa, int8_t* pt, double* st, int p, cudaStream_t stream) {
  ensure_smem((const void*)oz::slice_pair_kernel<S, MODE>, oz::kPairSmem);
  oz::slice_pair_kernel<S, MODE><<<3 * num_sms(), 32 * oz::kPairWarps, oz::kPairSmem, stream>>>(
      src, mstride, n, np, batch, act, nact, pa, sa, pt, st, p);
}

template <int S>
static void oz_slice_s(bool tm, const double* src, int64_t mstride, int n, int np, int batch, const int* act,
                       const int* nact, int8_t* planes, double* scale, int p, cudaStream_t stream) {
  const int grid = 8 * num_sms();
  if (tm)
    oz::slice_kernel<S, true><<<grid, 256, 0, stream>>>(src, mstride, n, np, batch, act, nact, planes, scale, p);
  else
    oz::slice_kernel<S, false><<<grid, 256, 0, stream>>>(src, mstride, n, np, batch, act, nact, planes, scale, p);
}

static void oz_slice(int S, bool tm, const double* src, int64_t mstride, int n, int np, int batch, const int* act,
                     const int* nact, int8_t* planes, double* scale, int p, cudaStream_t stream) {
  switch (S) {
    case 5: oz_slice_s<5>(tm, src, mstride, n, np, batch, act, nact, planes, scale, p, stream); break;
    case 6: oz_slice_s<6>(tm, src, mstride, n, np, batch, act, nact, planes, scale, p, stream); break;
    default: oz_slice_s<7>(tm, src, mstride, n, np, batch, act, nact, planes, scale, p, stream); break;
  }
}

// M_k and T_k in one pass over M_k (n <= 1024)
static void oz_slice_mt(int S, const double* src, int64_t mstride, int n, int np, int batch, const int* act,
                        const int* nact, int8_t* pm, double* sm, int8_t* pt, double* st, int p, cudaStream_t stream) {
  switch (S) {
    case 5: oz_slice_pair<5, 2>(src, mstride, n, np, batch, act, nact, pm, sm, pt, st, p, stream); break;
    case 6: oz_slice_pair<6, 2>(src, mstride, n, np, batch, act, nact, pm, sm, pt, st, p, stream); break;
    default: oz_slice_pair<7, 2>(src, mstride, n, np, batch, act, nact, pm, sm, pt, st, p, stream); break;
  }
}

// A non-blocking stream per (host thread, device) to capture the tail graph's body into (never destroyed): root
// calls from different host threads capture independently.
static cudaStream_t capture_stream() {
  thread_local cudaStream_t streams[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!streams[dev]) cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
  return streams[dev];
}

// Builds, launches on `stream` and releases a graph of one conditional WHILE node whose body is captured from
// body(capture_stream, handle); the handle is set on the device (root_tail_decide_graph_kernel).  The executable
// graph is destroyed right after its launch (freed when the launch completes).
template <class Body>
static int ozaki_tail_graph(cudaStream_t stream, Body body) {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return set_cuda_error("cudaGraphCreate");
  cudaGraphConditionalHandle h;
  cudaGraphNodeParams prm = {};
  prm.type = cudaGraphNodeTypeConditional;
  cudaGraphNode_t node;
  int rc = SHAMPOO_OK;
  if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) {
    rc = set_cuda_error("cudaGraphConditionalHandleCreate");
  } else {
    prm.conditional.handle = h;
    prm.conditional.type = cudaGraphCondTypeWhile;
    prm.conditional.size = 1;
    if (cudaGraphAddNode(&node, g, nullptr, 0, &prm) != cudaSuccess) rc = set_cuda_error("cudaGraphAddNode(while)");
  }
  if (rc == SHAMPOO_OK) {
    cudaGraph_t bodyg = prm.conditional.phGraph_out[0];
    cudaStream_t cs = capture_stream();
    if (cudaStreamBeginCaptureToGraph(cs, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      rc = set_cuda_error("cudaStreamBeginCaptureToGraph");
    } else {
      rc = body(cs, h);
      cudaGraph_t captured = nullptr;
      cudaError_t e = cudaStreamEndCapture(cs, &captured);
      if (rc == SHAMPOO_OK && e != cudaSuccess) rc = set_cuda_error("cudaStreamEndCapture", e);
    }
  }
  if (rc == SHAMPOO_OK && cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) rc = set_cuda_error("cudaGraphInstantiate");
  if (rc == SHAMPOO_OK && cudaGraphLaunch(ex, stream) != cudaSuccess) rc = set_cuda_error("cudaGraphLaunch");
  if (ex) cudaGraphExecDestroy(ex);
  cudaGraphDestroy(g);
  return rc;
}

int root_ozaki_launch(double* bufs, int batch, int n, int np, int p, int max_iter, double tol, double* errh,
                      const int4* res, shampoo_root_info_t* info, float* X, int64_t ldx, int64_t stride_x, int* act,
                      int* nact, void* oz_ws, int slices, double eps_rel, double slice_budget, cudaStream_t stream,
                      int64_t* launches) {
  // 64-byte k-chunks (measured on B200: 32-byte chunks with a 5-deep ring are 13% slower on the
  // 528-root call -- 585 vs 673 roots/s; SWIZZLE_32B TMA rows are short requests)
  if (slices != 6 && slices != 7)
    return set_error(SHAMPOO_ERR_INVALID_ARG, "ozaki root: slices must be 6 or 7 (got %d)", slices);
  if (batch > kTailMaxBatch) return set_error(SHAMPOO_ERR_UNSUPPORTED, "ozaki root: batch chunk > %d", kTailMaxBatch);
  if (np % 64) return set_error(SHAMPOO_ERR_UNSUPPORTED, "ozaki root: padded n must be a multiple of 64");
  char* w = static_cast<char*>(oz_ws);
  const size_t slot_planes = (size_t)batch * oz::kSMax * oz::plane_pitch(np);  // every slot at the kSMax pitch
  int8_t* planes = reinterpret_cast<int8_t*>(w);
  const size_t planes_bytes = ((size_t)OZ_SLOTS * slot_planes + 255) / 256 * 256;
  double* scales = reinterpret_cast<double*>(w + planes_bytes);
  const size_t scales_bytes = ((size_t)OZ_SLOTS * batch * np * sizeof(double) + 255) / 256 * 256;
  auto slot_planes_ptr = [&](int slot) { return planes + (size_t)slot * slot_planes; };
  auto slot_scale = [&](int slot) { return scales + (size_t)slot * batch * np; };
  const int64_t mstride = (int64_t)kTailRegions * np * np;
  auto region = [&](int r) { return bufs + (int64_t)r * np * np; };
  // tm: slice T_k = ((p+1)I - M_k)/p computed from M_k on the fly (T_k never stored in fp64)
  oz::OzArgs base;
  std::memset(&base, 0, sizeof base);
  base.act = act;
  base.nact = nact;
  base.batch = batch;
  base.n = n;
  base.np = np;
  base.tiles_m = (n + oz::kBM - 1) / oz::kBM;
  base.tiles_n = (n + oz::kBN - 1) / oz::kBN;
  base.sym = 1;
  base.p = p;
  base.errh = errh;
  base.max_iter = max_iter;
  base.jobs = 1;
  auto job = [&](int sa, int sb, int out_reg) {
    oz::OzJob j;
    j.a_planes = slot_planes_ptr(sa);
    j.b_planes = slot_planes_ptr(sb);
    j.a_scale = slot_scale(sa);
    j.b_scale = slot_scale(sb);
    j.out = region(out_reg);
    j.out_stride = mstride;
    j.planes = nullptr;
    j.out_scale = nullptr;
    j.out_e = 0;
    j.outf = nullptr;
    j.outf_ld = nullptr;
    j.outf_rows = nullptr;
    return j;
  };
  // T^m (m >= 2) sliced by the product's own epilogue: every row scaled by 2^e with
  // 2^e > ((p+1)/p)^m >= rho(T)^m >= |(T^m)_ij| (reading #28; a violated bound is
  // flagged as a non-finite err, status 2).  The sliced epilogue needs no shared memory.
  auto sliced_job = [&](int sa, int sb, int slot, int m) {
    oz::OzJob j = job(sa, sb, 0);
    j.out = nullptr;
    j.planes = slot_planes_ptr(slot);
    j.out_scale = slot_scale(slot);
    const double bound = std::pow((double)(p + 1) / (double)p, m) * (1.0 + 1e-9);
    int e = 0;
    while (std::ldexp(1.0, e) <= bound) ++e;
    j.out_e = e;
    return j;
  };
  // one iteration's launches on stream `st`: k = the iteration (direct) or, with kdev, its parity only (the tail
  // graph's body reads k from *kdev); `prof`: bracket the GEMMs with CUDA events (not inside a graph)
  int* kdev = reinterpret_cast<int*>(w + planes_bytes + scales_bytes);
  auto gemm = [&](int S, const oz::OzArgs& a, cudaStream_t st, bool prof) -> int {
    void* tok = nullptr;
    if (prof) prof_begin_launch("ozaki_gemm", st, &tok);
    cudaError_t e = oz_gemm(S, a, st);
    if (prof) prof_end_launch(tok, st);
    if (e != cudaSuccess) return set_cuda_error("ozaki gemm launch", e);
    ++*launches;
    return SHAMPOO_OK;
  };
  enum { RX0 = 0, RX1 = 1, RM0 = 2, RM1 = 3, RT = 4, RS0 = 5, RS1 = 6 };  // root.cu regions
  const int lead = 31 - __builtin_clz((unsigned)p);
  auto iteration = [&](int k, int S, int Sx, cudaStream_t st, const int* kd) -> int {
    const bool prof = kd == nullptr;
    const int xs = k & 1;
    oz_slice(Sx, false, region(RX0 + xs), mstride, n, np, batch, act, nact, slot_planes_ptr(OZ_SX), slot_scale(OZ_SX),
             p, st);
    ++*launches;
    if (n <= 1024) {  // M_k and T_k = ((p+1)I - M_k)/p in one pass over M_k (rows up to 1024 in registers)
      oz_slice_mt(S, region(RM0 + xs), mstride, n, np, batch, act, nact, slot_planes_ptr(OZ_SM), slot_scale(OZ_SM),
                  slot_planes_ptr(OZ_ST), slot_scale(OZ_ST), p, st);
      ++*launches;
    } else {
      oz_slice(S, false, region(RM0 + xs), mstride, n, np, batch, act, nact, slot_planes_ptr(OZ_SM),
               slot_scale(OZ_SM), p, st);
      oz_slice(S, true, region(RM0 + xs), mstride, n, np, batch, act, nact, slot_planes_ptr(OZ_ST), slot_scale(OZ_ST),
               p, st);
      *launches += 2;
    }
    oz::OzArgs b0 = base;
    b0.kcheck = k + 1;
    b0.kdev = kd;
    // P1: X_{k+1} = X_k T (fp64); then S0 = T T (p >= 2; sliced in the epilogue).  Two launches: a stage whose
    // jobs take different epilogue paths was measured 17-18 ms against 6 + 6 ms for the two alone (the
    // alternating paths thrash the instruction cache)
    oz::OzArgs a1 = b0;
    a1.job[0] = job(OZ_SX, OZ_ST, RX0 + (xs ^ 1));
    int rc = gemm(Sx, a1, st, prof);
    if (rc) return rc;
    if (p >= 2) {
      oz::OzArgs a2 = b0;
      a2.job[0] = sliced_job(OZ_ST, OZ_ST, OZ_SS0, 2);
      rc = gemm(S, a2, st, prof);
      if (rc) return rc;
    }
    int rb = RS0, sb = OZ_SS0, m = 2;
    for (int bit = lead - 1; bit >= 0; --bit) {
      if (bit != lead - 1) {  // square
        const int rd = rb == RS0 ? RS1 : RS0, sd = sb == OZ_SS0 ? OZ_SS1 : OZ_SS0;
        oz::OzArgs q = b0;
        q.job[0] = sliced_job(sb, sb, sd, 2 * m);
        rc = gemm(S, q, st, prof);
        if (rc) return rc;
        rb = rd;
        sb = sd;
        m *= 2;
      }
      if ((p >> bit) & 1) {  // times T
        const int rd = rb == RS0 ? RS1 : RS0, sd = sb == OZ_SS0 ? OZ_SS1 : OZ_SS0;
        oz::OzArgs q = b0;
        q.job[0] = job(sb, OZ_ST, rd);  // A != B: fp64 output and the slice kernel
        rc = gemm(S, q, st, prof);
        if (rc) return rc;
        oz_slice(S, false, region(rd), mstride, n, np, batch, act, nact, slot_planes_ptr(sd), slot_scale(sd), p, st);
        ++*launches;
        rb = rd;
        sb = sd;
        m += 1;
      }
    }
    // P3: M_{k+1} = T^p M_k ; err_{k+1} = max|M_{k+1} - I|
    oz::OzArgs a3 = b0;
    a3.job[0] = job(p == 1 ? OZ_ST : sb, OZ_SM, RM0 + (xs ^ 1));
    a3.mupdate = 1;
    return gemm(S, a3, st, prof);
  };
  auto sched = [&](int k, int& S, int& Sx) {
    // slices of iteration k's products (reading #29); the X-update reads the leading Sx planes of T
    S = ozaki_iteration_slices(k, p, n, eps_rel, slice_budget, slices);
    Sx = slice_budget > 0.0 ? std::min(S, kOzSX) : S;
  };
  // iterations 0 .. k_direct-1 one launch at a time (their slice counts may change), then the convergence-driven
  // tail: a CUDA graph whose conditional WHILE node repeats a two-iteration body until the decide kernel finds no
  // active matrix -- no host round trip, no launch after convergence (round 1 enqueued all max_iter iterations)
  // SHAMPOO_OZAKI_DIRECT (tests only): "all" -- every iteration launched directly; an integer k -- the tail graph
  // from k on (rounded up to even and to the schedule's floor), for the bit-identity check of the tail
  static const int direct_env = [] {
    const char* v = std::getenv("SHAMPOO_OZAKI_DIRECT");
    if (!v || !*v) return -1;
    if (std::strcmp(v, "all") == 0) return 1 << 30;
    return std::atoi(v);
  }();
  int k_direct = ozaki_direct_iterations(p, n, eps_rel, tol, max_iter, slice_budget, slices);
  if (direct_env >= 0) {
    const int s_floor = ozaki_iteration_slices(1000, p, n, eps_rel, slice_budget, slices);
    k_direct = std::min(direct_env, max_iter);
    while (k_direct < max_iter && ozaki_iteration_slices(k_direct, p, n, eps_rel, slice_budget, slices) != s_floor)
      ++k_direct;
    if (k_direct & 1) ++k_direct;
    k_direct = std::min(k_direct, max_iter);
  }
  int rc = SHAMPOO_OK;
  for (int k = 0; k < k_direct; ++k) {
    int S, Sx;
    sched(k, S, Sx);
    rc = iteration(k, S, Sx, stream, nullptr);
    if (rc) return rc;
    root_tail_decide_kernel<<<1, 1024, 0, stream>>>(act, nact, errh, max_iter, tol, 1.0, k + 1);
    ++*launches;
  }
  if (k_direct < max_iter) {
    int S, Sx;
    sched(k_direct, S, Sx);  // = the schedule's floor for every k >= k_direct
    const int kd_host = k_direct;
    if (cudaMemcpyAsync(kdev, &kd_host, sizeof(int), cudaMemcpyHostToDevice, stream) != cudaSuccess)
      return set_cuda_error("cudaMemcpyAsync(ozaki tail counter)");
    rc = ozaki_tail_graph(stream, [&](cudaStream_t cs, cudaGraphConditionalHandle h) -> int {
      for (int half = 0; half < 2; ++half) {
        int r = iteration(half, S, Sx, cs, kdev);  // parity of k_direct + half (k_direct is even)
        if (r) return r;
        root_tail_decide_graph_kernel<<<1, 1024, 0, cs>>>(act, nact, errh, max_iter, tol, 1.0, kdev, h, half);
        ++*launches;
      }
      return SHAMPOO_OK;
    });
    if (rc) return rc;
  }
  root_tail_finish_kernel<<<batch, 256, 0, stream>>>(bufs, res, errh, info, X, ldx, stride_x, batch, n, np, max_iter,
                                                     0, tol, 1.0, RX0, RX1, 1);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("ozaki root kernels", e);
  return SHAMPOO_OK;
}

}  // namespace shp
