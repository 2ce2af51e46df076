// ozaki.cuh -- fp64-accurate matrix products on the INT8 tensor cores
// (tcgen05.mma.kind::i8, exact int32 accumulation in TMEM): the Ozaki splitting
// used by the "ozaki" precision of the coupled-Newton root.
//
// Slicing (per operand matrix, per row i): e_i = exponent of max_k |A_ik|
// (frexp: max < 2^e_i), a = A_ik 2^-e_i in (-1, 1);  V = rint(a 2^(6+7(S-1)))
// (the only rounding, |V| < 2^48 for S = 7), then balanced base-128 digits from
// the bottom: d_S = ((V + 64) mod 128) - 64, V = (V - d_S) / 128, ..., d_1 = V;
// |d_s| <= 64 (int8), a = sum_s d_s 2^-(6+7(s-1)) + O(2^-(7S)).
// Product C = A B^T (B by rows): pairs (s, t) with s + t <= S + 1 accumulate,
// grouped by d = s + t - 2, in one int32 TMEM accumulator per d -- exact:
// |sum| <= S * K * 64^2 < 2^31 for K <= 4096, S <= 8.  Epilogue, in fp64:
//   C_ij = 2^e_i 2^f_j sum_{d = S-1 .. 0} acc_d 2^-(12 + 7d)
// (products by powers of two are exact; the sum is the only rounding).
// With S = 7 the product error is ~K 2^-49 max|A_i.| max|B_j.| (numpy
// emulation of the whole root at n = 256: 3.2e-8 vs the fp64 root, below the
// fp32 output rounding; S = 6: 3.7e-6).
//
// GEMM kernel: one CTA per SM, persistent over 128 x 64 output tiles; warp 0 =
// TMA producer (per 64-byte k-chunk: S A-planes 128 x 64 B and S B-planes 64 x
// 64 B, SWIZZLE_64B, 2-stage ring), warp 1 = TMEM allocator + MMA issuer (28
// tcgen05.mma.kind::i8 M=128 N=64 K=32 per k-step for S = 7), warps 2..5 =
// epilogue (7 tcgen05.ld per 16 columns, fp64 combination, mode-specific store).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace shp {
namespace oz {

constexpr int kS = 7;                       // slices per operand
constexpr int kBM = 128, kBN = 64, kBK = 64;  // tile M, N; k-chunk in bytes (int8 elements): two K=32 MMA steps
constexpr int kAPlane = kBM * kBK;          // 8 KB
constexpr int kBPlane = kBN * kBK;          // 4 KB
constexpr int kStageBytes = kS * (kAPlane + kBPlane);  // 84 KB
constexpr int kStages = 2;  // (measured: 32-byte k-chunks x 4 stages were 4% slower)
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;         // kS accumulators x 64 columns (448 used)
// accumulator weights 2^-(12 + 7d)
__device__ __constant__ const double kW[8] = {0x1p-12, 0x1p-19, 0x1p-26, 0x1p-33, 0x1p-40, 0x1p-47, 0x1p-54, 0x1p-61};

// K-major tile of kBK-byte rows, swizzled to match the TMA map (SWIZZLE_32B:
// layout type 6, 8-row atoms of 256 B; SWIZZLE_64B: type 4, 512 B)
TC_DEV uint64_t desc_sw(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)((8 * kBK) >> 4) << 32;     // SBO: 8 rows x kBK bytes
  d |= (uint64_t)1 << 46;                    // version 1 (sm_100)
  d |= (uint64_t)(kBK == 32 ? 6 : 4) << 61;  // SWIZZLE_32B / SWIZZLE_64B
  return d;
}

constexpr uint32_t idesc_i8(int M, int N) {
  // c_format S32 (2) [4,6), a/b format INT8 (1) [7,10) / [10,13), K-major, N>>3 [17,23), M>>4 [24,29)
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

TC_DEV void umma_i8(uint32_t tmem_c, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_c),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// --------------------------------------------------------------- slicing
// One warp per (matrix, row): scale[mat*np + i] = 2^e_i, planes
// [(mat*kS + s)*np + i]*np + j = d_s(A_ij) for j < n.
__global__ void __launch_bounds__(256) slice_kernel(const double* __restrict__ src, int64_t mat_stride, int n, int np,
                                                    int batch, const int* __restrict__ act, const int* nact,
                                                    int8_t* __restrict__ planes, double* __restrict__ scale) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int na = act ? *nact : batch;
  for (int64_t rid = gw; rid < (int64_t)na * n; rid += nw) {
    const int pos = (int)(rid / n), i = (int)(rid - (int64_t)pos * n);
    const int mat = act ? act[pos] : pos;
    const double* row = src + mat * mat_stride + (int64_t)i * np;
    double mx = 0.0;
    for (int j = lane; j < n; j += 32) mx = fmax(mx, fabs(row[j]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    if (lane == 0) scale[(int64_t)mat * np + i] = ldexp(1.0, e);
    const int sh = 6 - e;
    // 8 consecutive columns per lane (two double4 loads in flight, one 8-byte
    // store per plane); the row tail (n % 8) element-wise
    for (int j = 8 * lane; j < n; j += 256) {
      double r[8];
      if (j + 8 <= n) {
        const double4 u0 = *reinterpret_cast<const double4*>(row + j);
        const double4 u1 = *reinterpret_cast<const double4*>(row + j + 4);
        r[0] = u0.x; r[1] = u0.y; r[2] = u0.z; r[3] = u0.w;
        r[4] = u1.x; r[5] = u1.y; r[6] = u1.z; r[7] = u1.w;
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = (j + q < n) ? row[j + q] : 0.0;
      }
      // one rounding to the 2^-48 grid (|V| < 2^48), then balanced base-128 digits
      // by integer ops, lowest first: d = ((V + 64) mod 128) - 64, V = (V - d) / 128
      // (32-bit integer work: V = H 2^21 + L, the three low digits from L, the
      // carry into H, the four high digits from H)
      static_assert(kS == 7, "the 21 + 27-bit split assumes 7 slices");
      uint32_t dig[kS][2];
#pragma unroll
      for (int s = 0; s < kS; ++s) dig[s][0] = dig[s][1] = 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const long long V = __double2ll_rn(ldexp(r[q], sh + 7 * (kS - 1)));
        int H = (int)(V >> 21);
        int L = (int)(V & 0x1FFFFF);
        int d;
#pragma unroll
        for (int s = kS - 1; s >= kS - 3; --s) {
          d = ((L + 64) & 127) - 64;
          L = (L - d) >> 7;
          dig[s][q >> 2] |= ((uint32_t)d & 0xFFu) << (8 * (q & 3));
        }
        H += L;
#pragma unroll
        for (int s = kS - 4; s >= 1; --s) {
          d = ((H + 64) & 127) - 64;
          H = (H - d) >> 7;
          dig[s][q >> 2] |= ((uint32_t)d & 0xFFu) << (8 * (q & 3));
        }
        dig[0][q >> 2] |= ((uint32_t)H & 0xFFu) << (8 * (q & 3));
      }
#pragma unroll
      for (int s = 0; s < kS; ++s) {
        const uint32_t w[2] = {dig[s][0], dig[s][1]};
        int8_t* dst = planes + (((int64_t)mat * kS + s) * np + i) * np + j;
        if (j + 8 <= n) {
          *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (j + q < n) dst[q] = (int8_t)((w[q >> 2] >> (8 * (q & 3))) & 0xFFu);
        }
      }
    }
  }
}

// --------------------------------------------------------------- GEMM
struct OzJob {
  int a_map, b_map;         // TMA maps of the A-use (128-row box) / B-use (64-row box) planes
  const double* a_scale;    // [mat * np + row] = 2^e
  const double* b_scale;
  double* out;              // fp64 output of matrix 0; matrix m at out + m * out_stride
  int64_t out_stride;
};

struct OzArgs {
  const int* act;           // active matrices (nullptr: 0 .. batch-1)
  const int* nact;
  int batch, n, np, tiles_m, tiles_n;
  int sym;                  // upper tiles only (tj >= 2 ti), each stored twice (j >= i, mirrored)
  int jobs;
  OzJob job[2];
  int mupdate;              // job 0's epilogue: M-update (T_{k+1} and max|M - I|)
  double* t_out;
  int64_t t_stride;
  int p;
  double* errh;
  int max_iter, kcheck;
};

TC_DEV int oz_tiles_per_mat(const OzArgs& a) {
  if (!a.sym) return a.tiles_m * a.tiles_n;
  int t = 0;
  for (int ti = 0; ti < a.tiles_m; ++ti) t += max(0, a.tiles_n - 2 * ti);
  return t;
}

TC_DEV void oz_decode(const OzArgs& a, int per_mat, int64_t tile, int& mat, int& job, int& ti, int& tj) {
  const int64_t per = (int64_t)per_mat * a.jobs;
  const int pos = (int)(tile / per);
  int rem = (int)(tile - (int64_t)pos * per);
  job = rem % a.jobs;
  int t = rem / a.jobs;
  if (a.sym) {
    int i = 0;
    while (t >= a.tiles_n - 2 * i) {
      t -= a.tiles_n - 2 * i;
      ++i;
    }
    ti = i;
    tj = 2 * i + t;
  } else {
    ti = t / a.tiles_n;
    tj = t - ti * a.tiles_n;
  }
  mat = a.act ? a.act[pos] : pos;
}

__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ OzArgs a,
                                                          const CUtensorMap* __restrict__ maps) {
  const int na = a.act ? *a.nact : a.batch;
  if (na == 0) return;
  const int per_mat = oz_tiles_per_mat(a);
  const int64_t total = (int64_t)na * per_mat * a.jobs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    tc::mbar_init(tmem_full, 1);
    tc::mbar_init(tmem_empty, 128);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(tmem_base_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  const int k_chunks = (a.n + kBK - 1) / kBK;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (tc::elect_one()) {
      for (int q = 0; q < 2 * a.jobs; ++q) tc::tma_acquire(maps + (q & 1 ? a.job[q >> 1].b_map : a.job[q >> 1].a_map));
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        int mat, job, ti, tj;
        oz_decode(a, per_mat, tile, mat, job, ti, tj);
        const CUtensorMap* am = maps + a.job[job].a_map;
        const CUtensorMap* bm = maps + a.job[job].b_map;
        for (int kc = 0; kc < k_chunks; ++kc) {
          tc::mbar_wait(empty + stage, phase ^ 1);
          uint8_t* st = smem + stage * kStageBytes;
          tc::mbar_arrive_expect_tx(full + stage, kStageBytes);
#pragma unroll
          for (int s = 0; s < kS; ++s) {
            tc::tma_load_3d(st + s * kAPlane, am, full + stage, kc * kBK, ti * kBM, mat * kS + s);
            tc::tma_load_3d(st + kS * kAPlane + s * kBPlane, bm, full + stage, kc * kBK, tj * kBN, mat * kS + s);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc_phase = 0;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      tc::mbar_wait(tmem_empty, acc_phase ^ 1);
      tc::tc_fence_after();
      for (int kc = 0; kc < k_chunks; ++kc) {
        tc::mbar_wait(full + stage, phase);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t s0 = tc::smem_u32(smem + stage * kStageBytes);
          // plane and k-step offsets are added to the 14-bit (addr >> 4) field
          const uint64_t dA0 = desc_sw(s0), dB0 = desc_sw(s0 + kS * kAPlane);
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k) {
            const uint64_t adv = (uint64_t)((k * 32) >> 4);  // 32 bytes per K=32 step
            // A plane sa against up to 4 consecutive B planes at once: the B planes
            // are consecutive 64-row blocks of one K-major tile, and pairs (sa, tb..tb+3)
            // land in the consecutive accumulators d = sa + tb .. sa + tb + 3 (64
            // TMEM columns each) -- one MMA of N = 64 * count reads A once for all
            // of them (10 MMAs per k-step instead of 28: a third of the A traffic)
#pragma unroll
            for (int sa = 0; sa < kS; ++sa) {
#pragma unroll
              for (int tb = 0; tb < kS - sa; tb += 4) {
                const int cnt = (kS - sa - tb) < 4 ? (kS - sa - tb) : 4;
                const uint64_t da = dA0 + (uint64_t)((sa * kAPlane) >> 4) + adv;
                const uint64_t db = dB0 + (uint64_t)((tb * kBPlane) >> 4) + adv;
                // sa == 0 initialises every diagonal at the first k-step (it spans d = 0..6)
                const uint32_t acc = (kc == 0 && k == 0 && sa == 0) ? 0u : 1u;
                umma_i8(tmem_base + (uint32_t)((sa + tb) * kBN), da, db, idesc_i8(kBM, kBN * cnt), acc);
              }
            }
          }
          tc::umma_commit(empty + stage);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (tc::elect_one()) tc::umma_commit(tmem_full);
      __syncwarp();
      acc_phase ^= 1;
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;
    const int row_in_tile = quad * 32 + lane;
    uint32_t acc_phase = 0;
    const double inv_p = 1.0 / (double)a.p, pp1 = (double)(a.p + 1);
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      int mat, job, ti, tj;
      oz_decode(a, per_mat, tile, mat, job, ti, tj);
      tc::mbar_wait(tmem_full, acc_phase);
      tc::tc_fence_after();
      const int i = ti * kBM + row_in_tile;
      const bool row_ok = i < a.n;
      const OzJob& J = a.job[job];
      const bool mup = a.mupdate && job == 0;
      double* out = J.out + mat * J.out_stride;
      double* tout = mup ? a.t_out + mat * a.t_stride : nullptr;
      const double sa = row_ok ? J.a_scale[(int64_t)mat * a.np + i] : 0.0;
      // phase 1: drain the 7 accumulators of all 64 columns into fp64 registers
      // (sum over d, smallest weights first), then release TMEM so the next
      // tile's MMAs overlap this tile's scaling and stores
      double v[kBN];
#pragma unroll
      for (int c0 = 0; c0 < kBN; c0 += 16) {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[c0 + e] = 0.0;
#pragma unroll
        for (int d = kS - 1; d >= 0; --d) {
          uint32_t r[16];
          tc::tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(d * kBN + c0), r);
          tc::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) v[c0 + e] = v[c0 + e] + (double)(int)r[e] * kW[d];
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(tmem_empty);
      // phase 2: scale by 2^e_i 2^f_j, store row-major (16-byte vectors) and mirrored
      double emax = 0.0;
      if (row_ok) {
        const int j0 = tj * kBN;
        const double* bs = J.b_scale + (int64_t)mat * a.np + j0;
        double* orow = out + (int64_t)i * a.np + j0;
        double* trow = mup ? tout + (int64_t)i * a.np + j0 : nullptr;
        const bool full_row = j0 + kBN <= a.n && (!a.sym || j0 >= i);
#pragma unroll
        for (int e = 0; e < kBN; e += 2) {
          const double2 b2 = *reinterpret_cast<const double2*>(bs + e);
          const double c0 = v[e] * sa * b2.x, c1 = v[e + 1] * sa * b2.y;
          v[e] = c0;
          v[e + 1] = c1;
          if (full_row) {
            *reinterpret_cast<double2*>(orow + e) = make_double2(c0, c1);
          } else {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int j = j0 + e + q;
              if (j < a.n && (!a.sym || j >= i)) orow[e + q] = q ? c1 : c0;
            }
          }
          if (mup) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int j = j0 + e + q;
              if (j < a.n && (!a.sym || j >= i)) {
                const double c = q ? c1 : c0;
                const double dl = (i == j) ? 1.0 : 0.0;
                trow[e + q] = (pp1 * dl - c) * inv_p;
                emax = fmax_nan(emax, fabs(c - dl));
              }
            }
          }
        }
        if (a.sym) {  // mirror: lanes are consecutive rows -> coalesced
#pragma unroll
          for (int e = 0; e < kBN; ++e) {
            const int j = j0 + e;
            if (j >= a.n || j <= i) continue;
            out[(int64_t)j * a.np + i] = v[e];
            if (mup) tout[(int64_t)j * a.np + i] = (pp1 * 0.0 - v[e]) * inv_p;
          }
        }
      }
      if (mup) {
        emax = warp_max(emax);
        if (lane == 0) atomic_max_nonneg(a.errh + (int64_t)mat * (a.max_iter + 1) + a.kcheck, emax);
      }
      acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<kTmemCols>(tmem_base);
  }
}

inline size_t gemm_smem_bytes() { return 1024 + (size_t)kStages * kStageBytes + 256; }

// 3-D TMA map over int8 slice planes: (k bytes = n, rows = n, planes = batch * kS),
// row pitch np bytes, plane pitch np*np bytes, box (64 B, box_rows, 1), SWIZZLE_64B
template <class Encode>
inline CUresult make_plane_map(Encode enc, CUtensorMap* out, const int8_t* base, int n, int np, int batch,
                               int box_rows) {
  cuuint64_t gdim[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)batch * kS};
  cuuint64_t gstride[2] = {(cuuint64_t)np, (cuuint64_t)np * np};
  cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  return enc(out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), gdim, gstride, box, estride,
             CU_TENSOR_MAP_INTERLEAVE_NONE, kBK == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace oz
}  // namespace shp
