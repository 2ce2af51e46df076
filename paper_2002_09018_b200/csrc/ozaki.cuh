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
// With S = 7 the product error is ~K 2^-49 max|A_i.| max|B_j.| (host
// emulation of the whole root, tools/ozaki_precision.py, n = 256: 3.2e-8 vs the
// exact root, below the fp32 output rounding; S = 6: 3.8e-6; S = 5: 4.3e-4).
// S is a template parameter (6 or 7; the precision choice).
//
// GEMM kernel: one CTA per SM, persistent over 128 x 64 output tiles; warp 0 =
// bulk-copy producer (per 64-byte k-chunk: S A-planes 128 x 64 B and S B-planes
// 64 x 64 B, each one contiguous pre-swizzled block of the tiled plane layout;
// 2-stage ring for S = 7, 3 stages for S = 6, 5), warp 1 = TMEM allocator + MMA
// issuer (the S(S+1)/2 slice pairs of a k-step in 10 (S = 7) / 8 (S = 6)
// tcgen05.mma.kind::i8 of M = 128, N = 64..256, K = 32), warps 2..9 = epilogue
// (S tcgen05.ld per 8 columns behind one wait, fp64 combination, mode-specific
// store).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace shp {
namespace oz {

// most slices per operand: every operand's planes are laid out with this pitch
// (plane s of matrix mat is plane mat * kSMax + s), so products of different
// slice counts S <= kSMax read the leading S planes of the same buffers
// (the per-iteration slice schedule, reading #29)
constexpr int kSMax = 7;
constexpr int kBM = 128, kBN = 64;  // tile M, N

// Plane layout (round 2): every n x n int8 plane is stored as 64-row x 64-byte tiles, k-block major (tile (kb, rb)
// at (kb * nrb + rb) * 4096 bytes, nrb row blocks), each tile already in the shared-memory SWIZZLE_64B pattern the
// UMMA descriptors read (16-byte chunk c of row r at chunk c ^ ((r >> 1) & 3)).  An A tile (128 rows) is then ONE
// contiguous 8 KB block and a B tile one 4 KB block, moved by plain 1-D bulk copies: measured on B200 +8 / +11 /
// +14% executed TOPS at S = 7 / 6 / 5 over 3-D tensor-map copies of row-major planes (whose 64-byte rows are
// separate requests; 32-byte rows were slower still).  Rows are padded to a multiple of 128 (whole A tiles), the k
// extent to np (a multiple of 64).  Writers zero the k padding (columns n .. np-1) of rows < n; padding rows are
// never written and only reach outputs the epilogue discards.
__host__ __device__ constexpr int64_t plane_rows(int np) { return (int64_t)(np + 127) / 128 * 128; }
__host__ __device__ constexpr int64_t plane_pitch(int np) { return plane_rows(np) * np; }
__host__ __device__ __forceinline__ int64_t tiled_off(int i, int j, int np) {
  return ((int64_t)(j >> 6) * (plane_rows(np) >> 6) + (i >> 6)) * 4096 + ((i & 63) << 6) +
         ((((j >> 4) & 3) ^ ((i >> 1) & 3)) << 4) + (j & 15);
}
// k-chunk BK bytes (int8 elements) per pipeline stage: BK / 32 K=32 MMA steps
template <int S, int BK>
struct Cfg {
  static_assert(S >= 4 && S <= kSMax, "4 <= slices <= 7 (int32 digit split, TMEM columns)");
  static_assert(BK == 64, "64-byte k-chunks: the tiled plane layout");
  static constexpr int kAPlane = kBM * BK;                     // 8 KB (BK = 64)
  static constexpr int kBPlane = kBN * BK;                     // 4 KB
  static constexpr int kStageBytes = S * (kAPlane + kBPlane);  // 84 KB (S = 7, BK = 64), 72 KB (S = 6)
#ifdef OZ_STAGES  // microbenchmark probes only
  static constexpr int kStages = OZ_STAGES < (225 * 1024) / kStageBytes ? OZ_STAGES : (225 * 1024) / kStageBytes;
#else
  static constexpr int kStages = (225 * 1024) / kStageBytes;   // as many as fit: 2 / 5 (S = 7), 3 / 6 (S = 6)
#endif
};
// warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer, warps 2.. the epilogue: two warps per TMEM lane
// quadrant, each draining and storing 32 of the tile's 64 columns (kEpiCols) -- a tile's epilogue then costs half
// the time per warp, so it keeps pace with the MMAs of the next tile also at S = 5, 6 (round 1: 4 warps x 64
// columns).  10 warps put 3 on two of the SM's four 16K-register partitions: <= 168 registers per thread.
#ifndef OZ_EPI_WARPS
#define OZ_EPI_WARPS 8
#endif
constexpr int kEpiWarps = OZ_EPI_WARPS;  // 8 (library) or 16 (microbenchmark variant: 16 columns per warp)
static_assert(kEpiWarps == 8 || kEpiWarps == 16, "two or four epilogue warps per TMEM lane quadrant");
constexpr int kThreads = 64 + 32 * kEpiWarps;
// Bound probes for tools/microbench/ozaki_test.cu only (the library builds with 0):
// 1 = no MMAs (TMA data movement + barriers + epilogue), 2 = no TMA loads (MMAs on stale tiles),
// 4 = no loads and no epilogue (MMAs and the accumulator hand-off only), 5 = no epilogue (loads + MMAs),
// 6 = the drain (phase 1) but no scaling or stores, 7 = fp64 epilogue without its stores,
#ifndef OZ_PROBE
#define OZ_PROBE 0
#endif
constexpr uint32_t kTmemCols = 512;         // S accumulators x 64 columns (448 used for S = 7)

// K-major tile of BK-byte rows in the SWIZZLE_64B pattern of the tiled planes (layout type 4, 8-row atoms of
// 512 B; SWIZZLE_32B: type 6)
template <int kBK>
TC_DEV uint64_t desc_sw(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)((8 * kBK) >> 4) << 32;     // SBO: 8 rows x kBK bytes
  d |= (uint64_t)1 << 46;                    // version 1 (sm_100)
  d |= (uint64_t)(kBK == 32 ? 6 : 4) << 61;  // SWIZZLE_32B / SWIZZLE_64B
  return d;
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
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
// Digits of 8 consecutive elements r[0..7] of one row; scl = 2^(6 + 7(S-1) - e_i).
// One rounding to the integer grid, V = rint(r scl) (|V| < 2^(7S-1)), then the
// balanced base-128 digits d_s in [-64, 63] (top digit in [-64, 64]): with
// C = 64 sum_s 128^s, W = V + C >= 0 has unsigned base-128 digits u_s = d_s + 64
// (the carries of the balanced form are the carries of the addition).  Both
// steps in one fma: r scl + (1.5 2^52 + C) lands in [2^52, 2^53), where the
// fp64 grid is the integers, so its bit pattern is 0x4338000000000000 + W
// (RN ties-to-even, as rint).  Digits by bit-field extracts, packed 4 per word
// by bit-field inserts, d = u - 64 per byte (__vadd4).  dig[s] = 8 packed int8.
template <int S>
__device__ __forceinline__ void slice8(const double (&r)[8], double scl, uint32_t (&dig)[S][2]) {
  constexpr long long kC = (64LL * ((1LL << (7 * S)) - 1)) / 127;  // 64 sum_{s<S} 128^s
  constexpr double kMagic = (double)(0x18000000000000LL + kC);     // 1.5 2^52 + C, exact (< 2^53)
#pragma unroll
  for (int s = 0; s < S; ++s) dig[s][0] = dig[s][1] = 0u;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const long long b = __double_as_longlong(fma(r[q], scl, kMagic));
    const uint32_t lo = (uint32_t)b;                                    // W mod 2^32
    const uint32_t hi = (uint32_t)(b >> 32) - 0x43380000u;              // W >> 32 (W < 2^50)
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int pos = 7 * (S - 1 - s), len = s == 0 ? 8 : 7;
      uint32_t u;
      if (pos + len <= 32) u = __funnelshift_r(lo, 0u, pos) & ((1u << len) - 1u);
      else if (pos >= 32) u = (hi >> (pos - 32)) & ((1u << len) - 1u);
      else u = __funnelshift_r(lo, hi, pos) & ((1u << len) - 1u);
      dig[s][q >> 2] |= u << (8 * (q & 3));
    }
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    dig[s][0] = __vadd4(dig[s][0], 0xC0C0C0C0u);  // u - 64 in every byte (wrapping)
    dig[s][1] = __vadd4(dig[s][1], 0xC0C0C0C0u);
  }
}

// 2^(6 + 7(S-1) - e): the digit scale of a row with max < 2^e, e in [-960, 1024]
// (row_exponent), built in the exponent field directly
template <int S>
__device__ __forceinline__ double digit_scale(int e) {
  return __longlong_as_double((long long)(6 + 7 * (S - 1) - e + 1023) << 52);
}

// 8 consecutive elements of a row from column j (two 32-byte loads; the row
// tail n % 8 element-wise, zero beyond n)
__device__ __forceinline__ void load8(const double* row, int j, int n, double (&r)[8]) {
  if (j + 8 <= n) {
    const double4 u0 = *reinterpret_cast<const double4*>(row + j);
    const double4 u1 = *reinterpret_cast<const double4*>(row + j + 4);
    r[0] = u0.x; r[1] = u0.y; r[2] = u0.z; r[3] = u0.w;
    r[4] = u1.x; r[5] = u1.y; r[6] = u1.z; r[7] = u1.w;
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = (j + q < n) ? row[j + q] : 0.0;
  }
}

// digits of row i, columns j .. j+7 (j % 8 == 0, j < np: the k padding is stored as zeros) into a tiled plane
__device__ __forceinline__ void store8(int8_t* plane, int i, int j, int np, const uint32_t (&w)[2]) {
  *reinterpret_cast<uint2*>(plane + tiled_off(i, j, np)) = make_uint2(w[0], w[1]);
}

// Row exponent: e with max|row| < 2^e (0 for a zero row)
__device__ __forceinline__ int row_exponent(double mx) {
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
  return max(e, -960);          // keeps digit_scale<S>(e) a normal double (rows below 2^-960: fewer digits)
}

// |x| as an unsigned bit pattern (PTX, so it stays on the integer pipe): ordered like |x|
// for non-NaN x, NaN above +inf (the GEMM epilogue's max|M - I|, which must stay off the FP64 pipe)
__device__ __forceinline__ unsigned long long abs_bits(double x) {
  unsigned long long r;
  asm("and.b64 %0, %1, 0x7FFFFFFFFFFFFFFF;" : "=l"(r) : "l"(__double_as_longlong(x)));
  return r;
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) { return a > b ? a : b; }

// T_ij = ((p + 1) delta_ij - M_ij) / p, the same expression as the fp64 root's
// setup (root.cu) -- the coupled-Newton T_k is a function of M_k alone
__device__ __forceinline__ double t_of(double m, bool diag, double pp1, double inv_p) {
  return ((diag ? pp1 : 0.0) - m) * inv_p;
}

// One warp per (matrix, row): scale[mat*np + i] = 2^e_i, planes
// [(mat*kSMax + s)*np + i]*np + j = d_s(A_ij), s < S for j < n, where A = src, or, with TM,
// A = T_k = ((p+1)I - M_k)/p computed on the fly from src = M_k (T_k is never
// stored in fp64).  Rows of n <= 1024 are held in registers (32 doubles per
// lane, 8 KB in flight per warp, 16 warps per SM): ONE pass over HBM for the
// row maximum and the digits (measured 6.4 TB/s); longer rows take two passes
// (the second mostly from L1).
template <int S, bool TM>
__global__ void __launch_bounds__(256, 2) slice_kernel(const double* __restrict__ src, int64_t mat_stride, int n,
                                                       int np, int batch, const int* __restrict__ act,
                                                       const int* nact, int8_t* __restrict__ planes,
                                                       double* __restrict__ scale, int p) {
  constexpr int kRegChunks = 4;  // 4 x 256 columns per warp held in registers
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int na = act ? *nact : batch;
  const int64_t pitch = plane_pitch(np);
  const double pp1 = (double)(p + 1), inv_p = 1.0 / (double)p, ninv_p = -inv_p;
  for (int64_t rid = gw; rid < (int64_t)na * n; rid += nw) {
    const int pos = (int)(rid / n), i = (int)(rid - (int64_t)pos * n);
    const int mat = act ? act[pos] : pos;
    const double* row = src + mat * mat_stride + (int64_t)i * np;
    int8_t* pmat = planes + (int64_t)mat * kSMax * pitch;
    // TM: off the diagonal T_ij = -M_ij / p (one multiply: the same value as (0 - m) / p up to the sign
    // of zero); the diagonal element once per row
    const double tii = TM ? t_of(row[i], true, pp1, inv_p) : 0.0;
    if (n <= 256 * kRegChunks) {
      double r[kRegChunks][8];
      double mx = 0.0;
#pragma unroll
      for (int c = 0; c < kRegChunks; ++c) {
        const int j = 256 * c + 8 * lane;
        if (j < n) {
          load8(row, j, n, r[c]);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) r[c][q] = 0.0;
        }
        if (TM) {
#pragma unroll
          for (int q = 0; q < 8; ++q) r[c][q] = (j + q == i) ? tii : r[c][q] * ninv_p;  // beyond n: -0, never stored
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) mx = fmax(mx, fabs(r[c][q]));
      }
      const int e = row_exponent(mx);
      if (lane == 0) scale[(int64_t)mat * np + i] = ldexp(1.0, e);
#pragma unroll
      for (int c = 0; c < kRegChunks; ++c) {
        const int j = 256 * c + 8 * lane;
        if (j < np) {  // columns n .. np-1: zero digits (r = 0 there)
          uint32_t dig[S][2];
          slice8<S>(r[c], digit_scale<S>(e), dig);
#pragma unroll
          for (int s = 0; s < S; ++s) store8(pmat + s * pitch, i, j, np, dig[s]);
        }
      }
    } else {
      double mx = 0.0;
      for (int j = lane; j < n; j += 32) mx = fmax(mx, fabs(TM ? ((j == i) ? tii : row[j] * ninv_p) : row[j]));
      const int e = row_exponent(mx);
      if (lane == 0) scale[(int64_t)mat * np + i] = ldexp(1.0, e);
      for (int j = 8 * lane; j < np; j += 256) {
        double r[8];
        load8(row, j, n, r);
        if (TM) {
#pragma unroll
          for (int q = 0; q < 8; ++q) r[q] = (j + q == i) ? tii : r[q] * ninv_p;
        }
        uint32_t dig[S][2];
        slice8<S>(r, digit_scale<S>(e), dig);
#pragma unroll
        for (int s = 0; s < S; ++s) store8(pmat + s * pitch, i, j, np, dig[s]);
      }
    }
  }
}

// Row-pair slicer (rows of n <= 1024): one warp per pair of rows (i0, i0 + 1), i0 even, staged in shared memory by
// ONE bulk copy (the two rows are adjacent in HBM), then sliced from there.  Lanes 0-7 / 8-15 take 64 columns of row
// i0 / i0 + 1 in the same k-block, lanes 16-31 the next k-block, so every 8-byte-per-lane store instruction writes
// two WHOLE 128-byte lines of the tiled planes (rows i0, i0 + 1 of a tile are adjacent).  One row per warp wrote
// half lines: 3.5 vs 5.9 TB/s for the M/T slicer at S = 7 (tools/microbench/slice_layout.cu, r02ze).
// MODE 0: A = src;  MODE 1: T_k = ((p+1)I - M_k)/p from src = M_k (T_k is never stored in fp64);  MODE 2: both M_k
// (planes / scale) and T_k (planes_t / scale_t) in one pass over M_k.  Columns n .. np-1 get zero digits.
// W warps per CTA, B pair buffers (16 KB each) per warp: the next B - 1 pairs' copies are in flight while a pair is
// sliced.
constexpr int kPairWarps = 4, kPairBufs = 1;
template <int W, int B>
constexpr size_t pair_smem() { return (size_t)W * B * 2048 * sizeof(double) + (size_t)W * B * sizeof(uint64_t); }
constexpr size_t kPairSmem = pair_smem<kPairWarps, kPairBufs>();
template <int S, int MODE, int W = kPairWarps, int B = kPairBufs>
__global__ void __launch_bounds__(32 * W) slice_pair_kernel(
    const double* __restrict__ src, int64_t mat_stride, int n, int np, int batch, const int* __restrict__ act,
    const int* nact, int8_t* __restrict__ planes, double* __restrict__ scale, int8_t* __restrict__ planes_t,
    double* __restrict__ scale_t, int p) {
  extern __shared__ __align__(128) uint8_t pair_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* bufs = reinterpret_cast<double*>(pair_smem) + (size_t)wib * B * 2048;
  uint64_t* bars = reinterpret_cast<uint64_t*>(pair_smem + (size_t)W * B * 2048 * sizeof(double)) + wib * B;
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < B; ++b) tc::mbar_init(bars + b, 1);
    tc::fence_barrier_init();
  }
  __syncwarp();
  const int na = act ? *nact : batch;
  const int per_mat = (n + 1) >> 1;
  const int64_t total = (int64_t)na * per_mat;
  const int64_t gw = (int64_t)blockIdx.x * W + wib, nw = (int64_t)gridDim.x * W;
  // lane 0: the bulk copy of pair pid's two rows (adjacent in HBM; only the first n of the second) into buffer b
  auto issue = [&](int64_t pid, int b) {
    const int pos = (int)(pid / per_mat), i0 = 2 * (int)(pid - (int64_t)pos * per_mat);
    const int mat = act ? act[pos] : pos;
    const uint32_t bytes = (uint32_t)(((i0 + 1 < n ? np + n : n) * 8 + 15) & ~15);  // within the rows' padding
    tc::mbar_arrive_expect_tx(bars + b, bytes);
    tc::bulk_load(bufs + (size_t)b * 2048, src + mat * mat_stride + (int64_t)i0 * np, bytes, bars + b);
  };
  if (lane == 0)
    for (int b = 0; b < B; ++b)
      if (gw + b * nw < total) issue(gw + b * nw, b);
  const int64_t pitch = plane_pitch(np);
  const double pp1 = (double)(p + 1), inv_p = 1.0 / (double)p, ninv_p = -inv_p;
  const int r = (lane >> 3) & 1;        // this lane's row of the pair
  const int cl = 64 * (lane >> 4) + 8 * (lane & 7);  // its first column in each 128-column step
  const int steps = (np + 127) >> 7;
  int b = 0;
  uint32_t phase = 0;  // of buffer b (all buffers flip together, once per round of B pairs)
  for (int64_t pid = gw; pid < total; pid += nw) {
    const int pos = (int)(pid / per_mat), i0 = 2 * (int)(pid - (int64_t)pos * per_mat);
    const int mat = act ? act[pos] : pos;
    double* buf = bufs + (size_t)b * 2048;
    tc::mbar_wait(bars + b, phase);
    const int i = i0 + r;
    const bool live = i < n;
    const double* my = buf + r * np;
    const double mii = live ? my[i] : 0.0;
    const double tii = t_of(mii, true, pp1, inv_p);
    // row maxima over the 16 lanes of this row: |A| (MODE 0), |M| and |M| off the diagonal (MODE 1, 2)
    double mx = 0.0, mo = 0.0;
    for (int c = 0; c < steps; ++c) {
      const int j = 128 * c + cl;
      double v[8];
      if (live && j + 8 <= n) {
        const double4 a0 = *reinterpret_cast<const double4*>(my + j);
        const double4 a1 = *reinterpret_cast<const double4*>(my + j + 4);
        v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w; v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = (live && j + q < n) ? my[j + q] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        mx = fmax(mx, fabs(v[q]));
        if (MODE != 0) mo = fmax(mo, (j + q == i) ? 0.0 : fabs(v[q]));
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      if (o == 8) continue;
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mo = fmax(mo, __shfl_xor_sync(0xffffffffu, mo, o));
    }
    int e = 0, et = 0;
    if (mx > 0.0) frexp(mx, &e);
    e = max(e, -960);
    {
      const double mt = fmax(fabs(tii), mo * inv_p);  // max |T_ij|: fl(x inv_p) is monotone in x
      if (mt > 0.0) frexp(mt, &et);
      et = max(et, -960);
    }
    if ((lane & 23) == 0 && live) {  // lanes 0 and 8
      if (MODE != 1) scale[(int64_t)mat * np + i] = ldexp(1.0, e);
      if (MODE == 1) scale[(int64_t)mat * np + i] = ldexp(1.0, et);
      if (MODE == 2) scale_t[(int64_t)mat * np + i] = ldexp(1.0, et);
    }
    const double sa = digit_scale<S>(e), st = digit_scale<S>(et);
    int8_t* pa = planes + (int64_t)mat * kSMax * pitch;
    int8_t* pt = MODE == 2 ? planes_t + (int64_t)mat * kSMax * pitch : nullptr;
#pragma unroll 1
    for (int c = 0; c < steps; ++c) {
      const int j = 128 * c + cl;
      if (j < np) {
        double v[8];
        if (live && j + 8 <= n) {
          const double4 a0 = *reinterpret_cast<const double4*>(my + j);
          const double4 a1 = *reinterpret_cast<const double4*>(my + j + 4);
          v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w; v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = (live && j + q < n) ? my[j + q] : 0.0;
        }
        uint32_t dig[S][2];
        if (MODE != 1) {
          slice8<S>(v, sa, dig);
#pragma unroll
          for (int s = 0; s < S; ++s) store8(pa + s * pitch, i, j, np, dig[s]);
        }
        if (MODE != 0) {
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = (j + q == i) ? tii : v[q] * ninv_p;  // beyond n: -0 (zero digits)
          slice8<S>(v, st, dig);
          int8_t* dst = MODE == 2 ? pt : pa;
#pragma unroll
          for (int s = 0; s < S; ++s) store8(dst + s * pitch, i, j, np, dig[s]);
        }
      }
    }
    // the pair B ahead overwrites this buffer: order these generic reads before its bulk copy (async proxy)
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      if (pid + B * nw < total) issue(pid + B * nw, b);
    }
    __syncwarp();
    if (++b == B) {
      b = 0;
      phase ^= 1;
    }
  }
}

// --------------------------------------------------------------- GEMM
// W = V + C for an exact fp64 value c and a row scale 2^e_out, integer arithmetic
// only (the epilogue runs while the tensor pipe is busy): V = rint(c 2^(6 + 7(S-1)
// - e_out)) from the mantissa by a rounded shift (RN ties-to-even, as rint), so
// the base-128 digits of W are those slice8 produces for the same scale.
// ovf: |c| >= 2^e_out (the a-priori bound failed).
template <int S>
__device__ __forceinline__ unsigned long long int_w(double c, int e_out, bool& ovf) {
  constexpr long long kC = (64LL * ((1LL << (7 * S)) - 1)) / 127;
  const unsigned long long b = (unsigned long long)__double_as_longlong(c);
  const int ex = (int)((b >> 52) & 0x7FF);
  ovf |= (ex != 0) && (ex - 1023 >= e_out);
  const int sh = 1075 - (6 + 7 * (S - 1)) + e_out - ex;  // >= 5 when |c| < 2^e_out
  const int shc = min(max(sh, 1), 63);
  const unsigned long long m = (b & 0xFFFFFFFFFFFFFull) | (1ull << 52);
  unsigned long long q = m >> shc;
  const unsigned long long rem = m & ((1ull << shc) - 1ull), half = 1ull << (shc - 1);
  q += (rem > half || (rem == half && (q & 1ull))) ? 1ull : 0ull;
  q = (ex == 0 || sh >= 64 || sh < 1) ? 0ull : q;  // zero / subnormal / below the grid; overflow (flagged)
  const long long V = (b >> 63) ? -(long long)q : (long long)q;
  return (unsigned long long)(V + kC);
}

// 256-bit store of eight words (32-byte aligned; sm_100 STG.E.256)
__device__ __forceinline__ void st_v8(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e, uint32_t f,
                                      uint32_t g, uint32_t h) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d),
               "r"(e), "r"(f), "r"(g), "r"(h)
               : "memory");
}
// 256-bit evict-first store of four doubles (32-byte aligned; sm_100 STG.E.EF.256)
__device__ __forceinline__ void st_cs_v4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}


// fp32 round-to-nearest-even of a double on the integer pipe (normal fp32 results and zeros; anything else
// -- subnormal fp32 results, inf, NaN -- through the out-of-line conversion)
static __device__ __noinline__ float f32_of_slow(double x) { return __double2float_rn(x); }
__device__ __forceinline__ float f32_of(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  const unsigned sign = (unsigned)(b >> 32) & 0x80000000u;
  const int ex = (int)((b >> 52) & 0x7FF);
  const int e32 = ex - 1023 + 127;
  if ((b << 1) == 0ull) return __uint_as_float(sign);
  if (e32 >= 1 && e32 <= 254) {
    const unsigned long long m = b & 0xFFFFFFFFFFFFFull;
    unsigned q = (unsigned)(m >> 29);
    const unsigned long long rem = m & ((1ull << 29) - 1ull);
    q += (rem > (1ull << 28) || (rem == (1ull << 28) && (q & 1u))) ? 1u : 0u;
    return __uint_as_float(sign | (((unsigned)e32 << 23) + q));  // a mantissa carry bumps the exponent (inf past 254)
  }
  return f32_of_slow(x);
}

// byte of plane s (digit u_s - 64) from W; plane 0 takes 8 bits (top digit in [-64, 64])
template <int S>
__device__ __forceinline__ uint32_t w_byte(unsigned long long W, int s) {
  const int pos = 7 * (S - 1 - s);
  const uint32_t mask = s == 0 ? 0xFFu : 0x7Fu;
  return ((((uint32_t)(W >> pos)) & mask) + 192u) & 0xFFu;
}

// Integer-pipe helpers for the epilogue (no fp64 instruction while the tensor
// pipe runs; see the phase-2 note in gemm_kernel).
// e such that x = 2^e for the power-of-two row scales (exponent field - 1023)
__device__ __forceinline__ int exp2_of(double x) {
  return (int)((__double_as_longlong(x) >> 52) & 0x7FF) - 1023;
}
// x 2^k by two fp64 multiplies with exact power-of-two factors (|k| < 2000);
// out of line so the compiler cannot if-convert it into the common path
static __device__ __noinline__ double scale2_slow(double x, int k) {
  if (x == 0.0 || !isfinite(x)) return x;
  const int k1 = k / 2;
  return x * __longlong_as_double((long long)(k1 + 1023) << 52) * __longlong_as_double((long long)(k - k1 + 1023) << 52);
}
// x 2^k exactly by exponent arithmetic (integer pipe); zero, subnormal, inf,
// NaN or a result outside the normal range take scale2_slow (never on the
// Newton iterates' magnitudes, except exact zeros)
__device__ __forceinline__ double scale2(double x, int k) {
  const long long b = __double_as_longlong(x);
  const int ex = (int)((b >> 52) & 0x7FF);
  const int ne = ex + k;
  if (ex != 0 && ex != 0x7FF && ne >= 1 && ne <= 2046) return __longlong_as_double(b + ((long long)k << 52));
  return scale2_slow(x, k);
}

struct OzJob {
  const int8_t* a_planes;   // tiled planes of the A operand (plane s of matrix mat at (mat kSMax + s) plane_pitch)
  const int8_t* b_planes;   // and of the B operand (C = A B^T: both row-major in k)
  const double* a_scale;    // [mat * np + row] = 2^e
  const double* b_scale;
  double* out;              // fp64 output of matrix 0; matrix m at out + m * out_stride
  int64_t out_stride;
  // sliced output (out == nullptr, symmetric products only): the product's S int8 tiled planes at
  // planes + (mat kSMax + s) plane_pitch, every row scaled by the a-priori bound 2^out_e (|C_ij| < 2^out_e),
  // 2^out_e written to out_scale[mat np + row]
  int8_t* planes;
  double* out_scale;
  int out_e;
  // fp32 output (out == nullptr, planes == nullptr; the preconditioned gradient of one-sided blocks, a8):
  // matrix mat's rows i < outf_rows[mat] go to outf[mat] + i * outf_ld[mat] (columns j < n), rounded to
  // nearest fp32 by integer arithmetic (no fp64 instruction while the tensor pipe runs)
  float* const* outf;
  const int64_t* outf_ld;
  const int* outf_rows;
};

struct OzArgs {
  const int* act;           // active matrices (nullptr: 0 .. batch-1)
  const int* nact;
  int batch, n, np, tiles_m, tiles_n;
  int sym;                  // upper tiles only (tj >= 2 ti), each stored twice (j >= i, mirrored)
  int jobs;
  OzJob job[2];
  int mupdate;              // job 0's epilogue: max|M_{k+1} - I| into errh[mat][kcheck]
  int p;
  double* errh;
  int max_iter, kcheck;
  const int* kdev;          // non-null (the convergence-driven tail graph): the iteration index is *kdev, kcheck = *kdev + 1
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

// Each stage's planes arrive in 4 groups with their own full barriers, in the
// order the MMAs consume them, so the first MMAs of a stage start while the
// rest of its 84 KB is in flight: A plane sa in group gA(sa), B planes 0-3 in
// group 0, 4+ in group 1; MMA (sa, tb) needs group max(gA(sa), gB(tb)), which
// is nondecreasing in issue order (S = 7: 24 / 20 / 16 / 24 KB).
constexpr int kGroups = 4;
__host__ __device__ constexpr int grp_a(int sa) { return sa == 0 ? 0 : sa == 1 ? 1 : sa <= 3 ? 2 : 3; }
__host__ __device__ constexpr int grp_b(int tb) { return tb < 4 ? 0 : 1; }
template <int S, int BK>
__host__ __device__ constexpr int grp_bytes(int g) {
  int b = 0;
  for (int s = 0; s < S; ++s) {
    if (grp_a(s) == g) b += Cfg<S, BK>::kAPlane;
    if (grp_b(s) == g) b += Cfg<S, BK>::kBPlane;
  }
  return b;
}

template <int S, int BK>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ OzArgs a) {
  using C = Cfg<S, BK>;
  constexpr int kS = S, kBK = BK, kStages = C::kStages, kStageBytes = C::kStageBytes;
  static_assert(grp_bytes<S, BK>(0) + grp_bytes<S, BK>(1) + grp_bytes<S, BK>(2) + grp_bytes<S, BK>(3) == kStageBytes,
                "plane groups cover the stage");
  constexpr int kAPlane = C::kAPlane, kBPlane = C::kBPlane;
  const int na = a.act ? *a.nact : a.batch;
  if (na == 0) return;
  const int kcheck = a.kdev ? *a.kdev + 1 : a.kcheck;
  const int per_mat = oz_tiles_per_mat(a);
  const int64_t total = (int64_t)na * per_mat * a.jobs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);  // [stage][group]
  uint64_t* empty = full + kStages * kGroups;
  uint64_t* tmem_full = empty + kStages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      for (int g = 0; g < kGroups; ++g) tc::mbar_init(full + s * kGroups + g, 1);
      tc::mbar_init(empty + s, 1);
    }
    tc::mbar_init(tmem_full, 1);
    tc::mbar_init(tmem_empty, 32 * kEpiWarps);
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
      const int64_t pitch = plane_pitch(a.np);
      const int nrb = (int)(plane_rows(a.np) >> 6);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        int mat, job, ti, tj;
        oz_decode(a, per_mat, tile, mat, job, ti, tj);
        // this tile's planes: A rows 128 ti .. (row blocks 2 ti, 2 ti + 1: 8 KB), B rows 64 tj .. (4 KB) per k-block
        const int8_t* pa = a.job[job].a_planes + (int64_t)mat * kSMax * pitch + (int64_t)(2 * ti) * 4096;
        const int8_t* pb = a.job[job].b_planes + (int64_t)mat * kSMax * pitch + (int64_t)tj * 4096;
        for (int kc = 0; kc < k_chunks; ++kc) {
          tc::mbar_wait(empty + stage, phase ^ 1);
          uint8_t* st = smem + stage * kStageBytes;
#pragma unroll
          for (int g = 0; g < kGroups; ++g) {
            uint64_t* fb = full + stage * kGroups + g;
#if OZ_PROBE == 2 || OZ_PROBE == 4
            tc::mbar_arrive(fb);
            continue;
#endif
            tc::mbar_arrive_expect_tx(fb, grp_bytes<S, BK>(g));
            const int64_t kb = (int64_t)kc * nrb * 4096;
#pragma unroll
            for (int s = 0; s < kS; ++s) {
              if (grp_a(s) == g) tc::bulk_load(st + s * kAPlane, pa + s * pitch + kb, kAPlane, fb);
              if (grp_b(s) == g) tc::bulk_load(st + kS * kAPlane + s * kBPlane, pb + s * pitch + kb, kBPlane, fb);
            }
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
        const uint32_t s0 = tc::smem_u32(smem + stage * kStageBytes);
        // plane and k-step offsets are added to the 14-bit (addr >> 4) field
        const uint64_t dA0 = desc_sw<kBK>(s0), dB0 = desc_sw<kBK>(s0 + kS * kAPlane);
        int ready = -1;  // plane groups of this stage known to have landed (compile-time after unrolling)
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
              const int need = grp_a(sa) > grp_b(tb) ? grp_a(sa) : grp_b(tb);
              while (ready < need) {
                ++ready;
                tc::mbar_wait(full + stage * kGroups + ready, phase);
                tc::tc_fence_after();
              }
              const int cnt = (kS - sa - tb) < 4 ? (kS - sa - tb) : 4;
              const uint64_t da = dA0 + (uint64_t)((sa * kAPlane) >> 4) + adv;
              const uint64_t db = dB0 + (uint64_t)((tb * kBPlane) >> 4) + adv;
              // sa == 0 initialises every diagonal at the first k-step (it spans d = 0..6)
              const uint32_t acc = (kc == 0 && k == 0 && sa == 0) ? 0u : 1u;
              if (OZ_PROBE != 1 && lane == 0)
                umma_i8(tmem_base + (uint32_t)((sa + tb) * kBN), da, db, idesc_i8(kBM, kBN * cnt), acc);
            }
          }
        }
        if (lane == 0) tc::umma_commit(empty + stage);
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
    const int quad = warp & 3;                  // TMEM lane quadrant of this warp (hardware: warp % 4)
    constexpr int kEpiCols = kBN / (kEpiWarps / 4);
    const int cb = ((warp - 2) >> 2) * kEpiCols;  // this warp's first column of the tile
    const int row_in_tile = quad * 32 + lane;
    uint32_t acc_phase = 0;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      int mat, job, ti, tj;
      oz_decode(a, per_mat, tile, mat, job, ti, tj);
      // the tile's scales are loaded while its MMAs run: this lane's row scale, and ONE column-scale exponent per
      // lane (column j0 + cb + lane; phase 2 takes column e's from lane e - cb by a shuffle).  Round 2 loaded the
      // column scales in phase 2, after the release, where every load waited behind the epilogue's stores: the
      // stall samples sat on their first use (ncu r02zb)
      const int i = ti * kBM + row_in_tile;
      const bool row_ok = i < a.n;
      const OzJob& J = a.job[job];
      const double sa = row_ok ? J.a_scale[(int64_t)mat * a.np + i] : 0.0;
      const int bexp = exp2_of(J.b_scale[(int64_t)mat * a.np + tj * kBN + cb + lane]);
      tc::mbar_wait(tmem_full, acc_phase);
      tc::tc_fence_after();
#if OZ_PROBE >= 4  // no epilogue: release the accumulators at once
      tc::tc_fence_before();
      tc::mbar_arrive(tmem_empty);
      acc_phase ^= 1;
      continue;
#endif
      const bool mup = a.mupdate && job == 0;
      double* out = J.out + mat * J.out_stride;
      // phase 1: drain the S accumulators of all 64 columns, then release TMEM so
      // the next tile's MMAs overlap this tile's scaling and stores.  Per
      // 8-column chunk the S loads are issued back to back behind ONE wait.
      // Per element the exact value V = sum_d acc_d 2^(7(S-1-d)) (|V| < 2^68) is
      // rounded ONCE to fp64: H = sum_{d<4} acc_d 2^(7(3-d)) and L = sum_{d>=4}
      // acc_d 2^(7(S-1-d)) exactly in int64, both to fp64 exactly by the
      // 1.5 2^52 bit trick, x = fma(H, 2^(7(S-4)), L).  The FP64 work sits here,
      // where the tensor pipe is idle (the MMA warp waits for TMEM): measured
      // on B200, fp64 instructions issued while tcgen05 MMAs run stall ~100x
      // ("math pipe throttle"), so phase 2 below uses integer arithmetic only.
      double v[kEpiCols];  // columns cb .. cb + kEpiCols - 1 of the tile
#pragma unroll
      for (int c0 = 0; c0 < kEpiCols; c0 += 8) {
        uint32_t r[kS][8];
#pragma unroll
        for (int d = 0; d < kS; ++d)
          tc::tmem_ld8(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(d * kBN + cb + c0), r[d]);
        tc::tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          long long hi = 0, lo = 0;
#pragma unroll
          for (int d = 0; d < 4; ++d) hi += (long long)(int)r[d][e] << (7 * (3 - d));
#pragma unroll
          for (int d = 4; d < kS; ++d) lo += (long long)(int)r[d][e] << (7 * (kS - 1 - d));
          const double hd = __longlong_as_double(hi + 0x4338000000000000LL) - 0x1.8p52;  // exact, |hi| < 2^51
          const double ld = __longlong_as_double(lo + 0x4338000000000000LL) - 0x1.8p52;
          v[c0 + e] = fma(hd, (double)(1LL << (7 * (kS - 4))), ld);
        }
      }
      // pin the fp64 conversions before the release: the arrive's address depends
      // on every v (an OR of the high words; the offset is 0 at run time since
      // n > 0) -- otherwise ptxas sinks some of them past the arrive, into the
      // next tile's MMAs, where fp64 instructions crawl
      uint32_t dep = 0u;
#pragma unroll
      for (int e = 0; e < kEpiCols; ++e) dep |= (uint32_t)(__double_as_longlong(v[e]) >> 32);
      tc::tc_fence_before();
      tc::mbar_arrive(tmem_empty + ((dep == 0xFFFFFFFFu && a.n < 0) ? 1 : 0));
#if OZ_PROBE == 6  // drain only: no scaling, no stores
      acc_phase ^= 1;
      continue;
#endif
      // phase 2: scale by 2^(e_i + f_j - 12 - 7(S-1)) (exponent arithmetic), store
      // row-major (16-byte vectors) and mirrored, evict-first (st.global.cs: the
      // outputs must not push the operand planes other tiles still read out of L2); M-update: max|M - I| on the
      // bit patterns (T_{k+1} is sliced from M_{k+1} by slice_kernel<S, true>)
      unsigned long long emax_bits = 0ull, diag_bits = 0ull;
      if (J.planes) {
        // sliced output (symmetric products T^m): W of every element by integer arithmetic, then per plane
        // the row-major 64-byte segment (four 16-byte stores: whole sectors) and the mirror -- for tiles
        // strictly above the diagonal a warp-level 4 x 32 byte transpose (shuffles) turns it into 4-byte
        // stores of whole sectors; diagonal-band and ragged tiles store bytes
        const int j0 = tj * kBN;
        const int64_t pitch = plane_pitch(a.np);
        int8_t* pl = J.planes + (int64_t)mat * kSMax * pitch;
        // A = B (squarings): C is computed bit-symmetrically (the same exact integer pair sums, the same
        // scales), so the lower-triangle values a tile computes equal their mirrors and every in-range
        // tile may store whole rows and the whole transpose; otherwise only tiles above the diagonal
        const bool same_ab = J.a_planes == J.b_planes;
        const bool interior = (same_ab || j0 >= ti * kBM + kBM) && (j0 + kBN <= a.n) && (ti * kBM + kBM <= a.n);
        bool ovf = false;
        const int i0w = ti * kBM + quad * 32;  // this warp's first row
        const int ka = exp2_of(sa) - (12 + 7 * (kS - 1));
        if (row_ok && tj == 2 * ti && cb == 0)
          J.out_scale[(int64_t)mat * a.np + i] = __longlong_as_double((long long)(J.out_e + 1023) << 52);
        // this warp's kEpiCols columns
        {
          const int h = cb;
          unsigned long long w[kEpiCols];
          const int lim = a.n - (j0 + h);  // columns >= n (padding B rows, never written) stay 0: no false overflow
#pragma unroll
          for (int e = 0; e < kEpiCols; e += 2) {
            const int bx0 = __shfl_sync(0xffffffffu, bexp, e), bx1 = __shfl_sync(0xffffffffu, bexp, e + 1);
            if (row_ok) {
              w[e] = e < lim ? int_w<kS>(scale2(v[e], ka + bx0), J.out_e, ovf) : 0ull;
              w[e + 1] = e + 1 < lim ? int_w<kS>(scale2(v[e + 1], ka + bx1), J.out_e, ovf) : 0ull;
            } else {
              w[e] = w[e + 1] = 0ull;
            }
          }
#pragma unroll 1
          for (int s2 = 0; s2 < kS; ++s2) {
            int8_t* ps = pl + s2 * pitch;
            constexpr int kW = kEpiCols / 4;  // 4-byte words per row segment
            uint32_t wd[kW];
#pragma unroll
            for (int k = 0; k < kW; ++k)
              wd[k] = w_byte<kS>(w[4 * k], s2) | (w_byte<kS>(w[4 * k + 1], s2) << 8) |
                      (w_byte<kS>(w[4 * k + 2], s2) << 16) | (w_byte<kS>(w[4 * k + 3], s2) << 24);
            if (interior) {
              static_assert(kW == 8, "one 32-byte row segment per lane and plane");
              // the row's 32 bytes are the 16-byte chunks c, c+1 (c even) of one tile row, swizzled to the aligned
              // pair {c ^ x, (c+1) ^ x}, x = (i >> 1) & 3: one whole-sector 32-byte store, halves swapped for odd x
              int8_t* dst = ps + (tiled_off(i, j0 + h, a.np) & ~(int64_t)31);
              if ((i >> 1) & 1)
                st_v8(dst, wd[4], wd[5], wd[6], wd[7], wd[0], wd[1], wd[2], wd[3]);
              else
                st_v8(dst, wd[0], wd[1], wd[2], wd[3], wd[4], wd[5], wd[6], wd[7]);
              // mirror rows j0 + h + 4k + (lane >> 3), columns i0w + 4 (lane & 7) .. + 3
              const int src = 4 * (lane & 7), sel = 8 * (lane >> 3);
#pragma unroll
              for (int k = 0; k < kW; ++k) {
                const uint32_t x0 = __shfl_sync(0xffffffffu, wd[k], src);
                const uint32_t x1 = __shfl_sync(0xffffffffu, wd[k], src + 1);
                const uint32_t x2 = __shfl_sync(0xffffffffu, wd[k], src + 2);
                const uint32_t x3 = __shfl_sync(0xffffffffu, wd[k], src + 3);
                const uint32_t o = ((x0 >> sel) & 0xFFu) | (((x1 >> sel) & 0xFFu) << 8) |
                                   (((x2 >> sel) & 0xFFu) << 16) | (((x3 >> sel) & 0xFFu) << 24);
                *reinterpret_cast<uint32_t*>(ps + tiled_off(j0 + h + 4 * k + (lane >> 3), i0w + src, a.np)) = o;
              }
            } else if (row_ok) {
#pragma unroll
              for (int e = 0; e < kEpiCols; ++e) {
                const int j = j0 + h + e;
                const int8_t byte = (int8_t)((wd[e >> 2] >> (8 * (e & 3))) & 0xFFu);
                if (j < a.n && j >= i) ps[tiled_off(i, j, a.np)] = byte;
                if (j < a.n && j > i) ps[tiled_off(j, i, a.np)] = byte;
                if (j >= a.n && j < a.np) ps[tiled_off(i, j, a.np)] = 0;  // the k padding of row i
              }
            }
          }
        }
        if (ovf)  // the a-priori bound failed: poison this matrix's next err check (status 2, never silent)
          atomicMax(reinterpret_cast<unsigned long long*>(a.errh + (int64_t)mat * (a.max_iter + 1) + kcheck),
                    0x7FF8000000000000ull);
      } else if (J.outf) {
        // fp32 output (a8, one-sided blocks: P_b = G_b X_R; non-symmetric tiles, no mirror)
        {
          const bool live = row_ok && i < J.outf_rows[mat];
          const int j0 = tj * kBN;
          float* orow = live ? J.outf[mat] + (int64_t)i * J.outf_ld[mat] + j0 : nullptr;
          const int ka = exp2_of(sa) - (12 + 7 * (kS - 1));
          const bool vec = j0 + cb + kEpiCols <= a.n && ((reinterpret_cast<uintptr_t>(orow) & 15) == 0);
#pragma unroll
          for (int e = cb; e < cb + kEpiCols; e += 4) {
            const float f0 = f32_of(scale2(v[e - cb], ka + __shfl_sync(0xffffffffu, bexp, e - cb)));
            const float f1 = f32_of(scale2(v[e - cb + 1], ka + __shfl_sync(0xffffffffu, bexp, e - cb + 1)));
            const float f2 = f32_of(scale2(v[e - cb + 2], ka + __shfl_sync(0xffffffffu, bexp, e - cb + 2)));
            const float f3 = f32_of(scale2(v[e - cb + 3], ka + __shfl_sync(0xffffffffu, bexp, e - cb + 3)));
            if (!live) {
            } else if (vec) {
              __stcs(reinterpret_cast<float4*>(orow + e), make_float4(f0, f1, f2, f3));
            } else {
              if (j0 + e < a.n) orow[e] = f0;
              if (j0 + e + 1 < a.n) orow[e + 1] = f1;
              if (j0 + e + 2 < a.n) orow[e + 2] = f2;
              if (j0 + e + 3 < a.n) orow[e + 3] = f3;
            }
          }
        }
      } else {
        const int j0 = tj * kBN;
        double* orow = out + (int64_t)i * a.np + j0;
        const bool full_row = j0 + cb + kEpiCols <= a.n && (!a.sym || j0 + cb >= i);
        const int ka = exp2_of(sa) - (12 + 7 * (kS - 1));
#pragma unroll
        for (int e = cb; e < cb + kEpiCols; e += 2) {
          const double c0 = scale2(v[e - cb], ka + __shfl_sync(0xffffffffu, bexp, e - cb));
          const double c1 = scale2(v[e - cb + 1], ka + __shfl_sync(0xffffffffu, bexp, e - cb + 1));
          v[e - cb] = c0;
          v[e - cb + 1] = c1;
          if (!row_ok) continue;
          if (full_row) {
            // one 32-byte store per lane (a whole sector; STG.256): the row segments of 32 lanes are 32 rows apart,
            // so 16-byte stores left every sector half-written per instruction
#if OZ_PROBE != 7
            if ((e - cb) & 2) st_cs_v4(orow + e - 2, v[e - cb - 2], v[e - cb - 1], c0, c1);
#endif
          } else {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int j = j0 + e + q;
              if (j < a.n && (!a.sym || j >= i)) __stcs(orow + e + q, q ? c1 : c0);
            }
          }
          if (mup) {  // max|M_{k+1} - I|: integer max of |c| off the diagonal; the diagonal element kept
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int j = j0 + e + q;
              if (j < a.n && (!a.sym || j >= i)) {
                const double c = q ? c1 : c0;
                emax_bits = umax64(emax_bits, j == i ? 0ull : abs_bits(c));
                diag_bits = j == i ? (unsigned long long)__double_as_longlong(c) : diag_bits;
              }
            }
          }
        }
        // the one fp64 subtraction of the M-update, once per row of a diagonal tile
        if (mup && row_ok && i >= j0 + cb && i < j0 + cb + kEpiCols)
          emax_bits = umax64(emax_bits, abs_bits(__longlong_as_double((long long)diag_bits) - 1.0));
        if (a.sym && row_ok) {  // mirror: lanes are consecutive rows -> coalesced
#pragma unroll
          for (int e = cb; e < cb + kEpiCols; ++e) {
            const int j = j0 + e;
            if (j >= a.n || j <= i) continue;
#if OZ_PROBE == 7  // compute but no stores: one dependent store per lane keeps the values alive
            if (__double_as_longlong(v[e - cb]) == 0x7FF0000000000001ll) __stcs(out + (int64_t)j * a.np + i, v[e - cb]);
#else
            __stcs(out + (int64_t)j * a.np + i, v[e - cb]);
#endif
          }
        }
      }
      if (mup) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) emax_bits = umax64(emax_bits, __shfl_xor_sync(0xffffffffu, emax_bits, o));
        if (lane == 0)
          atomicMax(reinterpret_cast<unsigned long long*>(a.errh + (int64_t)mat * (a.max_iter + 1) + kcheck),
                    emax_bits);
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

template <int S, int BK>
inline size_t gemm_smem_bytes() { return 1024 + (size_t)Cfg<S, BK>::kStages * Cfg<S, BK>::kStageBytes + 512; }

}  // namespace oz
}  // namespace shp
