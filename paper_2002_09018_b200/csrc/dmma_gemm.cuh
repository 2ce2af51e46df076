// dmma_gemm.cuh -- 128x128 output-tile GEMM core on the FP64 tensor pipe (DMMA).
//
// C[i][j] = sum_k A_i[k] * B_j[k]  for a 128x128 tile, k ascending, fp64.
// Both operands are presented to the core as "panels": A_i[k] is row i of the
// left operand, B_j[k] is column j of the right operand.  For the symmetric
// operands of the Newton iteration and of the statistics this means both are
// row panels of a stored matrix (B[k][j] = B[j][k]).
//
// CTA = 256 threads = 8 warps, warp tile 64 (M) x 32 (N) = 8 x 4 DMMA 8x8 tiles,
// k tile 16, double-buffered shared memory (2 x 32 KB) filled through registers
// (global loads of k-tile t+1 are in flight while k-tile t is multiplied).
//
// Order of accumulation: every output element sees k = 0, 1, 2, ... in order
// (DMMA.8x8x4 chains k inside an instruction, the k loop chains instructions),
// which is exactly the sequential contract of the statistics.
#pragma once
#include "common.cuh"

namespace shp {

constexpr int kThreads = 256;
constexpr int kGemmSmemDoubles = 2 * 2 * kTileElems;  // 2 stages x (A, B)

struct Acc {
  double c[8][4][2];
};

SHP_DEV void acc_zero(Acc& a) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) a.c[i][j][0] = a.c[i][j][1] = 0.0;
}

// Output coordinates of accumulator (mt, nt, e) for this lane, inside the tile.
SHP_DEV int acc_row(int warp, int lane, int mt) { return (warp & 1) * 64 + mt * 8 + (lane >> 2); }
SHP_DEV int acc_col(int warp, int lane, int nt, int e) { return (warp >> 1) * 32 + nt * 8 + 2 * (lane & 3) + e; }

// ------------------------------------------------------------------ loaders
// fp64 row panel of a padded matrix (no masking: rows/k always in range).
struct F64Rows {
  const double* base;  // &M[m0][0]
  int64_t ld;
  using Regs = double2[4];
  SHP_DEV void load(int kt, Regs& r) const {
    const int t = threadIdx.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int id = t + kThreads * q, row = id >> 3, c = id & 7;
      r[q] = __ldg(reinterpret_cast<const double2*>(base + (int64_t)row * ld + kt * kTileK + 2 * c));
    }
  }
  SHP_DEV void store(double* s, const Regs& r) const {
    const int t = threadIdx.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int id = t + kThreads * q, row = id >> 3, c = id & 7;
      *reinterpret_cast<double2*>(s + row * kTileK + ((c ^ (row & 7)) << 1)) = r[q];
    }
  }
};

// fp32 panel with bounds.  kmaj == 0: source row = panel index m, contiguous k
// (A_m[k] = src[m][k]); kmaj == 1: source row = k, contiguous m (A_m[k] = src[k][m]).
// Elements with m >= m_valid or k >= k_valid read as 0.
struct F32Panel {
  const float* base;  // &src[origin]
  int64_t ld;
  int kmaj;
  int m0;  // first panel index of this tile
  int m_valid, k_valid;
  using Regs = float[8];
  SHP_DEV void load(int kt, Regs& r) const {
    const int t = threadIdx.x;
    if (!kmaj) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        int id = t + kThreads * q, row = id >> 2, c4 = id & 3;
        int m = m0 + row, k = kt * kTileK + 4 * c4;
        const float* src = base + (int64_t)m * ld + k;
#pragma unroll
        for (int e = 0; e < 4; ++e) r[4 * q + e] = (m < m_valid && k + e < k_valid) ? __ldg(src + e) : 0.0f;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        int id = t + kThreads * q, kk = id >> 5, c = id & 31;
        int k = kt * kTileK + kk, m = m0 + 4 * c;
        const float* src = base + (int64_t)k * ld + m;
#pragma unroll
        for (int e = 0; e < 4; ++e) r[4 * q + e] = (k < k_valid && m + e < m_valid) ? __ldg(src + e) : 0.0f;
      }
    }
  }
  SHP_DEV void store(double* s, const Regs& r) const {
    const int t = threadIdx.x;
    if (!kmaj) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        int id = t + kThreads * q, row = id >> 2, c4 = id & 3;
        double2 lo = make_double2((double)r[4 * q + 0], (double)r[4 * q + 1]);
        double2 hi = make_double2((double)r[4 * q + 2], (double)r[4 * q + 3]);
        *reinterpret_cast<double2*>(s + row * kTileK + (((2 * c4) ^ (row & 7)) << 1)) = lo;
        *reinterpret_cast<double2*>(s + row * kTileK + (((2 * c4 + 1) ^ (row & 7)) << 1)) = hi;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        int id = t + kThreads * q, kk = id >> 5, c = id & 31;
#pragma unroll
        for (int e = 0; e < 4; ++e) s[swz(4 * c + e, kk)] = (double)r[4 * q + e];
      }
    }
  }
};

// ------------------------------------------------------------------ compute
SHP_DEV void mma_ktile(Acc& acc, const double* sA, const double* sB, int warp, int lane) {
  const int ra = (warp & 1) * 64 + (lane >> 2);
  const int rb = (warp >> 1) * 32 + (lane >> 2);
#pragma unroll
  for (int g = 0; g < kTileK / 4; ++g) {
    const int k = 4 * g + (lane & 3);
    double a[8], b[4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) a[mt] = sA[swz(ra + mt * 8, k)];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) b[nt] = sB[swz(rb + nt * 8, k)];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma884(acc.c[mt][nt][0], acc.c[mt][nt][1], a[mt], b[nt]);
  }
}

// Full K loop for one output tile.  `smem` holds kGemmSmemDoubles doubles.
// All 256 threads must call it.  Ends with a __syncthreads (smem reusable).
template <class LA, class LB>
SHP_DEV void gemm_tile(Acc& acc, const LA& la, const LB& lb, int k_tiles, double* smem) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sA[2] = {smem, smem + 2 * kTileElems};
  double* sB[2] = {smem + kTileElems, smem + 3 * kTileElems};
  typename LA::Regs ra;
  typename LB::Regs rb;
  acc_zero(acc);
  la.load(0, ra);
  lb.load(0, rb);
  la.store(sA[0], ra);
  lb.store(sB[0], rb);
  __syncthreads();
  for (int kt = 0; kt < k_tiles; ++kt) {
    const int s = kt & 1;
    const bool more = kt + 1 < k_tiles;
    if (more) {
      la.load(kt + 1, ra);
      lb.load(kt + 1, rb);
    }
    mma_ktile(acc, sA[s], sB[s], warp, lane);
    if (more) {
      la.store(sA[s ^ 1], ra);
      lb.store(sB[s ^ 1], rb);
    }
    __syncthreads();
  }
}

// Upper-triangular tile index t -> (ti, tj), ti <= tj, row-major over the
// upper triangle of a T x T tile grid.
SHP_DEV void upper_tile(int t, int T, int& ti, int& tj) {
  int i = 0;
  while (t >= T - i) {
    t -= T - i;
    ++i;
  }
  ti = i;
  tj = i + t;
}

}  // namespace shp
