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
      *reinterpret_cast<double2*>(s + swc(row, c)) = r[q];
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
      // thread -> (m = t & 127, k = 8*(t >> 7) .. +7): per k, a warp reads 32
      // consecutive m (coalesced); the thread then owns 8 consecutive k of row m.
      const int m = m0 + (t & 127), kb = kt * kTileK + 8 * (t >> 7);
#pragma unroll
      for (int e = 0; e < 8; ++e) r[e] = (m < m_valid && kb + e < k_valid) ? __ldg(base + (int64_t)(kb + e) * ld + m) : 0.0f;
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
        // odd rows store their odd chunk first: the two rows of a quarter-warp then
        // cover disjoint chunk positions in each store instruction
        const int c0 = 2 * c4 + (row & 1), c1 = 2 * c4 + 1 - (row & 1);
        *reinterpret_cast<double2*>(s + swc(row, c0)) = (row & 1) ? hi : lo;
        *reinterpret_cast<double2*>(s + swc(row, c1)) = (row & 1) ? lo : hi;
      }
    } else {
      const int row = t & 127, cb = 4 * (t >> 7);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<double2*>(s + swc(row, cb + j)) = make_double2((double)r[2 * j], (double)r[2 * j + 1]);
    }
  }
};

// ------------------------------------------------------------------ compute
SHP_DEV void load_frags(double (&a)[8], double (&b)[4], const double* sA, const double* sB, int ra, int rb, int k) {
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) a[mt] = sA[swz(ra + mt * 8, k)];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) b[nt] = sB[swz(rb + nt * 8, k)];
}

// One 16-deep k tile: 4 k-groups x 32 DMMA per warp; the fragments of group
// g+1 are loaded while the DMMAs of group g issue (register double buffer).
SHP_DEV void mma_ktile(Acc& acc, const double* sA, const double* sB, int warp, int lane) {
  const int ra = (warp & 1) * 64 + (lane >> 2);
  const int rb = (warp >> 1) * 32 + (lane >> 2);
  double a[2][8], b[2][4];
  load_frags(a[0], b[0], sA, sB, ra, rb, lane & 3);
#pragma unroll
  for (int g = 0; g < kTileK / 4; ++g) {
    if (g + 1 < kTileK / 4) load_frags(a[(g + 1) & 1], b[(g + 1) & 1], sA, sB, ra, rb, 4 * (g + 1) + (lane & 3));
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma884(acc.c[mt][nt][0], acc.c[mt][nt][1], a[g & 1][mt], b[g & 1][nt]);
  }
}

// Full K loop for one output tile.  `smem` holds kGemmSmemDoubles doubles.
// All 256 threads must call it.  Ends with a __syncthreads (smem reusable).
template <class LA, class LB>
SHP_DEV void gemm_tile(Acc& acc, const LA& la, const LB& lb, int k_tiles, double* smem) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // stage s: A at smem + s*2*kTileElems, B right after it (offsets, not a pointer
  // array, so that the compiler keeps the shared address space: LDS, not LD)
  typename LA::Regs ra;
  typename LB::Regs rb;
  acc_zero(acc);
  la.load(0, ra);
  lb.load(0, rb);
  la.store(smem, ra);
  lb.store(smem + kTileElems, rb);
  __syncthreads();
  for (int kt = 0; kt < k_tiles; ++kt) {
    const int s = kt & 1;
    const bool more = kt + 1 < k_tiles;
    if (more) {
      la.load(kt + 1, ra);
      lb.load(kt + 1, rb);
    }
    const double* cur = smem + s * (2 * kTileElems);
    mma_ktile(acc, cur, cur + kTileElems, warp, lane);
    if (more) {
      double* nxt = smem + (s ^ 1) * (2 * kTileElems);
      la.store(nxt, ra);
      lb.store(nxt + kTileElems, rb);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------- cp.async fp64 pipeline
// For fp64 row panels (the Newton products).  A compact CTA: 64x64 output tile,
// 4 warps (2x2), warp tile 32x32 = 4x4 DMMA 8x8 tiles (64 accumulator
// registers), so that TWO CTAs fit on an SM (registers and 2 x 96 KB of shared
// memory) and one CTA's epilogue / pipeline fill / barrier overlaps the other
// CTA's DMMA stream.  Operands arrive by LDGSTS 16-byte copies straight into the
// swizzled tiles, a kStages-deep ring of 32-deep k tiles.  Rows are 256 B (a
// multiple of the 128-B bank window), so the same X(r) swizzle on the low 3
// chunk bits keeps fragment reads and copies conflict-free.
constexpr int kStages = 3;
constexpr int kAsyncK = 32;
constexpr int kNT = 64;                                     // Newton tile (square)
constexpr int kNThreads = 128;
constexpr int kAsyncTile = kNT * kAsyncK;                   // doubles per operand tile
constexpr int kAsyncSmemDoubles = kStages * 2 * kAsyncTile;  // 96 KB

struct AccN {
  double c[4][4][2];
};

SHP_DEV void accn_zero(AccN& a) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) a.c[i][j][0] = a.c[i][j][1] = 0.0;
}
SHP_DEV int accn_row(int warp, int lane, int mt) { return (warp & 1) * 32 + mt * 8 + (lane >> 2); }
SHP_DEV int accn_col(int warp, int lane, int nt, int e) { return (warp >> 1) * 32 + nt * 8 + 2 * (lane & 3) + e; }

SHP_DEV int swz32(int r, int k) { return r * kAsyncK + ((((k >> 1) ^ swx(r)) << 1) | (k & 1)); }

SHP_DEV void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
}
SHP_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
SHP_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

SHP_DEV void f64_issue(double* s, const double* base, int64_t ld, int kt) {
  const int t = threadIdx.x;
#pragma unroll
  for (int q = 0; q < kAsyncTile / 2 / kNThreads; ++q) {
    const int id = t + kNThreads * q, row = id >> 4, c = id & 15;
    cp_async16(s + row * kAsyncK + ((c ^ swx(row)) << 1), base + (int64_t)row * ld + kt * kAsyncK + 2 * c);
  }
}

SHP_DEV void load_fragsn(double (&a)[4], double (&b)[4], const double* sA, const double* sB, int ra, int rb, int k) {
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) a[mt] = sA[swz32(ra + mt * 8, k)];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) b[nt] = sB[swz32(rb + nt * 8, k)];
}

SHP_DEV void mma_ktilen(AccN& acc, const double* sA, const double* sB, int warp, int lane) {
  const int ra = (warp & 1) * 32 + (lane >> 2);
  const int rb = (warp >> 1) * 32 + (lane >> 2);
  double a[2][4], b[2][4];
  load_fragsn(a[0], b[0], sA, sB, ra, rb, lane & 3);
#pragma unroll
  for (int g = 0; g < kAsyncK / 4; ++g) {
    if (g + 1 < kAsyncK / 4) load_fragsn(a[(g + 1) & 1], b[(g + 1) & 1], sA, sB, ra, rb, 4 * (g + 1) + (lane & 3));
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma884(acc.c[mt][nt][0], acc.c[mt][nt][1], a[g & 1][mt], b[g & 1][nt]);
  }
}

// C = A_panel . B_panel^T over K = 32 * k_tiles for a 64x64 tile; both operands
// fp64 row panels (64 rows from A and B).  `smem` holds kAsyncSmemDoubles doubles.
// All kNThreads threads call it; ends with __syncthreads.
SHP_DEV void gemm_tile_f64(AccN& acc, const double* A, const double* B, int64_t ld, int k_tiles, double* smem) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  accn_zero(acc);
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < k_tiles) {
      f64_issue(smem + st * 2 * kAsyncTile, A, ld, st);
      f64_issue(smem + st * 2 * kAsyncTile + kAsyncTile, B, ld, st);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < k_tiles; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();  // stage kt visible to all; stage kt-1 fully consumed
    const int nk = kt + kStages - 1;
    if (nk < k_tiles) {
      double* s = smem + (nk % kStages) * 2 * kAsyncTile;
      f64_issue(s, A, ld, nk);
      f64_issue(s + kAsyncTile, B, ld, nk);
    }
    cp_async_commit();
    const double* cur = smem + (kt % kStages) * 2 * kAsyncTile;
    mma_ktilen(acc, cur, cur + kAsyncTile, warp, lane);
  }
  cp_async_wait<0>();
  __syncthreads();
}

// fp32 panel for the compact (64-row, 32-deep) tiles, register-staged and
// widened to fp64 on the way into shared memory; bounds-masked (zero fill).
// kmaj == 0: A_m[k] = src[m][k] (row panel); kmaj == 1: A_m[k] = src[k][m].
struct F32PanelN {
  const float* base;
  int64_t ld;
  int kmaj;
  int m0, m_valid, k_valid;
  using Regs = float[16];
  SHP_DEV void load(int kt, Regs& r) const {
    const int t = threadIdx.x;
    if (!kmaj) {
      // thread -> (row = t >> 1, 16 consecutive k at 16*(t & 1)): a warp reads 16 rows x 64 B
      const int m = m0 + (t >> 1), kb = kt * kAsyncK + 16 * (t & 1);
      const float* src = base + (int64_t)m * ld + kb;
#pragma unroll
      for (int e = 0; e < 16; ++e) r[e] = (m < m_valid && kb + e < k_valid) ? __ldg(src + e) : 0.0f;
    } else {
      // thread -> (m = t & 63, 16 consecutive k at 16*(t >> 6)): per k, 64 consecutive m
      const int m = m0 + (t & 63), kb = kt * kAsyncK + 16 * (t >> 6);
#pragma unroll
      for (int e = 0; e < 16; ++e) r[e] = (m < m_valid && kb + e < k_valid) ? __ldg(base + (int64_t)(kb + e) * ld + m) : 0.0f;
    }
  }
  SHP_DEV void store(double* s, const Regs& r) const {
    const int t = threadIdx.x;
    const int row = kmaj ? (t & 63) : (t >> 1);
    const int cb = kmaj ? 8 * (t >> 6) : 8 * (t & 1);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<double2*>(s + row * kAsyncK + (((cb + j) ^ swx(row)) << 1)) =
          make_double2((double)r[2 * j], (double)r[2 * j + 1]);
  }
};

// 64x64 tile over K = 32 * k_tiles from two fp32 panels (2-stage register-staged
// double buffer: global loads of k tile t+1 are in flight during the DMMAs of t).
// `smem` holds 2 * 2 * kAsyncTile doubles (64 KB).  Ends with __syncthreads.
SHP_DEV void gemm_tile_f32n(AccN& acc, const F32PanelN& la, const F32PanelN& lb, int k_tiles, double* smem) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  F32PanelN::Regs ra, rb;
  accn_zero(acc);
  la.load(0, ra);
  lb.load(0, rb);
  la.store(smem, ra);
  lb.store(smem + kAsyncTile, rb);
  __syncthreads();
  for (int kt = 0; kt < k_tiles; ++kt) {
    const int s = kt & 1;
    const bool more = kt + 1 < k_tiles;
    if (more) {
      la.load(kt + 1, ra);
      lb.load(kt + 1, rb);
    }
    const double* cur = smem + s * (2 * kAsyncTile);
    mma_ktilen(acc, cur, cur + kAsyncTile, warp, lane);
    if (more) {
      double* nxt = smem + (s ^ 1) * (2 * kAsyncTile);
      la.store(nxt, ra);
      lb.store(nxt + kAsyncTile, rb);
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
