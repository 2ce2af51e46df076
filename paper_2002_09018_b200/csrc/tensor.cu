// tensor.cu -- f3: Shampoo statistics and preconditioned gradient for tensors of
// order 1..4 (the method "holds for tensors of arbitrary order", P:113-116,
// P:132; readings #24-#26 of DESIGN.md; oracle/tensor.py).
//
// Statistics (one call per step, all blocks of all tensors):
//   check (non-finite per block) -> widen (mode-i unfoldings of owned blocks to
//   fp64 panels, e_i x roundup(K_i, 32), zero-padded in k) -> mode statistics
//   per 4096-column chunk: FP64 DMMA 64x64 tiles (modes > 32) or fp64 FMA
//   chains (modes <= 32) -> finish (chunk sums in ascending order + the EMA
//   epilogue, bit-exact with the oracle's chunked sequential contract)
//   -> diag (D and graft partials) -> diag finish.
// Preconditioning:
//   gather (block -> dense fp32) -> one stage per mode m = 0..3 (mode products
//   Y <- X_m x_m Y: FP64 DMMA tiles through the fp32 register-staged compact
//   core for modes > 32, fp64 FMA fibres for small modes) -> scatter into P +
//   den partials (diag-only blocks: D^{-1/2} o G) -> finish (graft scale).
// Job tables are derived from the HOST tables on every call and uploaded into
// the workspace with one cudaMemcpyAsync (the library stays stateless).
#include <algorithm>
#include <cstring>
#include <vector>

#include "dmma_gemm.cuh"
#include "internal.h"

namespace shp {

constexpr int KO = SHAMPOO_MAX_ORDER;
constexpr int kStatChunk = 4096;  // reading #25 (multiple of kAsyncK)
constexpr int kSmallMode = 32;    // modes <= 32 take the FMA paths
constexpr int kTChunks = 64;      // elementwise chunks per block
constexpr int kSmallThreads = 256;
constexpr int kSubK = 128;        // k columns staged per pass in the small-mode statistics kernel

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
static int64_t rup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct TBlk {  // one block: tensor pointers, origin offset, strides, extents
  const float* G;
  float* D;
  float* P;
  int64_t base;
  int64_t st[KO];
  int32_t ext[KO];
  int64_t numel;
  int64_t y0, y1;  // precondition: dense fp32 buffers (offsets in floats), -1 if unused
  int32_t fin;     // precondition: buffer holding the result (0 -> y0, 1 -> y1), -1 = diag-only
  int32_t pad;
};

struct TStatJob {  // one owned mode statistic
  int64_t K, kp, panel, part, soff;
  int64_t mst;      // stride of the mode
  int64_t ost[3];   // strides of the other modes (leading pads: 0)
  int32_t oext[3];  // extents of the other modes, row-major order (leading pads: 1)
  int32_t blk, e, nchunks, ld;
};

struct TItem {
  int32_t job, a, b, c;
};

struct TModeJob {  // one mode product of one block
  int64_t in, out;  // dense buffers (float offsets)
  int64_t xoff;     // root offset
  int64_t Pb, Sb;
  int32_t ld, e, blk, kind;  // kind 0: FMA fibres; 1: DMMA, Sb == 1; 2: DMMA, Sb > 1
};

SHP_DEV int64_t toff(const TBlk& b, int64_t f) {  // block-local flat index -> tensor offset
  int64_t o = b.base;
#pragma unroll
  for (int i = KO - 1; i >= 0; --i) {
    const int64_t e = b.ext[i];
    const int64_t q = f / e;
    o += (f - q * e) * b.st[i];
    f = q;
  }
  return o;
}

// ------------------------------------------------------------ statistics
__global__ void __launch_bounds__(256) t_check_kernel(const TBlk* blks, int* flag) {
  const int b = blockIdx.x / kTChunks, c = blockIdx.x % kTChunks;
  const TBlk k = blks[b];
  const int64_t per = (k.numel + kTChunks - 1) / kTChunks;
  const int64_t f0 = c * per, f1 = min(k.numel, f0 + per);
  int bad = 0;
  for (int64_t f = f0 + threadIdx.x; f < f1; f += blockDim.x) bad |= !isfinite(__ldg(k.G + toff(k, f)));
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag + b, 1);
}

// panel[a][k] = U_i[a][k] (fp64), zero for k >= K.  grid.y = job.
__global__ void __launch_bounds__(256) t_widen_kernel(const TStatJob* jobs, const TBlk* blks, const int* flag,
                                                      double* wide) {
  const TStatJob j = jobs[blockIdx.y];
  if (flag[j.blk]) return;
  const TBlk k = blks[j.blk];
  const int64_t total = (int64_t)j.e * j.kp;
  const int e1 = j.oext[1], e2 = j.oext[2];
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = idx / j.kp, kk = idx - a * j.kp;
    double v = 0.0;
    if (kk < j.K) {
      const int64_t q = kk / e2, k2 = kk - q * e2;
      const int64_t k0 = q / e1, k1 = q - k0 * e1;
      v = (double)__ldg(k.G + k.base + a * j.mst + k0 * j.ost[0] + k1 * j.ost[1] + k2 * j.ost[2]);
    }
    wide[j.panel + idx] = v;
  }
}

// cp.async of a 64-row fp64 k tile; rows >= rows_valid are zero-filled (src-size 0)
SHP_DEV void f64_issue_rows(double* s, const double* base, int64_t ld, int kt, int rows_valid) {
  const int t = threadIdx.x;
#pragma unroll
  for (int q = 0; q < kAsyncTile / 2 / kNThreads; ++q) {
    const int id = t + kNThreads * q, row = id >> 4, c = id & 15;
    const bool v = row < rows_valid;
    const double* src = v ? base + (int64_t)row * ld + kt * kAsyncK + 2 * c : base;
    const unsigned d = (unsigned)__cvta_generic_to_shared(s + row * kAsyncK + ((c ^ swx(row)) << 1));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(v ? 16 : 0));
  }
}

SHP_DEV void gemm_tile_f64_rows(AccN& acc, const double* A, const double* B, int64_t ld, int k_tiles, int ra,
                                int rb, double* smem) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  accn_zero(acc);
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < k_tiles) {
      f64_issue_rows(smem + st * 2 * kAsyncTile, A, ld, st, ra);
      f64_issue_rows(smem + st * 2 * kAsyncTile + kAsyncTile, B, ld, st, rb);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < k_tiles; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nk = kt + kStages - 1;
    if (nk < k_tiles) {
      double* s = smem + (nk % kStages) * 2 * kAsyncTile;
      f64_issue_rows(s, A, ld, nk, ra);
      f64_issue_rows(s + kAsyncTile, B, ld, nk, rb);
    }
    cp_async_commit();
    const double* cur = smem + (kt % kStages) * 2 * kAsyncTile;
    mma_ktilen(acc, cur, cur + kAsyncTile, warp, lane);
  }
  cp_async_wait<0>();
  __syncthreads();
}

// modes > 32: one (job, 64x64 upper tile (a, b), chunk c) per item; DMMA chains
// the chunk's k in ascending order from 0 (the chunk sum of the contract)
__global__ void __launch_bounds__(kNThreads, 2)
    t_stats_tile_kernel(const TStatJob* jobs, const TItem* items, int n_items, const int* flag, const double* wide,
                        double* part) {
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  AccN acc;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const TItem m = items[it];
    const TStatJob j = jobs[m.job];
    if (flag[j.blk]) continue;
    const int64_t k0 = (int64_t)m.c * kStatChunk;
    const int kt = (int)((min((int64_t)kStatChunk, j.kp - k0)) / kAsyncK);
    const double* P = wide + j.panel;
    gemm_tile_f64_rows(acc, P + (int64_t)m.a * kNT * j.kp + k0, P + (int64_t)m.b * kNT * j.kp + k0, j.kp, kt,
                       j.e - m.a * kNT, j.e - m.b * kNT, smem);
    double* dst = part + j.part + (int64_t)m.c * j.e * j.e;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int i = m.a * kNT + accn_row(warp, lane, mt);
      if (i >= j.e) continue;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jj = m.b * kNT + accn_col(warp, lane, nt, e);
          if (jj < j.e) dst[(int64_t)i * j.e + jj] = acc.c[mt][nt][e];
        }
    }
  }
}

// modes <= 32: one (job, chunk) per item; each thread owns up to 3 upper
// outputs (a <= b) and chains fma over the chunk's k in ascending order
__global__ void __launch_bounds__(kSmallThreads) t_stats_small_kernel(const TStatJob* jobs, const TItem* items,
                                                                     const int* flag, const double* wide,
                                                                     double* part) {
  __shared__ double s[kSmallMode][kSubK + 1];
  const TItem m = items[blockIdx.x];
  const TStatJob j = jobs[m.job];
  if (flag[j.blk]) return;
  const int e = j.e, nout = e * (e + 1) / 2;
  int oa[3], ob[3];
  double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    int o = threadIdx.x + q * kSmallThreads, a = 0;
    if (o >= nout) {
      oa[q] = -1;
      ob[q] = 0;
      continue;
    }
    while (o >= e - a) {  // upper-triangle row-major: row a holds e - a entries
      o -= e - a;
      ++a;
    }
    oa[q] = a;
    ob[q] = a + o;
  }
  const int64_t k0 = (int64_t)m.c * kStatChunk, k1 = min(j.kp, k0 + kStatChunk);
  const double* P = wide + j.panel;
  for (int64_t kb = k0; kb < k1; kb += kSubK) {
    const int w = (int)min((int64_t)kSubK, k1 - kb);
    __syncthreads();
    for (int idx = threadIdx.x; idx < e * kSubK; idx += kSmallThreads) {
      const int a = idx / kSubK, kk = idx - a * kSubK;
      s[a][kk] = kk < w ? P[(int64_t)a * j.kp + kb + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (oa[q] < 0) continue;
      const double* ra = s[oa[q]];
      const double* rb = s[ob[q]];
      double t = acc[q];
      for (int kk = 0; kk < w; ++kk) t = fma(ra[kk], rb[kk], t);
      acc[q] = t;
    }
  }
  double* dst = part + j.part + (int64_t)m.c * e * e;
#pragma unroll
  for (int q = 0; q < 3; ++q)
    if (oa[q] >= 0) dst[oa[q] * e + ob[q]] = acc[q];
}

// acc = sum over chunks (ascending) of the chunk sums; EMA epilogue; mirror
__global__ void __launch_bounds__(256) t_stats_finish_kernel(const TStatJob* jobs, const int* flag,
                                                             const double* part, float* stats, double decay,
                                                             double weight) {
  const TStatJob j = jobs[blockIdx.y];
  if (flag[j.blk]) return;
  const int e = j.e;
  float* S = stats + j.soff;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < e * e; idx += gridDim.x * blockDim.x) {
    const int a = idx / e, b = idx - a * e;
    if (a > b) continue;
    double acc = 0.0;
    for (int c = 0; c < j.nchunks; ++c) acc = __dadd_rn(acc, part[j.part + (int64_t)c * e * e + idx]);
    const double t1 = __dmul_rn(weight, acc);
    const double t2 = __dmul_rn(decay, (double)S[(int64_t)a * j.ld + b]);
    const float r = __double2float_rn(__dadd_rn(t1, t2));
    S[(int64_t)a * j.ld + b] = r;
    if (a != b) S[(int64_t)b * j.ld + a] = r;
  }
}

// D <- D + G o G and graft partials per (block, chunk), fixed order
__global__ void __launch_bounds__(256) t_diag_kernel(const TBlk* blks, const int* flag, double* part) {
  const int b = blockIdx.x / kTChunks, c = blockIdx.x % kTChunks;
  __shared__ double red[8];
  const TBlk k = blks[b];
  const int64_t per = (k.numel + kTChunks - 1) / kTChunks;
  const int64_t f0 = c * per, f1 = min(k.numel, f0 + per);
  double num = 0.0;
  if (!flag[b] && k.D != nullptr) {
    for (int64_t f = f0 + threadIdx.x; f < f1; f += blockDim.x) {
      const int64_t o = toff(k, f);
      const double g = (double)__ldg(k.G + o);
      const double gg = __dmul_rn(g, g);
      const float dn = __double2float_rn(__dadd_rn((double)k.D[o], gg));
      k.D[o] = dn;
      const double den = (double)dn > 1e-30 ? (double)dn : 1e-30;
      num = __dadd_rn(num, __ddiv_rn(gg, den));
    }
  }
  num = warp_sum_fixed(num);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = num;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s = __dadd_rn(s, red[w]);
    part[(int64_t)b * kTChunks + c] = s;
  }
}

__global__ void t_diag_finish_kernel(int n_blocks, const int* flag, const double* part, double* graft_num,
                                     int32_t* block_status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  double s = 0.0;
  for (int c = 0; c < kTChunks; ++c) s = __dadd_rn(s, part[(int64_t)b * kTChunks + c]);
  if (graft_num) graft_num[b] = flag[b] ? 0.0 : s;
  if (block_status) block_status[b] = flag[b] ? 2 : 0;
}

// ------------------------------------------------------------ preconditioning
__global__ void __launch_bounds__(256) t_gather_kernel(const TBlk* blks, float* Y) {
  const int b = blockIdx.x / kTChunks, c = blockIdx.x % kTChunks;
  const TBlk k = blks[b];
  if (k.fin < 0) return;
  const int64_t per = (k.numel + kTChunks - 1) / kTChunks;
  const int64_t f0 = c * per, f1 = min(k.numel, f0 + per);
  for (int64_t f = f0 + threadIdx.x; f < f1; f += blockDim.x) Y[k.y0 + f] = __ldg(k.G + toff(k, f));
}

// small modes: one thread per fibre (pb, s): out[pb, a, s] = sum_c X[a][c] in[pb, c, s]
__global__ void __launch_bounds__(kSmallThreads) t_mode_small_kernel(const TModeJob* jobs, const TItem* items,
                                                                    const float* roots, float* Y) {
  __shared__ double X[kSmallMode][kSmallMode + 1];
  const TItem m = items[blockIdx.x];
  const TModeJob j = jobs[m.job];
  const int e = j.e;
  for (int idx = threadIdx.x; idx < e * e; idx += kSmallThreads) {
    const int a = idx / e, c = idx - a * e;
    X[a][c] = (double)roots[j.xoff + (int64_t)a * j.ld + c];
  }
  __syncthreads();
  const int64_t f = (int64_t)m.a * kSmallThreads + threadIdx.x;
  if (f >= j.Pb * j.Sb) return;
  const int64_t pb = f / j.Sb, s = f - pb * j.Sb;
  const float* in = Y + j.in + pb * e * j.Sb + s;
  float* out = Y + j.out + pb * e * j.Sb + s;
  double v[kSmallMode];
#pragma unroll
  for (int c = 0; c < kSmallMode; ++c) v[c] = c < e ? (double)in[(int64_t)c * j.Sb] : 0.0;
  for (int a = 0; a < e; ++a) {
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < kSmallMode; ++c)
      if (c < e) t = fma(X[a][c], v[c], t);
    out[(int64_t)a * j.Sb] = (float)t;
  }
}

// large modes: 64x64 DMMA tiles (fp32 panels widened in registers)
//   kind 1 (Sb == 1): out[pb][a] = sum_c in[pb][c] X[a][c]   tile (pb-tile a, a-tile b)
//   kind 2 (Sb > 1):  out[pb][a][s] = sum_c X[a][c] in[pb][c][s]   (pb = c field, a-tile a, s-tile b)
__global__ void __launch_bounds__(kNThreads, 2) t_mode_tile_kernel(const TModeJob* jobs, const TItem* items,
                                                                   int n_items, const float* roots, float* Y) {
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  AccN acc;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const TItem m = items[it];
    const TModeJob j = jobs[m.job];
    const float* X = roots + j.xoff;
    const int kt = (j.e + kAsyncK - 1) / kAsyncK;
    int rows, cols;
    int64_t ldo;
    float* out;
    if (j.kind == 1) {
      F32PanelN la{Y + j.in, (int64_t)j.e, 0, m.a * kNT, (int)j.Pb, j.e};
      F32PanelN lb{X, (int64_t)j.ld, 0, m.b * kNT, j.e, j.e};
      gemm_tile_f32n(acc, la, lb, kt, smem);
      rows = (int)j.Pb;
      cols = j.e;
      ldo = j.e;
      out = Y + j.out;
    } else {
      const int64_t pb = m.c;
      F32PanelN la{X, (int64_t)j.ld, 0, m.a * kNT, j.e, j.e};
      F32PanelN lb{Y + j.in + pb * j.e * j.Sb, j.Sb, 1, m.b * kNT, (int)j.Sb, j.e};
      gemm_tile_f32n(acc, la, lb, kt, smem);
      rows = j.e;
      cols = (int)j.Sb;
      ldo = j.Sb;
      out = Y + j.out + pb * j.e * j.Sb;
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int i = m.a * kNT + accn_row(warp, lane, mt);
      if (i >= rows) continue;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = m.b * kNT + accn_col(warp, lane, nt, e);
          if (c < cols) out[(int64_t)i * ldo + c] = (float)acc.c[mt][nt][e];
        }
    }
  }
}

// P_B <- result (or D^{-1/2} o G for diag-only blocks); den partials
__global__ void __launch_bounds__(256) t_scatter_kernel(const TBlk* blks, const float* Y, double* part) {
  const int b = blockIdx.x / kTChunks, c = blockIdx.x % kTChunks;
  __shared__ double red[8];
  const TBlk k = blks[b];
  const int64_t per = (k.numel + kTChunks - 1) / kTChunks;
  const int64_t f0 = c * per, f1 = min(k.numel, f0 + per);
  double s = 0.0;
  for (int64_t f = f0 + threadIdx.x; f < f1; f += blockDim.x) {
    const int64_t o = toff(k, f);
    float pv;
    if (k.fin < 0) {
      double dv = (double)k.D[o];
      dv = dv > 1e-30 ? dv : 1e-30;
      pv = (float)((double)__ldg(k.G + o) / sqrt(dv));
    } else {
      pv = Y[(k.fin ? k.y1 : k.y0) + f];
    }
    k.P[o] = pv;
    s = fma((double)pv, (double)pv, s);
  }
  s = warp_sum_fixed(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t = __dadd_rn(t, red[w]);
    part[(int64_t)b * kTChunks + c] = t;
  }
}

__global__ void t_prec_finish_kernel(int n_blocks, const double* part, const double* graft_num, float* graft_scale,
                                     double* den) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  double s = 0.0;
  for (int c = 0; c < kTChunks; ++c) s = __dadd_rn(s, part[(int64_t)b * kTChunks + c]);
  if (den) den[b] = s;
  if (graft_scale) {
    float sc = 0.0f;
    if (graft_num && s > 0.0) sc = (float)(sqrt(graft_num[b]) / sqrt(s));
    graft_scale[b] = sc;
  }
}

// ---------------------------------------------------------------- host side
template <class T>
static size_t put(std::vector<uint8_t>& blob, const T* p, size_t n) {
  const size_t off = al(blob.size());
  blob.resize(off + n * sizeof(T));
  if (n) std::memcpy(blob.data() + off, p, n * sizeof(T));
  return off;
}

static void strides_of(const shampoo_ttensor_t& t, int64_t* st) {
  int64_t s = 1;
  for (int i = KO - 1; i >= 0; --i) {
    st[i] = (i < t.order) ? s : 0;
    if (i < t.order) s *= t.dims[i];
  }
}

static TBlk make_blk(const shampoo_ttensor_t& t, const shampoo_tblock_t& b) {
  TBlk k;
  std::memset(&k, 0, sizeof k);
  k.G = t.G;
  k.D = t.D;
  k.P = t.P;
  strides_of(t, k.st);
  k.base = 0;
  k.numel = 1;
  for (int i = 0; i < KO; ++i) {
    k.ext[i] = i < b.order ? b.extent[i] : 1;
    k.base += (i < b.order ? b.origin[i] : 0) * k.st[i];
    k.numel *= k.ext[i];
  }
  k.y0 = k.y1 = -1;
  k.fin = -1;
  return k;
}

struct TStatsLayout {
  std::vector<uint8_t> blob;
  size_t off_blk = 0, off_jobs = 0, off_small = 0, off_tiles = 0;
  int n_jobs = 0, n_small = 0, n_tiles = 0;
  int64_t max_panel = 0;
  size_t off_flag = 0, off_part2 = 0, off_part = 0, off_wide = 0, total = 0;
};

static void stats_layout(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks, int only_owner,
                         TStatsLayout& L) {
  std::vector<TBlk> blks(n_blocks);
  std::vector<TStatJob> jobs;
  std::vector<TItem> small, tiles;
  int64_t wide = 0, part = 0;
  for (int b = 0; b < n_blocks; ++b) {
    const shampoo_tblock_t& bk = B[b];
    blks[b] = make_blk(T[bk.tensor_id], bk);
    for (int i = 0; i < bk.order; ++i) {
      if (!bk.p[i] || !(only_owner < 0 || bk.owner[i] == only_owner)) continue;
      TStatJob j;
      std::memset(&j, 0, sizeof j);
      j.blk = b;
      j.e = bk.extent[i];
      j.K = blks[b].numel / j.e;
      j.kp = rup(j.K, kAsyncK);
      j.nchunks = (int)((j.kp + kStatChunk - 1) / kStatChunk);
      j.mst = blks[b].st[i];
      int q = 3;
      for (int l = 0; l < 3; ++l) {
        j.oext[l] = 1;
        j.ost[l] = 0;
      }
      for (int l = bk.order - 1; l >= 0; --l)  // the other modes, packed to the right (row-major)
        if (l != i) {
          --q;
          j.oext[q] = bk.extent[l];
          j.ost[q] = blks[b].st[l];
        }
      j.panel = wide;
      wide += (int64_t)j.e * j.kp;
      j.part = part;
      part += (int64_t)j.nchunks * j.e * j.e;
      j.soff = bk.off[i];
      j.ld = bk.ld[i];
      const int jid = (int)jobs.size();
      jobs.push_back(j);
      if (j.e <= kSmallMode) {
        for (int c = 0; c < j.nchunks; ++c) small.push_back({jid, 0, 0, c});
      } else {
        const int Tn = (j.e + kNT - 1) / kNT;
        for (int c = 0; c < j.nchunks; ++c)
          for (int a = 0; a < Tn; ++a)
            for (int bb = a; bb < Tn; ++bb) tiles.push_back({jid, a, bb, c});
      }
      L.max_panel = std::max(L.max_panel, (int64_t)j.e * j.kp);
    }
  }
  L.blob.clear();
  L.off_blk = put(L.blob, blks.data(), blks.size());
  L.off_jobs = put(L.blob, jobs.data(), jobs.size());
  L.off_small = put(L.blob, small.data(), small.size());
  L.off_tiles = put(L.blob, tiles.data(), tiles.size());
  L.n_jobs = (int)jobs.size();
  L.n_small = (int)small.size();
  L.n_tiles = (int)tiles.size();
  size_t q = al(L.blob.size());
  L.off_flag = q;
  q = al(q + (size_t)n_blocks * sizeof(int));
  L.off_part2 = q;
  q = al(q + (size_t)n_blocks * kTChunks * sizeof(double));
  L.off_part = q;
  q = al(q + (size_t)part * sizeof(double));
  L.off_wide = q;
  q = al(q + (size_t)wide * sizeof(double));
  L.total = q;
}

size_t tensor_stats_workspace_bytes(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks,
                                    int only_owner) {
  TStatsLayout L;
  stats_layout(T, B, n_blocks, only_owner, L);
  return L.total;
}

int tensor_stats_launch(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks, int only_owner,
                        float* stats, double decay, double weight, double* graft_num, int32_t* block_status,
                        void* ws, size_t ws_bytes, cudaStream_t stream, int64_t* launches) {
  if (n_blocks == 0) return SHAMPOO_OK;
  TStatsLayout L;
  stats_layout(T, B, n_blocks, only_owner, L);
  if (ws_bytes < L.total)
    return set_error(SHAMPOO_ERR_WORKSPACE, "tensor stats workspace: have %zu bytes, need %zu", ws_bytes, L.total);
  char* w = static_cast<char*>(ws);
  if (cudaMemcpyAsync(w, L.blob.data(), L.blob.size(), cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return set_cuda_error("cudaMemcpyAsync(tensor stats tables)");
  const TBlk* blks = reinterpret_cast<const TBlk*>(w + L.off_blk);
  const TStatJob* jobs = reinterpret_cast<const TStatJob*>(w + L.off_jobs);
  int* flag = reinterpret_cast<int*>(w + L.off_flag);
  double* part2 = reinterpret_cast<double*>(w + L.off_part2);
  double* part = reinterpret_cast<double*>(w + L.off_part);
  double* wide = reinterpret_cast<double*>(w + L.off_wide);
  if (cudaMemsetAsync(flag, 0, (size_t)n_blocks * sizeof(int), stream) != cudaSuccess)
    return set_cuda_error("cudaMemsetAsync");
  const unsigned eg = (unsigned)n_blocks * kTChunks;
  t_check_kernel<<<eg, 256, 0, stream>>>(blks, flag);
  ++*launches;
  if (L.n_jobs) {
    const unsigned gx = (unsigned)std::min<int64_t>(1024, (L.max_panel + 255) / 256);
    t_widen_kernel<<<dim3(gx, L.n_jobs), 256, 0, stream>>>(jobs, blks, flag, wide);
    ++*launches;
    if (L.n_tiles) {
      const size_t smem = (size_t)kAsyncSmemDoubles * sizeof(double);
      if (ensure_smem((const void*)t_stats_tile_kernel, smem) !=
          cudaSuccess)
        return set_cuda_error("cudaFuncSetAttribute(t_stats_tile_kernel)");
      const int grid = std::min(L.n_tiles, 2 * num_sms());
      t_stats_tile_kernel<<<grid, kNThreads, smem, stream>>>(
          jobs, reinterpret_cast<const TItem*>(w + L.off_tiles), L.n_tiles, flag, wide, part);
      ++*launches;
    }
    if (L.n_small) {
      t_stats_small_kernel<<<L.n_small, kSmallThreads, 0, stream>>>(
          jobs, reinterpret_cast<const TItem*>(w + L.off_small), flag, wide, part);
      ++*launches;
    }
    t_stats_finish_kernel<<<dim3(16, L.n_jobs), 256, 0, stream>>>(jobs, flag, part, stats, decay, weight);
    ++*launches;
  }
  t_diag_kernel<<<eg, 256, 0, stream>>>(blks, flag, part2);
  t_diag_finish_kernel<<<(n_blocks + 255) / 256, 256, 0, stream>>>(n_blocks, flag, part2, graft_num, block_status);
  *launches += 2;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("tensor stats kernels", e);
  return SHAMPOO_OK;
}

// ---------------------------------------------------------------- precondition
struct TPrecLayout {
  std::vector<uint8_t> blob;
  size_t off_blk = 0;
  size_t off_jobs[KO] = {0}, off_small[KO] = {0}, off_tiles[KO] = {0};
  int n_small[KO] = {0}, n_tiles[KO] = {0};
  size_t off_part = 0, off_Y = 0, total = 0;
};

static void prec_layout(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks, TPrecLayout& L) {
  std::vector<TBlk> blks(n_blocks);
  std::vector<TModeJob> jobs[KO];
  std::vector<TItem> small[KO], tiles[KO];
  int64_t y = 0;
  for (int b = 0; b < n_blocks; ++b) {
    const shampoo_tblock_t& bk = B[b];
    TBlk& k = blks[b];
    k = make_blk(T[bk.tensor_id], bk);
    bool any = false;
    for (int i = 0; i < bk.order; ++i) any |= bk.p[i] != 0;
    if (!any) continue;  // diag-only: fin = -1
    k.y0 = y;
    k.y1 = y + k.numel;
    y += 2 * k.numel;
    int cur = 0;
    int64_t pre = 1;
    for (int i = 0; i < KO; ++i) {
      const int64_t e = k.ext[i];
      int64_t post = 1;
      for (int l = i + 1; l < KO; ++l) post *= k.ext[l];
      if (i < bk.order && bk.p[i]) {
        TModeJob j;
        std::memset(&j, 0, sizeof j);
        j.in = cur ? k.y1 : k.y0;
        j.out = cur ? k.y0 : k.y1;
        j.xoff = bk.off[i];
        j.ld = bk.ld[i];
        j.e = (int)e;
        j.Pb = pre;
        j.Sb = post;
        j.blk = b;
        const int jid = (int)jobs[i].size();
        if (e <= kSmallMode) {
          j.kind = 0;
          const int64_t nf = pre * post;
          for (int64_t f = 0; f < nf; f += kSmallThreads) small[i].push_back({jid, (int)(f / kSmallThreads), 0, 0});
        } else if (post == 1) {
          j.kind = 1;
          const int ta = (int)((pre + kNT - 1) / kNT), tb = (int)((e + kNT - 1) / kNT);
          for (int a = 0; a < ta; ++a)
            for (int c = 0; c < tb; ++c) tiles[i].push_back({jid, a, c, 0});
        } else {
          j.kind = 2;
          const int ta = (int)((e + kNT - 1) / kNT), tb = (int)((post + kNT - 1) / kNT);
          for (int64_t p = 0; p < pre; ++p)
            for (int a = 0; a < ta; ++a)
              for (int c = 0; c < tb; ++c) tiles[i].push_back({jid, a, c, (int)p});
        }
        jobs[i].push_back(j);
        cur ^= 1;
      }
      pre *= e;
    }
    k.fin = cur;
  }
  L.blob.clear();
  L.off_blk = put(L.blob, blks.data(), blks.size());
  for (int i = 0; i < KO; ++i) {
    L.off_jobs[i] = put(L.blob, jobs[i].data(), jobs[i].size());
    L.off_small[i] = put(L.blob, small[i].data(), small[i].size());
    L.off_tiles[i] = put(L.blob, tiles[i].data(), tiles[i].size());
    L.n_small[i] = (int)small[i].size();
    L.n_tiles[i] = (int)tiles[i].size();
  }
  size_t q = al(L.blob.size());
  L.off_part = q;
  q = al(q + (size_t)n_blocks * kTChunks * sizeof(double));
  L.off_Y = q;
  q = al(q + (size_t)y * sizeof(float));
  L.total = q;
}

size_t tensor_precondition_workspace_bytes(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks) {
  TPrecLayout L;
  prec_layout(T, B, n_blocks, L);
  return L.total;
}

int tensor_precondition_launch(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks,
                               const float* roots, const double* graft_num, float* graft_scale, double* den,
                               void* ws, size_t ws_bytes, cudaStream_t stream, int64_t* launches) {
  if (n_blocks == 0) return SHAMPOO_OK;
  TPrecLayout L;
  prec_layout(T, B, n_blocks, L);
  if (ws_bytes < L.total)
    return set_error(SHAMPOO_ERR_WORKSPACE, "tensor precondition workspace: have %zu bytes, need %zu", ws_bytes,
                     L.total);
  char* w = static_cast<char*>(ws);
  if (cudaMemcpyAsync(w, L.blob.data(), L.blob.size(), cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return set_cuda_error("cudaMemcpyAsync(tensor precondition tables)");
  const TBlk* blks = reinterpret_cast<const TBlk*>(w + L.off_blk);
  double* part = reinterpret_cast<double*>(w + L.off_part);
  float* Y = reinterpret_cast<float*>(w + L.off_Y);
  const unsigned eg = (unsigned)n_blocks * kTChunks;
  t_gather_kernel<<<eg, 256, 0, stream>>>(blks, Y);
  ++*launches;
  const size_t smem = (size_t)2 * 2 * kAsyncTile * sizeof(double);
  if (ensure_smem((const void*)t_mode_tile_kernel, smem) !=
      cudaSuccess)
    return set_cuda_error("cudaFuncSetAttribute(t_mode_tile_kernel)");
  for (int i = 0; i < KO; ++i) {
    const TModeJob* jobs = reinterpret_cast<const TModeJob*>(w + L.off_jobs[i]);
    if (L.n_small[i]) {
      t_mode_small_kernel<<<L.n_small[i], kSmallThreads, 0, stream>>>(
          jobs, reinterpret_cast<const TItem*>(w + L.off_small[i]), roots, Y);
      ++*launches;
    }
    if (L.n_tiles[i]) {
      const int grid = std::min(L.n_tiles[i], 2 * num_sms());
      t_mode_tile_kernel<<<grid, kNThreads, smem, stream>>>(jobs, reinterpret_cast<const TItem*>(w + L.off_tiles[i]),
                                                            L.n_tiles[i], roots, Y);
      ++*launches;
    }
  }
  t_scatter_kernel<<<eg, 256, 0, stream>>>(blks, Y, part);
  t_prec_finish_kernel<<<(n_blocks + 255) / 256, 256, 0, stream>>>(n_blocks, part, graft_num, graft_scale, den);
  *launches += 2;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("tensor precondition kernels", e);
  return SHAMPOO_OK;
}

}  // namespace shp
