// precondition.cu -- preconditioned gradient and grafting (rows a8, a9).
//
//   two-sided  P_b = X_L G_b X_R   (L^{-1/4} G R^{-1/4})
//   one-sided  P_b = G_b X_R or X_L G_b
//   none       P_b = D_b^{-1/2} o G_b     (grafted diagonal AdaGrad; reading #17)
//   scale_b    = sqrt(num_b) / ||P_b||_F  (grafting; per block, reading #9)
//
// Launch sequence: prep (tile/offset prefix sums) -> phase 1 (Y = X_L G_b, or
// P = X_L G_b for left-only blocks) -> phase 2 (P = Y X_R, or P = G_b X_R)
// -> diag-only blocks -> den partials -> finish (fixed-order sums, scale).
// The products run on the FP64 tensor pipe through dmma_gemm.cuh; Y is kept
// in fp32 in the workspace (L2-resident for a 1024^2 block).
#include <algorithm>
#include <cstring>
#include <vector>

#include "dmma_gemm.cuh"
#include "internal.h"
#include "oz_precondition.h"
#include "tc_gemm.h"

namespace shp {

constexpr int kPChunks = 64;

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

SHP_DEV int ntile(int n) { return (n + kTileM - 1) / kTileM; }

// DMMA-path work of a block (blocks served by the tcgen05 path have tc_flag set)
SHP_DEV void block_counts(const shampoo_block_t& b, int tc_flag, int64_t& n1, int64_t& n2, int64_t& ny) {
  const int64_t t = (int64_t)ntile(b.rows) * ntile(b.cols);
  n1 = (b.p_left && !tc_flag) ? t : 0;
  n2 = (b.p_right && !tc_flag) ? t : 0;
  ny = (b.p_left && b.p_right && !tc_flag) ? (int64_t)b.rows * b.cols : 0;
}

__global__ void __launch_bounds__(1024) prec_prep_kernel(const shampoo_block_t* blocks, const int* tc_flags,
                                                         int n_blocks, int64_t* pre1, int64_t* pre2, int64_t* yoff) {
  __shared__ int64_t s1[1024], s2[1024], s3[1024];
  const int t = threadIdx.x;
  const int per = (n_blocks + 1023) / 1024;
  const int b0 = t * per, b1 = min(n_blocks, b0 + per);
  int64_t a1 = 0, a2 = 0, a3 = 0;
  for (int b = b0; b < b1; ++b) {
    int64_t n1, n2, ny;
    block_counts(blocks[b], tc_flags[b], n1, n2, ny);
    a1 += n1;
    a2 += n2;
    a3 += ny;
  }
  s1[t] = a1;
  s2[t] = a2;
  s3[t] = a3;
  __syncthreads();
  if (t == 0) {
    int64_t c1 = 0, c2 = 0, c3 = 0;
    for (int i = 0; i < 1024; ++i) {
      int64_t v1 = s1[i], v2 = s2[i], v3 = s3[i];
      s1[i] = c1;
      s2[i] = c2;
      s3[i] = c3;
      c1 += v1;
      c2 += v2;
      c3 += v3;
    }
    pre1[n_blocks] = c1;
    pre2[n_blocks] = c2;
    yoff[n_blocks] = c3;
  }
  __syncthreads();
  a1 = s1[t];
  a2 = s2[t];
  a3 = s3[t];
  for (int b = b0; b < b1; ++b) {
    pre1[b] = a1;
    pre2[b] = a2;
    yoff[b] = a3;
    int64_t n1, n2, ny;
    block_counts(blocks[b], tc_flags[b], n1, n2, ny);
    a1 += n1;
    a2 += n2;
    a3 += ny;
  }
}

SHP_DEV int find_blk(const int64_t* prefix, int n_blocks, int64_t item) {
  int lo = 0, hi = n_blocks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= item) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

SHP_DEV void store_tile_f32(const Acc& acc, float* dst, int64_t ld, int ti, int tj, int rows, int cols) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    const int i = ti * kTileM + acc_row(warp, lane, mt);
    if (i >= rows) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tj * kTileM + acc_col(warp, lane, nt, e);
        if (j < cols) dst[(int64_t)i * ld + j] = (float)acc.c[mt][nt][e];
      }
  }
}

// phase 1: Y (or P) = X_L G_b ; phase 2: P = Y X_R (or G_b X_R)
template <int PHASE>
__global__ void __launch_bounds__(kThreads, 1)
    prec_gemm_kernel(const shampoo_tensor_t* tensors, const shampoo_block_t* blocks, int n_blocks,
                     const float* roots, const int64_t* prefix, const int64_t* yoff, float* Y) {
  extern __shared__ __align__(16) double smem[];
  const int64_t total = prefix[n_blocks];
  Acc acc;
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
    const int b = find_blk(prefix, n_blocks, item);
    const shampoo_block_t blk = blocks[b];
    const int64_t local = item - prefix[b];
    const int tc = ntile(blk.cols);
    const int ti = (int)(local / tc), tj = (int)(local % tc);
    const shampoo_tensor_t ten = tensors[blk.tensor_id];
    const float* gb = ten.G + blk.row0 * ten.ldg + blk.col0;
    float* pb = ten.P + blk.row0 * ten.ldp + blk.col0;
    if (PHASE == 1) {
      // C[i][j] = sum_k X_L[i][k] G_b[k][j];  K = rows
      F32Panel la{roots + blk.left_off, blk.left_ld, 0, ti * kTileM, blk.rows, blk.rows};
      F32Panel lb{gb, ten.ldg, 1, tj * kTileM, blk.cols, blk.rows};
      gemm_tile(acc, la, lb, (blk.rows + kTileK - 1) / kTileK, smem);
      if (blk.p_right) store_tile_f32(acc, Y + yoff[b], blk.cols, ti, tj, blk.rows, blk.cols);
      else store_tile_f32(acc, pb, ten.ldp, ti, tj, blk.rows, blk.cols);
    } else {
      // C[i][j] = sum_k Z[i][k] X_R[j][k] (X_R symmetric);  K = cols
      const bool two = blk.p_left != 0;
      const float* z = two ? Y + yoff[b] : gb;
      const int64_t ldz = two ? (int64_t)blk.cols : ten.ldg;
      F32Panel la{z, ldz, 0, ti * kTileM, blk.rows, blk.cols};
      F32Panel lb{roots + blk.right_off, blk.right_ld, 0, tj * kTileM, blk.cols, blk.cols};
      gemm_tile(acc, la, lb, (blk.cols + kTileK - 1) / kTileK, smem);
      store_tile_f32(acc, pb, ten.ldp, ti, tj, blk.rows, blk.cols);
    }
  }
}

// diagonal-only blocks: P = G / sqrt(max(D, 1e-30))
__global__ void __launch_bounds__(kThreads) prec_diag_kernel(const shampoo_tensor_t* tensors,
                                                             const shampoo_block_t* blocks) {
  const int b = blockIdx.x / kPChunks, c = blockIdx.x % kPChunks;
  const shampoo_block_t blk = blocks[b];
  if (blk.p_left || blk.p_right) return;
  const shampoo_tensor_t ten = tensors[blk.tensor_id];
  const int rows_per = (blk.rows + kPChunks - 1) / kPChunks;
  const int r0 = c * rows_per, r1 = min(blk.rows, r0 + rows_per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = r0 + warp; r < r1; r += kThreads / 32) {
    const float* g = ten.G + (blk.row0 + r) * ten.ldg + blk.col0;
    const float* d = ten.D + (blk.row0 + r) * ten.ldd + blk.col0;
    float* p = ten.P + (blk.row0 + r) * ten.ldp + blk.col0;
    for (int col = lane; col < blk.cols; col += 32) {
      double dv = (double)d[col];
      dv = dv > 1e-30 ? dv : 1e-30;
      p[col] = (float)((double)g[col] / sqrt(dv));
    }
  }
}

__global__ void __launch_bounds__(kThreads) prec_den_kernel(const shampoo_tensor_t* tensors,
                                                            const shampoo_block_t* blocks, double* part) {
  const int b = blockIdx.x / kPChunks, c = blockIdx.x % kPChunks;
  __shared__ double red[kThreads / 32];
  const shampoo_block_t blk = blocks[b];
  const shampoo_tensor_t ten = tensors[blk.tensor_id];
  const int rows_per = (blk.rows + kPChunks - 1) / kPChunks;
  const int r0 = c * rows_per, r1 = min(blk.rows, r0 + rows_per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s = 0.0;
  for (int r = r0 + warp; r < r1; r += kThreads / 32) {
    const float* p = ten.P + (blk.row0 + r) * ten.ldp + blk.col0;
    for (int col = lane; col < blk.cols; col += 32) {
      const double v = (double)p[col];
      s = fma(v, v, s);
    }
  }
  s = warp_sum_fixed(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t = __dadd_rn(t, red[w]);
    part[(int64_t)b * kPChunks + c] = t;
  }
}

__global__ void prec_finish_kernel(int n_blocks, const double* part, const double* graft_num, float* graft_scale,
                                   double* den) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  double s = 0.0;
  for (int c = 0; c < kPChunks; ++c) s = __dadd_rn(s, part[(int64_t)b * kPChunks + c]);
  if (den) den[b] = s;
  if (graft_scale) {
    float sc = 0.0f;
    if (graft_num && s > 0.0) sc = (float)(sqrt(graft_num[b]) / sqrt(s));
    graft_scale[b] = sc;
  }
}

// ---------------------------------------------------------------- host plan
// Everything the call needs is derived from the HOST tables on every call:
// tcgen05 eligibility, TMA maps, per-block GEMM jobs, split segments and the
// workspace layout.  One pageable cudaMemcpyAsync uploads the tables.
struct RootRun {  // consecutive equal-size roots at a constant stride (one 3-D TMA map)
  int64_t off0, stride;
  int n, ld, count;
};

struct PrecLayout {
  // host staging (uploaded as one blob at ws + 0)
  std::vector<uint8_t> blob;
  size_t off_tensors = 0, off_blocks = 0, off_flags = 0, off_maps = 0, off_jobs1 = 0, off_jobs2 = 0, off_segs = 0;
  int n_maps = 0, n_jobs1 = 0, n_jobs2 = 0, n_segs = 0;
  int64_t tiles1 = 0, tiles2 = 0;
  bool any_dmma = false;
  // device regions (offsets from ws)
  size_t off_pre = 0, off_part = 0, off_Y = 0, off_rlo = 0, off_glo = 0, off_zhi = 0, off_zlo = 0, off_oz = 0,
         total = 0;
  std::vector<int> flags;  // per block: 1 tcgen05 3xTF32, 2 INT8 Ozaki (oz_precondition.cu), 0 DMMA / diagonal
  int64_t roots_elems = 0;
};

static bool tc_eligible(const shampoo_block_t& b, const shampoo_tensor_t& t) {
  // one-sided blocks (P = G_b X_R, X_L G_b) never take the 3xTF32 path: their statistic is often rank-deficient
  // (the vocabulary rows of an embedding gradient: G_b's rows span few dimensions), so the root's largest
  // eigenvalues sit in directions G_b is orthogonal to and the product cancels them exactly; an fp32
  // accumulation (the tensor core's 3xTF32) loses up to ~kappa^{1/2} of its relative accuracy there -- measured
  // on B200: P rel. error 6.2e-3 on a 4-nonzero-row vocabulary block (north-star bar 1e-3), against 3.2e-5 for
  // the exact product of the same fp32 root (tests/test_gpu_bench_path.py).  Right-only blocks run on the INT8
  // Ozaki path (oz_precondition.cu, exact int32 products), the rest on FP64 DMMA.
  if (!b.p_right || !b.p_left) return false;  // one-sided / diagonal-only blocks: Ozaki / DMMA / elementwise
  // the raw G is the TMA "hi" operand: contiguous rows, 16-byte aligned
  if (t.ldg != t.n || (t.n & 3) || (reinterpret_cast<uintptr_t>(t.G) & 15)) return false;
  const bool rows_ok = (b.rows % 32 == 0) || (b.row0 + b.rows == t.m);
  const bool cols_ok = (b.cols % 32 == 0) || (b.col0 + b.cols == t.n);
  return rows_ok && cols_ok;
}

static int64_t r4(int64_t x) { return (x + 3) / 4 * 4; }

template <class T>
static size_t put(std::vector<uint8_t>& blob, const T* p, size_t n, size_t align = 256) {
  size_t off = (blob.size() + align - 1) / align * align;
  blob.resize(off + n * sizeof(T));
  if (n) std::memcpy(blob.data() + off, p, n * sizeof(T));
  return off;
}

// Builds the layout; when `ws` is null only sizes are computed (maps need real pointers).
static int build_layout(const shampoo_tensor_t* T, int n_tensors, const shampoo_block_t* B, int n_blocks,
                        const float* roots, const float* roots_lo, char* ws, PrecLayout& L) {
  std::vector<int>& flags = L.flags;
  flags.assign(n_blocks, 0);
  std::vector<char> t_g(n_tensors, 0), t_z(n_tensors, 0);
  size_t y_elems = 0;
  for (int b = 0; b < n_blocks; ++b) {
    flags[b] = tc_eligible(B[b], T[B[b].tensor_id]) ? 1 : oz_precondition_eligible(B[b]) ? 2 : 0;
    if (flags[b] == 2) continue;
    if (flags[b]) {
      t_g[B[b].tensor_id] = 1;
      if (B[b].p_left) t_z[B[b].tensor_id] = 1;
    } else if (B[b].p_left || B[b].p_right) {
      L.any_dmma = true;
      if (B[b].p_left && B[b].p_right) y_elems += (size_t)B[b].rows * B[b].cols;
    }
  }
  // roots runs
  struct R { int64_t off; int n, ld; };
  std::vector<R> rs;
  for (int b = 0; b < n_blocks; ++b) {
    if (B[b].p_left) rs.push_back({B[b].left_off, B[b].rows, B[b].left_ld});
    if (B[b].p_right) rs.push_back({B[b].right_off, B[b].cols, B[b].right_ld});
  }
  std::sort(rs.begin(), rs.end(), [](const R& a, const R& c) { return a.off < c.off; });
  std::vector<RootRun> runs;
  int64_t rend = 0;
  for (const R& r : rs) {
    const int64_t stride = ((int64_t)r.n * r.ld + 63) / 64 * 64;
    rend = std::max(rend, r.off + (int64_t)r.n * r.ld);
    if (!runs.empty()) {
      RootRun& q = runs.back();
      if (q.n == r.n && q.ld == r.ld && q.stride == stride && r.off == q.off0 + (int64_t)q.count * q.stride) {
        ++q.count;
        continue;
      }
    }
    runs.push_back({r.off, stride, r.n, r.ld, 1});
  }
  L.roots_elems = rend;
  // device layout
  const size_t pb = al((size_t)(n_blocks + 1) * sizeof(int64_t));
  size_t q = 0;
  auto region = [&](size_t bytes) { size_t o = q; q = al(q + bytes); return o; };
  // header blob size is unknown until maps are built; reserve generously
  const size_t n_maps_max = 4 * runs.size() + 4 * (size_t)n_tensors;
  const size_t hdr = al((size_t)n_tensors * sizeof(shampoo_tensor_t)) + al((size_t)n_blocks * sizeof(shampoo_block_t)) +
                     al((size_t)n_blocks * sizeof(int)) + al(n_maps_max * sizeof(CUtensorMap)) +
                     2 * al((size_t)n_blocks * sizeof(TcJob)) + al(((size_t)n_tensors + 64) * sizeof(SplitSeg)) + 4096;
  region(hdr);
  L.off_pre = region(3 * pb);
  L.off_part = region((size_t)n_blocks * kPChunks * sizeof(double));
  L.off_Y = region(y_elems * sizeof(float));
  L.off_rlo = region(roots_lo ? 0 : (size_t)rend * sizeof(float));
  std::vector<size_t> goff(n_tensors, 0), zoff(n_tensors, 0);
  size_t gsz = 0, zsz = 0;
  for (int t = 0; t < n_tensors; ++t) {
    if (t_g[t]) { goff[t] = gsz; gsz += (size_t)al((size_t)T[t].m * T[t].n * sizeof(float)); }
    if (t_z[t]) { zoff[t] = zsz; zsz += (size_t)al((size_t)T[t].n * r4(T[t].m) * sizeof(float)); }
  }
  L.off_glo = region(gsz);
  L.off_zhi = region(zsz);
  L.off_zlo = region(zsz);
  L.off_oz = region(oz_precondition_bytes(B, n_blocks, flags.data()));
  L.total = q;
  if (!ws) return SHAMPOO_OK;

  // ---- tensor maps
  std::vector<CUtensorMap> maps;
  auto add_map = [&](const void* base, int dims, const uint64_t* size, const uint64_t* strides,
                     int box = 128) -> int {
    CUtensorMap m;
    int rc = make_map_f32(&m, base, dims, size, strides, box);
    if (rc) return -1;
    maps.push_back(m);
    return (int)maps.size() - 1;
  };
  const float* rhi = roots;  // raw fp32 roots: the tensor core reads trunc_tf32
  float* rlo = roots_lo ? const_cast<float*>(roots_lo) : reinterpret_cast<float*>(ws + L.off_rlo);
  std::vector<int> run_map_hi(runs.size()), run_map_lo(runs.size()), run_map_hib(runs.size()),
      run_map_lob(runs.size());  // ...b: the B-operand (kTcGemmBN-row box) variants
  for (size_t i = 0; i < runs.size(); ++i) {
    const RootRun& r = runs[i];
    uint64_t size[3] = {(uint64_t)r.n, (uint64_t)r.n, (uint64_t)r.count};
    uint64_t st[2] = {(uint64_t)r.ld * 4, (uint64_t)r.stride * 4};
    run_map_hi[i] = add_map(rhi + r.off0, 3, size, st);
    run_map_lo[i] = add_map(rlo + r.off0, 3, size, st);
    run_map_hib[i] = add_map(rhi + r.off0, 3, size, st, kTcGemmBN);
    run_map_lob[i] = add_map(rlo + r.off0, 3, size, st, kTcGemmBN);
    if (run_map_hi[i] < 0 || run_map_lo[i] < 0 || run_map_hib[i] < 0 || run_map_lob[i] < 0) return SHAMPOO_ERR_CUDA;
  }
  auto find_root = [&](int64_t off, int& map_hi, int& map_lo, int& z, bool as_b) {
    for (size_t i = 0; i < runs.size(); ++i) {
      const RootRun& r = runs[i];
      if (off >= r.off0 && off < r.off0 + (int64_t)r.count * r.stride) {
        map_hi = as_b ? run_map_hib[i] : run_map_hi[i];
        map_lo = as_b ? run_map_lob[i] : run_map_lo[i];
        z = (int)((off - r.off0) / r.stride);
        return;
      }
    }
  };
  std::vector<int> g_hi(n_tensors, -1), g_lo(n_tensors, -1), z_hi(n_tensors, -1), z_lo(n_tensors, -1);
  std::vector<SplitSeg> segs;
  for (int t = 0; t < n_tensors; ++t) {
    const int64_t ldz = r4(T[t].m);
    if (t_g[t]) {
      float* gl = reinterpret_cast<float*>(ws + L.off_glo + goff[t]);
      uint64_t size[2] = {(uint64_t)T[t].n, (uint64_t)T[t].m};
      uint64_t st[1] = {(uint64_t)T[t].n * 4};
      g_hi[t] = add_map(T[t].G, 2, size, st);
      g_lo[t] = add_map(gl, 2, size, st);
      if (g_hi[t] < 0 || g_lo[t] < 0) return SHAMPOO_ERR_CUDA;
      segs.push_back({T[t].G, gl, T[t].m * T[t].n});
    }
    if (t_z[t]) {
      float* zh = reinterpret_cast<float*>(ws + L.off_zhi + zoff[t]);
      float* zl = reinterpret_cast<float*>(ws + L.off_zlo + zoff[t]);
      uint64_t size[2] = {(uint64_t)T[t].m, (uint64_t)T[t].n};
      uint64_t st[1] = {(uint64_t)ldz * 4};
      z_hi[t] = add_map(zh, 2, size, st, kTcGemmBN);
      z_lo[t] = add_map(zl, 2, size, st, kTcGemmBN);
      if (z_hi[t] < 0 || z_lo[t] < 0) return SHAMPOO_ERR_CUDA;
    }
  }
  // roots: the whole packed range (a multiple of 4 floats) as one flat segment
  if (rend && !roots_lo) segs.push_back({roots, rlo, rend});  // else: the caller's precomputed split
  // ---- jobs
  std::vector<TcJob> j1, j2;
  int64_t t1 = 0, t2 = 0;
  for (int b = 0; b < n_blocks; ++b) {
    if (flags[b] != 1) continue;
    const shampoo_block_t& bk = B[b];
    const shampoo_tensor_t& tt = T[bk.tensor_id];
    const int tm = (bk.rows + 127) / 128, tn = (bk.cols + kTcGemmBN - 1) / kTcGemmBN;
    TcJob j;
    std::memset(&j, 0, sizeof j);
    // phase 1: C = G_b . X_R   (M = rows, N = cols, K = cols)
    j.a = {g_hi[bk.tensor_id], g_lo[bk.tensor_id], (int32_t)bk.col0, (int32_t)bk.row0, 0, 2};
    int mh = -1, ml = -1, z = 0;
    find_root(bk.right_off, mh, ml, z, true);
    j.b = {mh, ml, 0, 0, z, 3};
    j.M = bk.rows;
    j.N = bk.cols;
    j.K = bk.cols;
    j.tiles_n = tn;
    j.tile_begin = t1;
    if (bk.p_left) {
      const int64_t ldz = r4(tt.m);
      float* zh = reinterpret_cast<float*>(ws + L.off_zhi + zoff[bk.tensor_id]);
      float* zl = reinterpret_cast<float*>(ws + L.off_zlo + zoff[bk.tensor_id]);
      j.out_mode = 1;
      j.out_hi = zh + bk.col0 * ldz + bk.row0;
      j.out_lo = zl + bk.col0 * ldz + bk.row0;
      j.ld_out = ldz;
    } else {
      j.out_mode = 0;
      j.out_hi = tt.P + bk.row0 * tt.ldp + bk.col0;
      j.ld_out = tt.ldp;
    }
    j1.push_back(j);
    t1 += (int64_t)tm * tn;
    if (bk.p_left) {
      // phase 2: P = X_L . Z   (B_j[k] = Zt[col0 + j][row0 + k]; K = rows)
      TcJob k2;
      std::memset(&k2, 0, sizeof k2);
      find_root(bk.left_off, mh, ml, z, false);
      k2.a = {mh, ml, 0, 0, z, 3};
      k2.b = {z_hi[bk.tensor_id], z_lo[bk.tensor_id], (int32_t)bk.row0, (int32_t)bk.col0, 0, 2};
      k2.M = bk.rows;
      k2.N = bk.cols;
      k2.K = bk.rows;
      k2.out_mode = 0;
      k2.out_hi = tt.P + bk.row0 * tt.ldp + bk.col0;
      k2.ld_out = tt.ldp;
      k2.tiles_n = tn;
      k2.tile_begin = t2;
      j2.push_back(k2);
      t2 += (int64_t)tm * tn;
    }
  }
  L.tiles1 = t1;
  L.tiles2 = t2;
  L.n_jobs1 = (int)j1.size();
  L.n_jobs2 = (int)j2.size();
  L.n_maps = (int)maps.size();
  L.n_segs = (int)segs.size();
  L.blob.clear();
  L.off_tensors = put(L.blob, T, n_tensors);
  L.off_blocks = put(L.blob, B, n_blocks);
  L.off_flags = put(L.blob, flags.data(), flags.size());
  L.off_maps = put(L.blob, maps.data(), maps.size());
  L.off_jobs1 = put(L.blob, j1.data(), j1.size());
  L.off_jobs2 = put(L.blob, j2.data(), j2.size());
  L.off_segs = put(L.blob, segs.data(), segs.size());
  if (L.blob.size() > hdr) return set_error(SHAMPOO_ERR_WORKSPACE, "precondition header overflow");
  return SHAMPOO_OK;
}

size_t precondition_workspace_bytes(const shampoo_tensor_t* tensors_host, int n_tensors,
                                    const shampoo_block_t* blocks_host, int n_blocks) {
  PrecLayout L;
  build_layout(tensors_host, n_tensors, blocks_host, n_blocks, nullptr, nullptr, nullptr, L);
  return L.total;
}

int precondition_launch(const shampoo_tensor_t* tensors_host, int n_tensors, const shampoo_block_t* blocks_host,
                        int n_blocks, const float* roots, const float* roots_lo, const double* graft_num,
                        float* graft_scale, double* den, void* ws, size_t ws_bytes, cudaStream_t stream,
                        int64_t* launches) {
  if (n_blocks == 0) return SHAMPOO_OK;
  PrecLayout L;
  build_layout(tensors_host, n_tensors, blocks_host, n_blocks, nullptr, roots_lo, nullptr, L);
  if (ws_bytes < L.total)
    return set_error(SHAMPOO_ERR_WORKSPACE, "precondition workspace: have %zu bytes, need %zu", ws_bytes, L.total);
  char* w = static_cast<char*>(ws);
  int rc = build_layout(tensors_host, n_tensors, blocks_host, n_blocks, roots, roots_lo, w, L);
  if (rc) return rc;
  if (cudaMemcpyAsync(w, L.blob.data(), L.blob.size(), cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return set_cuda_error("cudaMemcpyAsync(precondition tables)");
  const shampoo_tensor_t* tensors = reinterpret_cast<const shampoo_tensor_t*>(w + L.off_tensors);
  const shampoo_block_t* blocks = reinterpret_cast<const shampoo_block_t*>(w + L.off_blocks);
  const int* flags = reinterpret_cast<const int*>(w + L.off_flags);
  const CUtensorMap* maps = reinterpret_cast<const CUtensorMap*>(w + L.off_maps);
  const size_t pb = al((size_t)(n_blocks + 1) * sizeof(int64_t));
  int64_t* pre1 = reinterpret_cast<int64_t*>(w + L.off_pre);
  int64_t* pre2 = reinterpret_cast<int64_t*>(w + L.off_pre + pb);
  int64_t* yoff = reinterpret_cast<int64_t*>(w + L.off_pre + 2 * pb);
  double* part = reinterpret_cast<double*>(w + L.off_part);
  float* Y = reinterpret_cast<float*>(w + L.off_Y);

  // tcgen05 3xTF32 path
  rc = tf32_split_launch(reinterpret_cast<const SplitSeg*>(w + L.off_segs), L.n_segs, stream, launches);
  if (rc) return rc;
  rc = tc_gemm_launch(reinterpret_cast<const TcJob*>(w + L.off_jobs1), L.n_jobs1, L.tiles1, maps, stream, launches);
  if (rc) return rc;
  rc = tc_gemm_launch(reinterpret_cast<const TcJob*>(w + L.off_jobs2), L.n_jobs2, L.tiles2, maps, stream, launches);
  if (rc) return rc;
  // INT8 Ozaki path for the one-sided blocks (exact int32 products, fp32 P)
  rc = oz_precondition_launch(tensors_host, blocks_host, n_blocks, L.flags.data(), roots, w + L.off_oz, stream,
                              launches);
  if (rc) return rc;
  // DMMA path for the remaining blocks (left-only, unaligned)
  if (L.any_dmma) {
    const size_t smem = (size_t)kGemmSmemDoubles * sizeof(double);
    if (ensure_smem((const void*)prec_gemm_kernel<1>, smem) !=
            cudaSuccess ||
        ensure_smem((const void*)prec_gemm_kernel<2>, smem) !=
            cudaSuccess)
      return set_cuda_error("cudaFuncSetAttribute(prec_gemm_kernel)");
    prec_prep_kernel<<<1, 1024, 0, stream>>>(blocks, flags, n_blocks, pre1, pre2, yoff);
    prec_gemm_kernel<1><<<num_sms(), kThreads, smem, stream>>>(tensors, blocks, n_blocks, roots, pre1, yoff, Y);
    prec_gemm_kernel<2><<<num_sms(), kThreads, smem, stream>>>(tensors, blocks, n_blocks, roots, pre2, yoff, Y);
    *launches += 3;
  }
  const unsigned eg = (unsigned)n_blocks * kPChunks;
  prec_diag_kernel<<<eg, kThreads, 0, stream>>>(tensors, blocks);
  prec_den_kernel<<<eg, kThreads, 0, stream>>>(tensors, blocks, part);
  prec_finish_kernel<<<(n_blocks + 255) / 256, 256, 0, stream>>>(n_blocks, part, graft_num, graft_scale, den);
  *launches += 3;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("precondition kernels", e);
  return SHAMPOO_OK;
}

}  // namespace shp
