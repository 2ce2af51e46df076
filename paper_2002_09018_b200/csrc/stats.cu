// stats.cu -- per-step Shampoo statistics (row a2): L/R EMA update under the
// sequential fp64 contract (bit-exact with the oracle), the diagonal AdaGrad
// accumulator D and the per-block graft numerator.
//
// Alg. 1:  L <- decay*L + weight*G G^T ; R <- decay*R + weight*G^T G ;
//                      D <- D + G o G ;  num_b = sum g^2 / max(D, 1e-30)
// Contract (oracle/csrc/oracle_stats.c): acc = sum_k ascending of
// (double)a_k*(double)b_k in fp64; t1 = weight*acc; t2 = decay*old; (float)(t1+t2).
//
// Launch sequence (one step, all blocks of all tensors):
//   memset(flags) -> check (non-finite G per block) -> prep (tile / buffer prefix sums)
//   -> widen (owned blocks: fp32 G_b -> zero-padded fp64 row panels, G_b and G_b^T,
//      so the DMMA tiles stream from the cp.async fp64 pipeline of the Newton core)
//   -> stats (persistent DMMA tiles, L and R, owned blocks only)
//   -> diag (D update + per-chunk graft partials) -> finish (fixed-order sums)
#include <algorithm>

#include "dmma_gemm.cuh"
#include "internal.h"

namespace shp {

constexpr int kChunks = 64;  // row chunks per block for the elementwise passes
constexpr int kPrefixSmem = 1536;  // prefix entries cached in shared memory (12 KB; 2 CTAs/SM)

struct StatsWs {
  int* flag;         // n_blocks (non-finite marker)
  int64_t* prefix;   // n_blocks + 1 (stats tiles)
  int64_t* offL;     // n_blocks: fp64 offset of the widened G_b   (rows_p64 x roundup(cols, 32)), -1 if none
  int64_t* offR;     // n_blocks: fp64 offset of the widened G_b^T (cols_p64 x roundup(rows, 32)), -1 if none
  double* part;      // n_blocks * kChunks
  double* wide;      // widened operands
};

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
static int64_t rup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

static bool owns_l(const shampoo_block_t& b, int only_owner) { return b.p_left && (only_owner < 0 || b.owner_left == only_owner); }
static bool owns_r(const shampoo_block_t& b, int only_owner) { return b.p_right && (only_owner < 0 || b.owner_right == only_owner); }

static size_t fixed_bytes(int n_blocks) {
  return al((size_t)n_blocks * sizeof(int)) + 3 * al((size_t)(n_blocks + 1) * sizeof(int64_t)) +
         al((size_t)n_blocks * kChunks * sizeof(double));
}

size_t stats_workspace_bytes(const shampoo_block_t* blocks_host, int n_blocks, int only_owner) {
  size_t wide = 0;
  for (int b = 0; b < n_blocks; ++b) {
    const shampoo_block_t& k = blocks_host[b];
    if (owns_l(k, only_owner)) wide += (size_t)rup(k.rows, 64) * rup(k.cols, 32);
    if (owns_r(k, only_owner)) wide += (size_t)rup(k.cols, 64) * rup(k.rows, 32);
  }
  return fixed_bytes(n_blocks) + al(wide * sizeof(double));
}

static StatsWs carve(void* ws, int n_blocks) {
  char* q = static_cast<char*>(ws);
  StatsWs w;
  w.flag = reinterpret_cast<int*>(q);
  q += al((size_t)n_blocks * sizeof(int));
  const size_t pb = al((size_t)(n_blocks + 1) * sizeof(int64_t));
  w.prefix = reinterpret_cast<int64_t*>(q);
  q += pb;
  w.offL = reinterpret_cast<int64_t*>(q);
  q += pb;
  w.offR = reinterpret_cast<int64_t*>(q);
  q += pb;
  w.part = reinterpret_cast<double*>(q);
  q += al((size_t)n_blocks * kChunks * sizeof(double));
  w.wide = reinterpret_cast<double*>(q);
  return w;
}

SHP_DEV int tiles_of(int n) { return (n + kNT - 1) / kNT; }  // 64x64 output tiles
SHP_DEV int64_t upper_count(int n) {
  const int64_t T = tiles_of(n);
  return T * (T + 1) / 2;
}

// ----------------------------------------------------- non-finite check
__global__ void __launch_bounds__(kThreads) check_kernel(const shampoo_tensor_t* tensors,
                                                         const shampoo_block_t* blocks, int* flag) {
  const int b = blockIdx.x / kChunks, c = blockIdx.x % kChunks;
  const shampoo_block_t blk = blocks[b];
  const shampoo_tensor_t ten = tensors[blk.tensor_id];
  const int rows_per = (blk.rows + kChunks - 1) / kChunks;
  const int r0 = c * rows_per, r1 = min(blk.rows, r0 + rows_per);
  if (r0 >= r1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int bad = 0;
  for (int r = r0 + warp; r < r1; r += kThreads / 32) {
    const float* row = ten.G + (blk.row0 + r) * ten.ldg + blk.col0;
    for (int col = lane; col < blk.cols; col += 32) bad |= !isfinite(__ldg(row + col));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag + b, 1);
}

// ----------------------------------------------------- tile prefix sums
// Single CTA of 1024 threads: chunked exclusive scans of the per-block tile
// counts and of the widened-operand sizes.
SHP_DEV int64_t rupd(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

SHP_DEV void block_sizes(const shampoo_block_t& blk, int only_owner, int64_t& tiles, int64_t& szl, int64_t& szr) {
  const bool l = blk.p_left && (only_owner < 0 || blk.owner_left == only_owner);
  const bool r = blk.p_right && (only_owner < 0 || blk.owner_right == only_owner);
  tiles = (l ? upper_count(blk.rows) : 0) + (r ? upper_count(blk.cols) : 0);
  szl = l ? rupd(blk.rows, 64) * rupd(blk.cols, 32) : 0;
  szr = r ? rupd(blk.cols, 64) * rupd(blk.rows, 32) : 0;
}

__global__ void __launch_bounds__(1024) prep_kernel(const shampoo_block_t* blocks, int n_blocks, int only_owner,
                                                    int64_t* prefix, int64_t* offL, int64_t* offR) {
  __shared__ int64_t pt[1024], pw[1024];
  const int t = threadIdx.x;
  const int per = (n_blocks + 1023) / 1024;
  const int b0 = t * per, b1 = min(n_blocks, b0 + per);
  int64_t st = 0, sw = 0;
  for (int b = b0; b < b1; ++b) {
    int64_t tl, zl, zr;
    block_sizes(blocks[b], only_owner, tl, zl, zr);
    st += tl;
    sw += zl + zr;
  }
  pt[t] = st;
  pw[t] = sw;
  __syncthreads();
  if (t == 0) {
    int64_t a = 0, c = 0;
    for (int i = 0; i < 1024; ++i) {
      const int64_t v = pt[i], u = pw[i];
      pt[i] = a;
      pw[i] = c;
      a += v;
      c += u;
    }
    prefix[n_blocks] = a;
  }
  __syncthreads();
  int64_t a = pt[t], c = pw[t];
  for (int b = b0; b < b1; ++b) {
    prefix[b] = a;
    int64_t tl, zl, zr;
    block_sizes(blocks[b], only_owner, tl, zl, zr);
    offL[b] = zl ? c : -1;
    offR[b] = zr ? c + zl : -1;
    a += tl;
    c += zl + zr;
  }
}

// ------------------------------------------------- widen fp32 -> fp64 panels
// For every owned side: GL = G_b (rows_p64 x kp, kp = roundup(cols, 32)) and
// GR = G_b^T (cols_p64 x roundup(rows, 32)), zero-padded; 64x64 tiles through
// shared memory so both the straight and the transposed writes are coalesced.
constexpr int kWideCTAs = 64;

__global__ void __launch_bounds__(256) widen_kernel(const shampoo_tensor_t* tensors, const shampoo_block_t* blocks,
                                                    const int* flag, const int64_t* offL, const int64_t* offR,
                                                    double* wide) {
  __shared__ float tile[64][65];
  const int b = blockIdx.x / kWideCTAs, c = blockIdx.x % kWideCTAs;
  if (flag[b] || (offL[b] < 0 && offR[b] < 0)) return;
  const shampoo_block_t blk = blocks[b];
  const shampoo_tensor_t ten = tensors[blk.tensor_id];
  const int tr = (blk.rows + 63) / 64, tc = (blk.cols + 63) / 64;
  const int kpl = (int)rupd(blk.cols, 32), kpr = (int)rupd(blk.rows, 32);
  for (int t = c; t < tr * tc; t += kWideCTAs) {
    const int i0 = (t / tc) * 64, j0 = (t % tc) * 64;
    for (int e = threadIdx.x; e < 64 * 64; e += 256) {
      const int i = e >> 6, j = e & 63;
      const bool v = i0 + i < blk.rows && j0 + j < blk.cols;
      tile[i][j] = v ? ten.G[(blk.row0 + i0 + i) * ten.ldg + blk.col0 + j0 + j] : 0.0f;
    }
    __syncthreads();
    if (offL[b] >= 0) {  // rows i0.., columns j0.. (< kpl)
      double* dst = wide + offL[b];
      for (int e = threadIdx.x; e < 64 * 64; e += 256) {
        const int i = e >> 6, j = e & 63;
        if (j0 + j < kpl) dst[(int64_t)(i0 + i) * kpl + j0 + j] = (double)tile[i][j];
      }
    }
    if (offR[b] >= 0) {  // rows j0.. of G^T, columns i0.. (< kpr)
      double* dst = wide + offR[b];
      for (int e = threadIdx.x; e < 64 * 64; e += 256) {
        const int j = e >> 6, i = e & 63;
        if (i0 + i < kpr) dst[(int64_t)(j0 + j) * kpr + i0 + i] = (double)tile[i][j];
      }
    }
    __syncthreads();
  }
}

SHP_DEV int find_block(const int64_t* prefix, int n_blocks, int64_t item) {
  int lo = 0, hi = n_blocks - 1;  // largest b with prefix[b] <= item
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= item) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ------------------------------------------------------------ statistics
__global__ void __launch_bounds__(kNThreads, 2)
    stats_kernel(const shampoo_block_t* blocks, int n_blocks, int only_owner, float* stats, double decay,
                 double weight, const int* flag, const int64_t* prefix, const int64_t* offL, const int64_t* offR,
                 const double* wide) {
  extern __shared__ __align__(16) double smem[];
  const int64_t total = prefix[n_blocks];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tile -> block lookups binary-search the prefix array; keep it in shared
  // memory (after the GEMM buffers) when it fits, instead of 9 dependent
  // global loads at every tile start
  int64_t* spre = reinterpret_cast<int64_t*>(smem + kAsyncSmemDoubles);
  const bool pre_in_smem = n_blocks + 1 <= kPrefixSmem;
  if (pre_in_smem)
    for (int i = threadIdx.x; i <= n_blocks; i += kNThreads) spre[i] = prefix[i];
  __syncthreads();
  const int64_t* pre = pre_in_smem ? spre : prefix;
  AccN acc;
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
    const int b = find_block(pre, n_blocks, item);
    const shampoo_block_t blk = blocks[b];
    if (flag[b]) continue;  // uniform across the CTA
    int64_t local = item - pre[b];
    const bool has_l = blk.p_left && (only_owner < 0 || blk.owner_left == only_owner);
    int side = 1;
    if (has_l) {
      const int64_t nl = upper_count(blk.rows);
      if (local < nl) side = 0;
      else local -= nl;
    }
    const int nvalid = side == 0 ? blk.rows : blk.cols;
    const int K = side == 0 ? blk.cols : blk.rows;
    int ti, tj;
    upper_tile((int)local, tiles_of(nvalid), ti, tj);
    // widened, zero-padded fp64 panels (K padded with zeros at its END: the
    // ascending-k sequential sum is unchanged)
    const int kp = (int)rupd(K, 32);
    const double* base = wide + (side == 0 ? offL[b] : offR[b]);
    float* S = stats + (side == 0 ? blk.left_off : blk.right_off);
    const int64_t ld = side == 0 ? blk.left_ld : blk.right_ld;
    gemm_tile_f64(acc, base + (int64_t)ti * kNT * kp, base + (int64_t)tj * kNT * kp, kp, kp / kAsyncK, smem);
    // epilogue: EMA with the fixed rounding sequence, upper triangle + mirror
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int i = ti * kNT + accn_row(warp, lane, mt);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = tj * kNT + accn_col(warp, lane, nt, e);
          if (i < nvalid && j < nvalid && i <= j) {
            const double old = (double)S[(int64_t)i * ld + j];
            const double t1 = __dmul_rn(weight, acc.c[mt][nt][e]);
            const double t2 = __dmul_rn(decay, old);
            const float r = __double2float_rn(__dadd_rn(t1, t2));
            S[(int64_t)i * ld + j] = r;
            if (i != j) S[(int64_t)j * ld + i] = r;
          }
        }
    }
  }
}

// ------------------------------------------------ D update + graft partials
// HBM-bound (read G, D; write D: 12 B per element).  A warp owns a row; lanes
// take float4 column chunks (two in flight) when the row is 16-B aligned, else
// scalars.  The numerator is summed in a fixed order (per lane, then the
// fixed butterfly, then the warps in order).
__global__ void __launch_bounds__(kThreads) diag_kernel(const shampoo_tensor_t* tensors,
                                                        const shampoo_block_t* blocks, const int* flag,
                                                        double* part) {
  const int b = blockIdx.x / kChunks, c = blockIdx.x % kChunks;
  __shared__ double red[kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const shampoo_block_t blk = blocks[b];
  const shampoo_tensor_t ten = tensors[blk.tensor_id];
  const int rows_per = (blk.rows + kChunks - 1) / kChunks;
  const int r0 = c * rows_per, r1 = min(blk.rows, r0 + rows_per);
  double num = 0.0;
  auto one = [&](float gf, float& d) {
    const double g = (double)gf;
    const double gg = __dmul_rn(g, g);
    const float dn = __double2float_rn(__dadd_rn((double)d, gg));
    d = dn;
    const double den = (double)dn > 1e-30 ? (double)dn : 1e-30;
    num = __dadd_rn(num, __ddiv_rn(gg, den));
  };
  if (!flag[b] && ten.D != nullptr && r0 < r1) {
    for (int r = r0 + warp; r < r1; r += kThreads / 32) {
      const float* grow = ten.G + (blk.row0 + r) * ten.ldg + blk.col0;
      float* drow = ten.D + (blk.row0 + r) * ten.ldd + blk.col0;
      const bool vec = ((reinterpret_cast<uintptr_t>(grow) | reinterpret_cast<uintptr_t>(drow)) & 15) == 0;
      int col = 0;
      if (vec) {
        const int c4 = blk.cols & ~3;
        for (col = 4 * lane; col + 128 < c4; col += 256) {
          const float4 g0 = __ldg(reinterpret_cast<const float4*>(grow + col));
          const float4 g1 = __ldg(reinterpret_cast<const float4*>(grow + col + 128));
          float4 d0 = *reinterpret_cast<const float4*>(drow + col);
          float4 d1 = *reinterpret_cast<const float4*>(drow + col + 128);
          one(g0.x, d0.x); one(g0.y, d0.y); one(g0.z, d0.z); one(g0.w, d0.w);
          one(g1.x, d1.x); one(g1.y, d1.y); one(g1.z, d1.z); one(g1.w, d1.w);
          *reinterpret_cast<float4*>(drow + col) = d0;
          *reinterpret_cast<float4*>(drow + col + 128) = d1;
        }
        for (; col < c4; col += 128) {
          const float4 g0 = __ldg(reinterpret_cast<const float4*>(grow + col));
          float4 d0 = *reinterpret_cast<const float4*>(drow + col);
          one(g0.x, d0.x); one(g0.y, d0.y); one(g0.z, d0.z); one(g0.w, d0.w);
          *reinterpret_cast<float4*>(drow + col) = d0;
        }
        col = c4 + lane;  // scalar tail
      } else {
        col = lane;
      }
      for (; col < blk.cols; col += 32) one(__ldg(grow + col), drow[col]);
    }
  }
  num = warp_sum_fixed(num);
  if (lane == 0) red[warp] = num;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s = __dadd_rn(s, red[w]);
    part[(int64_t)b * kChunks + c] = s;
  }
}

__global__ void finish_kernel(int n_blocks, const int* flag, const double* part, double* graft_num,
                              int32_t* block_status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  double s = 0.0;
  for (int c = 0; c < kChunks; ++c) s = __dadd_rn(s, part[(int64_t)b * kChunks + c]);
  if (graft_num) graft_num[b] = flag[b] ? 0.0 : s;
  if (block_status) block_status[b] = flag[b] ? 2 : 0;
}

int stats_launch(const shampoo_tensor_t* tensors, int n_tensors, const shampoo_block_t* blocks, int n_blocks,
                 int only_owner, float* stats, double decay, double weight, double* graft_num, int32_t* block_status,
                 void* ws, cudaStream_t stream, int64_t* launches) {
  (void)n_tensors;
  if (n_blocks == 0) return SHAMPOO_OK;
  StatsWs w = carve(ws, n_blocks);
  const size_t smem_max = (size_t)kAsyncSmemDoubles * sizeof(double) + (size_t)kPrefixSmem * sizeof(int64_t);
  const size_t smem =
      (size_t)kAsyncSmemDoubles * sizeof(double) + (size_t)std::min(n_blocks + 1, kPrefixSmem) * sizeof(int64_t);
  if (ensure_smem((const void*)stats_kernel, smem_max) != cudaSuccess)
    return set_cuda_error("cudaFuncSetAttribute(stats_kernel)");
  if (cudaMemsetAsync(w.flag, 0, (size_t)n_blocks * sizeof(int), stream) != cudaSuccess)
    return set_cuda_error("cudaMemsetAsync");
  const unsigned eg = (unsigned)n_blocks * kChunks;
  check_kernel<<<eg, kThreads, 0, stream>>>(tensors, blocks, w.flag);
  prep_kernel<<<1, 1024, 0, stream>>>(blocks, n_blocks, only_owner, w.prefix, w.offL, w.offR);
  widen_kernel<<<(unsigned)n_blocks * kWideCTAs, 256, 0, stream>>>(tensors, blocks, w.flag, w.offL, w.offR, w.wide);
  stats_kernel<<<2 * num_sms(), kNThreads, smem, stream>>>(blocks, n_blocks, only_owner, stats, decay, weight, w.flag,
                                                           w.prefix, w.offL, w.offR, w.wide);
  diag_kernel<<<eg, kThreads, 0, stream>>>(tensors, blocks, w.flag, w.part);
  finish_kernel<<<(n_blocks + 255) / 256, 256, 0, stream>>>(n_blocks, w.flag, w.part, graft_num, block_status);
  *launches += 6;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("stats kernels", e);
  return SHAMPOO_OK;
}

}  // namespace shp
