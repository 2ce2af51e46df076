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
#include "dmma_gemm.cuh"
#include "internal.h"

namespace shp {

constexpr int kPChunks = 64;

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct PrecWs {
  int64_t* pre1;  // n_blocks + 1 phase-1 tiles
  int64_t* pre2;  // n_blocks + 1 phase-2 tiles
  int64_t* yoff;  // n_blocks + 1 Y offsets (elements)
  double* part;   // n_blocks * kPChunks
  float* Y;
};

static size_t y_elems(const shampoo_block_t* blocks, int n_blocks) {
  size_t s = 0;
  for (int b = 0; b < n_blocks; ++b)
    if (blocks[b].p_left && blocks[b].p_right) s += (size_t)blocks[b].rows * blocks[b].cols;
  return s;
}

static size_t fixed_bytes(int n_blocks) {
  return 3 * al((size_t)(n_blocks + 1) * sizeof(int64_t)) + al((size_t)n_blocks * kPChunks * sizeof(double));
}

size_t precondition_workspace_bytes(const shampoo_block_t* blocks_host, int n_blocks) {
  return fixed_bytes(n_blocks) + al(y_elems(blocks_host, n_blocks) * sizeof(float));
}

static PrecWs carve(void* ws, int n_blocks) {
  char* q = static_cast<char*>(ws);
  PrecWs w;
  const size_t pb = al((size_t)(n_blocks + 1) * sizeof(int64_t));
  w.pre1 = reinterpret_cast<int64_t*>(q);
  q += pb;
  w.pre2 = reinterpret_cast<int64_t*>(q);
  q += pb;
  w.yoff = reinterpret_cast<int64_t*>(q);
  q += pb;
  w.part = reinterpret_cast<double*>(q);
  q += al((size_t)n_blocks * kPChunks * sizeof(double));
  w.Y = reinterpret_cast<float*>(q);
  return w;
}

SHP_DEV int ntile(int n) { return (n + kTileM - 1) / kTileM; }

SHP_DEV void block_counts(const shampoo_block_t& b, int64_t& n1, int64_t& n2, int64_t& ny) {
  const int64_t t = (int64_t)ntile(b.rows) * ntile(b.cols);
  n1 = b.p_left ? t : 0;
  n2 = b.p_right ? t : 0;
  ny = (b.p_left && b.p_right) ? (int64_t)b.rows * b.cols : 0;
}

__global__ void __launch_bounds__(1024) prec_prep_kernel(const shampoo_block_t* blocks, int n_blocks,
                                                         int64_t* pre1, int64_t* pre2, int64_t* yoff) {
  __shared__ int64_t s1[1024], s2[1024], s3[1024];
  const int t = threadIdx.x;
  const int per = (n_blocks + 1023) / 1024;
  const int b0 = t * per, b1 = min(n_blocks, b0 + per);
  int64_t a1 = 0, a2 = 0, a3 = 0;
  for (int b = b0; b < b1; ++b) {
    int64_t n1, n2, ny;
    block_counts(blocks[b], n1, n2, ny);
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
    block_counts(blocks[b], n1, n2, ny);
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

int precondition_launch(const shampoo_tensor_t* tensors, int n_tensors, const shampoo_block_t* blocks, int n_blocks,
                        const float* roots, const double* graft_num, float* graft_scale, double* den, void* ws,
                        size_t ws_bytes, cudaStream_t stream, int64_t* launches) {
  (void)n_tensors;
  (void)ws_bytes;
  if (n_blocks == 0) return SHAMPOO_OK;
  PrecWs w = carve(ws, n_blocks);
  const size_t smem = (size_t)kGemmSmemDoubles * sizeof(double);
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(prec_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(prec_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
      return set_cuda_error("cudaFuncSetAttribute(prec_gemm_kernel)");
    configured = true;
  }
  const unsigned eg = (unsigned)n_blocks * kPChunks;
  prec_prep_kernel<<<1, 1024, 0, stream>>>(blocks, n_blocks, w.pre1, w.pre2, w.yoff);
  prec_gemm_kernel<1><<<num_sms(), kThreads, smem, stream>>>(tensors, blocks, n_blocks, roots, w.pre1, w.yoff, w.Y);
  prec_gemm_kernel<2><<<num_sms(), kThreads, smem, stream>>>(tensors, blocks, n_blocks, roots, w.pre2, w.yoff, w.Y);
  prec_diag_kernel<<<eg, kThreads, 0, stream>>>(tensors, blocks);
  prec_den_kernel<<<eg, kThreads, 0, stream>>>(tensors, blocks, w.part);
  prec_finish_kernel<<<(n_blocks + 255) / 256, 256, 0, stream>>>(n_blocks, w.part, graft_num, graft_scale, den);
  *launches += 6;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("precondition kernels", e);
  return SHAMPOO_OK;
}

}  // namespace shp
