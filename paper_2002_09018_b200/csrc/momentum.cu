// momentum.cu -- f2: the tail of Algorithm 1 after the preconditioned gradient,
// per block (reading #9):
//   M_t = beta1 M_{t-1} + (1-beta1) D_t^{-1/2} o G_t          (line 12, D floor 1e-30)
//   t > tau:  P_t = beta1 P_{t-1} + (1-beta1) L^{-1/4} G R^{-1/4}   (line 18)
//             eta_t = eta0 ||M_t||_F / ||P_t||_F                    (line 19; 0 if ||P_t|| = 0)
//             W_t = W_{t-1} - eta_t P_t                             (line 20)
//   else:     W_t = W_{t-1} - eta0 M_t                              (lines 22-23)
// Launches: pass 1 (M, P momentum + fixed-order norm partials) -> finish (eta per
// block) -> pass 2 (W update).  Elementwise, HBM-bound; arithmetic in fp64,
// storage fp32.
#include "common.cuh"
#include "internal.h"

namespace shp {

constexpr int kMChunks = 64;
constexpr int kMThreads = 256;

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

size_t momentum_workspace_bytes(int n_blocks) { return al((size_t)n_blocks * kMChunks * 2 * sizeof(double)) + al((size_t)n_blocks * sizeof(double)); }

__global__ void __launch_bounds__(kMThreads) momentum_pass1(const shampoo_tensor_t* tensors, const shampoo_state_t* states,
                                                           const shampoo_block_t* blocks, double beta1, int shampoo_branch,
                                                           double* part) {
  const int b = blockIdx.x / kMChunks, c = blockIdx.x % kMChunks;
  __shared__ double red[2][kMThreads / 32];
  const shampoo_block_t blk = blocks[b];
  const shampoo_tensor_t ten = tensors[blk.tensor_id];
  const shampoo_state_t st = states[blk.tensor_id];
  const int rows_per = (blk.rows + kMChunks - 1) / kMChunks;
  const int r0 = c * rows_per, r1 = min(blk.rows, r0 + rows_per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double sm = 0.0, sp = 0.0;
  const double omb = 1.0 - beta1;
  for (int r = r0 + warp; r < r1; r += kMThreads / 32) {
    const int64_t gr = blk.row0 + r;
    const float* g = ten.G + gr * ten.ldg + blk.col0;
    const float* d = ten.D + gr * ten.ldd + blk.col0;
    float* m = st.M + gr * st.ldm + blk.col0;
    const float* p = ten.P + gr * ten.ldp + blk.col0;
    float* pm = st.Pm + gr * st.ldpm + blk.col0;
    for (int col = lane; col < blk.cols; col += 32) {
      double dv = (double)d[col];
      dv = dv > 1e-30 ? dv : 1e-30;
      const double mn = beta1 * (double)m[col] + omb * ((double)g[col] / sqrt(dv));
      const float mf = (float)mn;
      m[col] = mf;
      sm = fma((double)mf, (double)mf, sm);
      if (shampoo_branch) {
        const double pn = beta1 * (double)pm[col] + omb * (double)p[col];
        const float pf = (float)pn;
        pm[col] = pf;
        sp = fma((double)pf, (double)pf, sp);
      }
    }
  }
  sm = warp_sum_fixed(sm);
  sp = warp_sum_fixed(sp);
  if (lane == 0) {
    red[0][warp] = sm;
    red[1][warp] = sp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, q = 0.0;
    for (int w = 0; w < kMThreads / 32; ++w) {
      a = __dadd_rn(a, red[0][w]);
      q = __dadd_rn(q, red[1][w]);
    }
    part[((int64_t)b * kMChunks + c) * 2] = a;
    part[((int64_t)b * kMChunks + c) * 2 + 1] = q;
  }
}

__global__ void momentum_finish(int n_blocks, const double* part, double eta0, int shampoo_branch, double* eta) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  double a = 0.0, q = 0.0;
  for (int c = 0; c < kMChunks; ++c) {
    a = __dadd_rn(a, part[((int64_t)b * kMChunks + c) * 2]);
    q = __dadd_rn(q, part[((int64_t)b * kMChunks + c) * 2 + 1]);
  }
  double e = eta0;
  if (shampoo_branch) e = (q > 0.0) ? eta0 * sqrt(a) / sqrt(q) : 0.0;
  eta[b] = e;
}

__global__ void __launch_bounds__(kMThreads) momentum_pass2(const shampoo_state_t* states, const shampoo_block_t* blocks,
                                                           int shampoo_branch, const double* eta) {
  const int b = blockIdx.x / kMChunks, c = blockIdx.x % kMChunks;
  const shampoo_block_t blk = blocks[b];
  const shampoo_state_t st = states[blk.tensor_id];
  const double e = eta[b];
  const int rows_per = (blk.rows + kMChunks - 1) / kMChunks;
  const int r0 = c * rows_per, r1 = min(blk.rows, r0 + rows_per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = r0 + warp; r < r1; r += kMThreads / 32) {
    const int64_t gr = blk.row0 + r;
    float* w = st.W + gr * st.ldw + blk.col0;
    const float* dir = shampoo_branch ? st.Pm + gr * st.ldpm + blk.col0 : st.M + gr * st.ldm + blk.col0;
    for (int col = lane; col < blk.cols; col += 32) w[col] = (float)((double)w[col] - e * (double)dir[col]);
  }
}

int momentum_launch(const shampoo_tensor_t* tensors, const shampoo_state_t* states, const shampoo_block_t* blocks,
                    int n_blocks, double beta1, double eta0, int shampoo_branch, double* eta_out, void* ws,
                    cudaStream_t stream, int64_t* launches) {
  if (n_blocks == 0) return SHAMPOO_OK;
  double* part = static_cast<double*>(ws);
  double* eta = eta_out ? eta_out
                        : reinterpret_cast<double*>(static_cast<char*>(ws) + al((size_t)n_blocks * kMChunks * 2 * sizeof(double)));
  const unsigned g = (unsigned)n_blocks * kMChunks;
  momentum_pass1<<<g, kMThreads, 0, stream>>>(tensors, states, blocks, beta1, shampoo_branch, part);
  momentum_finish<<<(n_blocks + 255) / 256, 256, 0, stream>>>(n_blocks, part, eta0, shampoo_branch, eta);
  momentum_pass2<<<g, kMThreads, 0, stream>>>(states, blocks, shampoo_branch, eta);
  *launches += 3;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("momentum kernels", e);
  return SHAMPOO_OK;
}

}  // namespace shp
