// oz_precondition.cu -- the preconditioned gradient of one-sided blocks on the INT8
// tensor cores (row a8: "G R^{-1/2}"): P_b = G_b X_R with fp64-level
// products (Ozaki splitting, ozaki.cuh).
//
// Why not 3xTF32 here: a one-sided block's statistic R_b = G_b^T G_b is often
// rank-deficient (the vocabulary rows of an embedding gradient span few
// dimensions), so X_R = (R_b + eps I)^{-1/2} is largest exactly in the
// directions G_b's rows are orthogonal to and the product cancels those
// components; an fp32 accumulation keeps only ~2^-24 of the uncancelled sum
// (measured on B200: 6.2e-3 relative error on a 4-nonzero-row block, north
// star 1e-3).  Here every product is exact in int32 (6 slices, 2^-41 per
// operand row), then rounded once to fp32.
//
// Per call: slice the rows of every G_b and of every X_R (fp32 sources) into 6
// tiled int8 planes at the kSMax pitch, then one persistent gemm_kernel<6, 64> launch
// per distinct n = cols over all eligible blocks (non-symmetric 128 x 64 tiles,
// fp32 epilogue into P).  The graft denominator is computed afterwards from P
// by precondition.cu's den kernel, as for every other block.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"
#include "ozaki.cuh"
#include "oz_precondition.h"

namespace shp {

constexpr int kOzPrecS = 6;

// One warp per (job, row < np): digits of an fp32 row src[row * ld + j], j < cols
// (zero beyond cols and for rows >= rows), tiled planes of job q at planes + q kSMax plane_pitch(np).
template <int S>
__global__ void __launch_bounds__(256, 2) slice_f32_kernel(const OzSliceJob* __restrict__ jobs, int n_jobs, int np,
                                                           int8_t* __restrict__ planes, double* __restrict__ scale) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t pitch = oz::plane_pitch(np);
  for (int64_t rid = gw; rid < (int64_t)n_jobs * np; rid += nw) {
    const int q = (int)(rid / np), i = (int)(rid - (int64_t)q * np);
    const OzSliceJob J = jobs[q];
    int8_t* pmat = planes + (int64_t)q * oz::kSMax * pitch;
    const bool live = i < J.rows;
    const float* row = J.src + (int64_t)i * J.ld;
    double r[4][8];
    double mx = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = 256 * c + 8 * lane;
#pragma unroll
      for (int e = 0; e < 8; ++e) r[c][e] = (live && j + e < J.cols) ? (double)__ldg(row + j + e) : 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) mx = fmax(mx, fabs(r[c][e]));
    }
    const int e = oz::row_exponent(mx);
    if (lane == 0) scale[(int64_t)q * np + i] = ldexp(1.0, e);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = 256 * c + 8 * lane;
      if (j < np) {
        uint32_t dig[S][2];
        oz::slice8<S>(r[c], oz::digit_scale<S>(e), dig);
#pragma unroll
        for (int s = 0; s < S; ++s) oz::store8(pmat + s * pitch, i, j, np, dig[s]);
      }
    }
  }
}

bool oz_precondition_eligible(const shampoo_block_t& b) {
  // right-only blocks whose rows fit the n x n plane grid (rows <= cols <= 1024: one register-resident row per warp)
  return !b.p_left && b.p_right && b.rows <= b.cols && b.cols <= 1024;
}

static int64_t npad(int n) { return (n + 63) / 64 * 64; }

// Layout of one call: groups of equal n; per group: job tables, planes, scales.
struct OzPrecGroup {
  int n, np, count;
  std::vector<int> blocks;
};

static std::vector<OzPrecGroup> oz_groups(const shampoo_block_t* B, int n_blocks, const int* flags) {
  std::vector<OzPrecGroup> gs;
  for (int b = 0; b < n_blocks; ++b) {
    if (flags[b] != 2) continue;
    const int n = B[b].cols;
    auto it = std::find_if(gs.begin(), gs.end(), [&](const OzPrecGroup& g) { return g.n == n; });
    if (it == gs.end()) {
      gs.push_back({n, (int)npad(n), 0, {}});
      it = gs.end() - 1;
    }
    it->blocks.push_back(b);
    ++it->count;
  }
  return gs;
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t group_bytes(const OzPrecGroup& g) {
  const size_t planes = (size_t)g.count * oz::kSMax * oz::plane_pitch(g.np);
  return 2 * al256(planes) + 2 * al256((size_t)g.count * g.np * sizeof(double)) +
         2 * al256((size_t)g.count * sizeof(OzSliceJob)) + al256((size_t)g.count * sizeof(float*)) +
         al256((size_t)g.count * sizeof(int64_t)) + al256((size_t)g.count * sizeof(int));
}

size_t oz_precondition_bytes(const shampoo_block_t* B, int n_blocks, const int* flags) {
  size_t t = 0;
  for (const OzPrecGroup& g : oz_groups(B, n_blocks, flags)) t += group_bytes(g);
  return t;
}

int oz_precondition_launch(const shampoo_tensor_t* T, const shampoo_block_t* B, int n_blocks, const int* flags,
                           const float* roots, void* ws, cudaStream_t stream, int64_t* launches) {
  const std::vector<OzPrecGroup> gs = oz_groups(B, n_blocks, flags);
  if (gs.empty()) return SHAMPOO_OK;
  constexpr int S = kOzPrecS;
  const size_t smem = oz::gemm_smem_bytes<S, 64>();
  if (ensure_smem((const void*)oz::gemm_kernel<S, 64>, smem) != cudaSuccess)
    return set_cuda_error("cudaFuncSetAttribute(ozaki gemm_kernel, precondition)");
  char* w = static_cast<char*>(ws);
  for (const OzPrecGroup& g : gs) {
    const size_t planes_b = al256((size_t)g.count * oz::kSMax * oz::plane_pitch(g.np));
    const size_t scale_b = al256((size_t)g.count * g.np * sizeof(double));
    int8_t* pg = reinterpret_cast<int8_t*>(w);
    int8_t* px = reinterpret_cast<int8_t*>(w + planes_b);
    double* sg = reinterpret_cast<double*>(w + 2 * planes_b);
    double* sx = reinterpret_cast<double*>(w + 2 * planes_b + scale_b);
    char* q = w + 2 * planes_b + 2 * scale_b;
    OzSliceJob* jg = reinterpret_cast<OzSliceJob*>(q);
    q += al256((size_t)g.count * sizeof(OzSliceJob));
    OzSliceJob* jx = reinterpret_cast<OzSliceJob*>(q);
    q += al256((size_t)g.count * sizeof(OzSliceJob));
    float** outf = reinterpret_cast<float**>(q);
    q += al256((size_t)g.count * sizeof(float*));
    int64_t* outld = reinterpret_cast<int64_t*>(q);
    q += al256((size_t)g.count * sizeof(int64_t));
    int* outrows = reinterpret_cast<int*>(q);
    w += group_bytes(g);
    // host tables: one async copy each (the library stays stateless; the host vectors live until the copies are
    // issued -- pageable sources are staged by cudaMemcpyAsync before it returns)
    std::vector<OzSliceJob> hg(g.count), hx(g.count);
    std::vector<float*> ho(g.count);
    std::vector<int64_t> hl(g.count);
    std::vector<int> hr(g.count);
    for (int k = 0; k < g.count; ++k) {
      const shampoo_block_t& b = B[g.blocks[k]];
      const shampoo_tensor_t& t = T[b.tensor_id];
      hg[k] = {t.G + b.row0 * t.ldg + b.col0, t.ldg, b.rows, b.cols};
      hx[k] = {roots + b.right_off, (int64_t)b.right_ld, b.cols, b.cols};
      ho[k] = t.P + b.row0 * t.ldp + b.col0;
      hl[k] = t.ldp;
      hr[k] = b.rows;
    }
    if (cudaMemcpyAsync(jg, hg.data(), g.count * sizeof(OzSliceJob), cudaMemcpyHostToDevice, stream) ||
        cudaMemcpyAsync(jx, hx.data(), g.count * sizeof(OzSliceJob), cudaMemcpyHostToDevice, stream) ||
        cudaMemcpyAsync(outf, ho.data(), g.count * sizeof(float*), cudaMemcpyHostToDevice, stream) ||
        cudaMemcpyAsync(outld, hl.data(), g.count * sizeof(int64_t), cudaMemcpyHostToDevice, stream) ||
        cudaMemcpyAsync(outrows, hr.data(), g.count * sizeof(int), cudaMemcpyHostToDevice, stream))
      return set_cuda_error("cudaMemcpyAsync(ozaki precondition tables)");
    const int grid = 8 * num_sms();
    slice_f32_kernel<S><<<grid, 256, 0, stream>>>(jg, g.count, g.np, pg, sg);
    slice_f32_kernel<S><<<grid, 256, 0, stream>>>(jx, g.count, g.np, px, sx);
    oz::OzArgs a;
    std::memset(&a, 0, sizeof a);
    a.batch = g.count;
    a.n = g.n;
    a.np = g.np;
    a.tiles_m = (g.n + oz::kBM - 1) / oz::kBM;
    a.tiles_n = (g.n + oz::kBN - 1) / oz::kBN;
    a.sym = 0;
    a.jobs = 1;
    a.p = 1;
    a.job[0].a_planes = pg;
    a.job[0].b_planes = px;
    a.job[0].a_scale = sg;
    a.job[0].b_scale = sx;
    a.job[0].outf = outf;
    a.job[0].outf_ld = outld;
    a.job[0].outf_rows = outrows;
    void* tok;
    prof_begin_launch("ozaki_precondition", stream, &tok);
    oz::gemm_kernel<S, 64><<<num_sms(), oz::kThreads, smem, stream>>>(a);
    prof_end_launch(tok, stream);
    *launches += 3;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("ozaki precondition kernels", e);
  return SHAMPOO_OK;
}

}  // namespace shp
