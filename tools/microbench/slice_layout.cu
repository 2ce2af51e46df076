// Slicer store-layout probe: a one-row-per-warp M/T slicer (round 2's first tiled slice_mt_kernel) with three plane
// layouts for its int8 stores -- 0 row-major (round 1), 1 tiled k-block major (the GEMM's bulk-copy layout), 2 tiled
// row-block major -- and the library's row-pair slicer (oz::slice_pair_kernel, whole-line stores, layout 1), timed on
// 528 (or argv[1]) 1024^2 fp64 matrices.  Timing only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2002_09018_b200/csrc \
//        tools/microbench/slice_layout.cu -o tools/microbench/bin/slice_layout
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ozaki.cuh"

using namespace shp;

__device__ __forceinline__ int srow_chunk(int q) { return q ^ ((q >> 2) & 1); }

template <int L>
__device__ __forceinline__ int64_t off(int i, int j, int np) {
  if (L == 0) return (int64_t)i * np + j;
  if (L == 1) return oz::tiled_off(i, j, np);
  return ((int64_t)(i >> 6) * (np >> 6) + (j >> 6)) * 4096 + ((i & 63) << 6) + ((((j >> 4) & 3) ^ ((i >> 1) & 3)) << 4) +
         (j & 15);
}

template <int S, int L>
__global__ void __launch_bounds__(128, 4) mt(const double* __restrict__ src, int n, int np, int batch,
                                             int8_t* __restrict__ pm, int8_t* __restrict__ pt, double* sm_,
                                             double* st_, int p) {
  __shared__ __align__(16) double srow[4][1024];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* my = srow[wib];
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t pitch = oz::plane_pitch(np);
  const double pp1 = p + 1, inv_p = 1.0 / p, ninv_p = -inv_p;
  for (int64_t rid = gw; rid < (int64_t)batch * n; rid += nw) {
    const int mat = (int)(rid / n), i = (int)(rid % n);
    const double* row = src + (int64_t)mat * np * np + (int64_t)i * np;
    const int64_t pmat = (int64_t)mat * oz::kSMax * pitch;
    const double tii = ((pp1 - row[i]) * inv_p);
    double mx = 0, mo = 0;
    double4 r[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) r[h] = *reinterpret_cast<const double4*>(row + 4 * (32 * h + lane));
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const int q = 32 * h + lane, j = 4 * q;
      const double a4[4] = {r[h].x, r[h].y, r[h].z, r[h].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        mx = fmax(mx, fabs(a4[t]));
        mo = fmax(mo, (j + t == i) ? 0.0 : fabs(a4[t]));
      }
      reinterpret_cast<double4*>(my)[srow_chunk(q)] = r[h];
    }
    const int e = oz::row_exponent(mx), et = oz::row_exponent(fmax(fabs(tii), mo * inv_p));
    if (lane == 0) {
      sm_[(int64_t)mat * np + i] = ldexp(1.0, e);
      st_[(int64_t)mat * np + i] = ldexp(1.0, et);
    }
    const double sc_m = oz::digit_scale<S>(e), sc_t = oz::digit_scale<S>(et);
    __syncwarp();
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      const int j = 256 * c + 8 * lane;
      double rr[8];
      const double4 a0 = reinterpret_cast<const double4*>(my)[srow_chunk(j >> 2)];
      const double4 a1 = reinterpret_cast<const double4*>(my)[srow_chunk((j >> 2) + 1)];
      rr[0] = a0.x; rr[1] = a0.y; rr[2] = a0.z; rr[3] = a0.w; rr[4] = a1.x; rr[5] = a1.y; rr[6] = a1.z; rr[7] = a1.w;
      uint32_t dig[S][2];
      oz::slice8<S>(rr, sc_m, dig);
#pragma unroll
      for (int s = 0; s < S; ++s)
        *reinterpret_cast<uint2*>(pm + pmat + s * pitch + off<L>(i, j, np)) = make_uint2(dig[s][0], dig[s][1]);
#pragma unroll
      for (int q = 0; q < 8; ++q) rr[q] = (j + q == i) ? tii : rr[q] * ninv_p;
      oz::slice8<S>(rr, sc_t, dig);
#pragma unroll
      for (int s = 0; s < S; ++s)
        *reinterpret_cast<uint2*>(pt + pmat + s * pitch + off<L>(i, j, np)) = make_uint2(dig[s][0], dig[s][1]);
    }
    __syncwarp();
  }
}

template <class K>
static float time_it(K launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;
  }
  if (cudaGetLastError() != cudaSuccess) {
    printf("CUDA error\n");
    exit(1);
  }
  return best;
}

template <int S, int L>
static void run(const double* src, int8_t* pm, int8_t* pt, double* sm, double* st, int batch) {
  const int n = 1024, np = 1024;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const float best = time_it([&] { mt<S, L><<<4 * sms, 128>>>(src, n, np, batch, pm, pt, sm, st, 4); });
  const double bytes = (double)batch * n * n * (8.0 + 2.0 * S);
  printf("S %d one row per warp, layout %d, batch %d: %.3f ms, %.2f TB/s (read fp64 + write 2S planes)\n", S, L, batch,
         best, bytes / (best * 1e-3) / 1e12);
}

// the library's row-pair slicer with W warps per CTA and B pair buffers per warp
template <int S, int MODE, int W, int B>
static void runp(const double* src, int8_t* pm, int8_t* pt, double* sm, double* st, int batch) {
  const int n = 1024, np = 1024;
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = oz::pair_smem<W, B>();
  cudaFuncSetAttribute(oz::slice_pair_kernel<S, MODE, W, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, oz::slice_pair_kernel<S, MODE, W, B>, 32 * W, smem);
  const float best = time_it([&] {
    oz::slice_pair_kernel<S, MODE, W, B><<<per_sm * sms, 32 * W, smem>>>(src, (int64_t)np * np, n, np, batch, nullptr,
                                                                           nullptr, pm, sm, pt, st, 4);
  });
  const double bytes = (double)batch * n * n * (8.0 + (MODE == 2 ? 2.0 : 1.0) * S);
  printf("S %d pair slicer MODE %d, %d warps x %d buffers, %d CTAs/SM, batch %d: %.3f ms, %.2f TB/s\n", S, MODE, W, B,
         per_sm, batch, best, bytes / (best * 1e-3) / 1e12);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const int batch = argc > 1 ? atoi(argv[1]) : 528;
  const size_t mat = (size_t)1024 * 1024;
  double *src, *sm, *st;
  int8_t *pm, *pt;
  if (cudaMalloc(&src, batch * mat * 8) || cudaMalloc(&pm, batch * mat * oz::kSMax) ||
      cudaMalloc(&pt, batch * mat * oz::kSMax) || cudaMalloc(&sm, batch * 1024 * 8) || cudaMalloc(&st, batch * 1024 * 8)) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(src, 0x3f, batch * mat * 8);  // finite doubles (~0.49)
  cudaMemset(pm, 0, batch * mat * oz::kSMax);
  cudaMemset(pt, 0, batch * mat * oz::kSMax);
  run<7, 0>(src, pm, pt, sm, st, batch);
  runp<7, 2, 4, 1>(src, pm, pt, sm, st, batch);
  runp<7, 2, 8, 1>(src, pm, pt, sm, st, batch);
  runp<7, 2, 10, 1>(src, pm, pt, sm, st, batch);
  runp<7, 2, 12, 1>(src, pm, pt, sm, st, batch);
  runp<6, 2, 4, 1>(src, pm, pt, sm, st, batch);
  runp<6, 2, 8, 1>(src, pm, pt, sm, st, batch);
  runp<6, 2, 12, 1>(src, pm, pt, sm, st, batch);
  runp<5, 2, 4, 1>(src, pm, pt, sm, st, batch);
  runp<5, 2, 8, 1>(src, pm, pt, sm, st, batch);
  runp<5, 2, 12, 1>(src, pm, pt, sm, st, batch);
  runp<5, 0, 8, 1>(src, pm, pt, sm, st, batch);
  runp<5, 0, 12, 1>(src, pm, pt, sm, st, batch);
  printf("done\n");
  return 0;
}
