// Microbenchmark: FP64 pipe peaks on B200 (sm_100a) and DMMA rounding semantics.
// Evidence for DESIGN.md's choice of the Newton-product and statistics arithmetic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pipes fp64_pipes.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_peak(double* out, int iters) {
  double a[8];
  double b = 1.0000001 + threadIdx.x * 1e-9, c = 0.999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = i * 0.1 + blockIdx.x * 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_884_peak(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 + blockIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_1684_peak(double* out, int iters) {
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 0.25, b = 0.5 + blockIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_16816_peak(double* out, int iters) {
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + i * 1e-3 + threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i * 1e-3 + blockIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.678) out[0] = s;
}

// Mixed: even warps run DMMA chains, odd warps run DFMA chains -- do the two
// FP64 datapaths (tensor DMMA subpipe vs FP64 ALU pipe) add up?
__global__ void mixed_peak(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double a[8];
    double b = 1.0000001 + threadIdx.x * 1e-9, c = 0.999999;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = i * 0.1 + blockIdx.x * 1e-7;
    for (int it = 0; it < iters * 16; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
  } else {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 + blockIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  }
  if (s == 12345.678) out[0] = s;
}

// Rounding semantics: one m8n8k4 per trial. A row-major 8x4, B col-major (4x8), C 8x8.
__global__ void dmma_semantics(const double* A, const double* B, const double* C, double* D, int trials) {
  int lane = threadIdx.x;
  for (int t = 0; t < trials; ++t) {
    const double* a = A + t * 32; const double* b = B + t * 32; const double* c = C + t * 64;
    double av = a[(lane >> 2) * 4 + (lane & 3)];
    double bv = b[(lane >> 2) * 4 + (lane & 3)];          // B stored as [n][k]
    int r = lane >> 2, c0 = (lane & 3) * 2;
    double d0 = c[r * 8 + c0], d1 = c[r * 8 + c0 + 1];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(av), "d"(bv));
    D[t * 64 + r * 8 + c0] = d0; D[t * 64 + r * 8 + c0 + 1] = d1;
  }
}

template <typename K>
static void timeit(const char* name, K kern, int blocks, int threads, int iters, double flop_per_thread_iter, double* dout) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kern<<<blocks, threads>>>(dout, iters); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0)); kern<<<blocks, threads>>>(dout, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  double flops = flop_per_thread_iter * (double)blocks * threads * iters;
  printf("%-16s blocks=%d threads=%d  %.3f ms  %.2f TFLOP/s\n", name, blocks, threads, best, flops / best / 1e9);
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs=%d l2=%d MB smemOptin=%zu clock=%d kHz\n", prop.name, prop.multiProcessorCount,
         prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin, prop.clockRate);
  double* dout; CK(cudaMalloc(&dout, 64));
  int sms = prop.multiProcessorCount;
  for (int occ : {1, 2, 4}) {
    timeit("dfma", dfma_peak, sms * occ, 256, 20000, 8 * 2.0, dout);
    timeit("dmma_m8n8k4", dmma_884_peak, sms * occ, 256, 20000, 8 * 2.0 * 256 / 32, dout);
    timeit("dmma_m16n8k4", dmma_1684_peak, sms * occ, 256, 20000, 8 * 2.0 * 512 / 32, dout);
    timeit("dmma_m16n8k16", dmma_16816_peak, sms * occ, 256, 10000, 4 * 2.0 * 2048 / 32, dout);
  }
  // mixed: per warp pair, DMMA warp does iters*8*256 FMA, DFMA warp iters*16*8*32 = same count
  for (int occ : {1, 2}) timeit("mixed dmma+dfma", mixed_peak, sms * occ, 256, 10000, 8 * 2.0 * 256 / 32, dout);
  // semantics
  const int T = 4096;
  double *hA = (double*)malloc(T * 32 * 8), *hB = (double*)malloc(T * 32 * 8), *hC = (double*)malloc(T * 64 * 8), *hD = (double*)malloc(T * 64 * 8);
  srand(1234);
  for (int t = 0; t < T; ++t) {
    for (int i = 0; i < 32; ++i) {
      // fp32-representable values with wide exponent spread, mixed signs
      int e1 = rand() % 60 - 30, e2 = rand() % 60 - 30;
      float fa = ldexpf((float)(rand() % (1 << 24)) / (1 << 24) + 0.5f, e1) * ((rand() & 1) ? -1.f : 1.f);
      float fb = ldexpf((float)(rand() % (1 << 24)) / (1 << 24) + 0.5f, e2) * ((rand() & 1) ? -1.f : 1.f);
      hA[t * 32 + i] = fa; hB[t * 32 + i] = fb;
    }
    for (int i = 0; i < 64; ++i) {
      int e = rand() % 60 - 30;
      hC[t * 64 + i] = ldexp((double)rand() / RAND_MAX + 0.5, e) * ((rand() & 1) ? -1. : 1.);
    }
  }
  double *dA, *dB, *dC, *dD;
  CK(cudaMalloc(&dA, T * 32 * 8)); CK(cudaMalloc(&dB, T * 32 * 8)); CK(cudaMalloc(&dC, T * 64 * 8)); CK(cudaMalloc(&dD, T * 64 * 8));
  CK(cudaMemcpy(dA, hA, T * 32 * 8, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, hB, T * 32 * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dC, hC, T * 64 * 8, cudaMemcpyHostToDevice));
  dmma_semantics<<<1, 32>>>(dA, dB, dC, dD, T); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hD, dD, T * 64 * 8, cudaMemcpyDeviceToHost));
  int seq_fwd = 0, seq_rev = 0, total = 0;
  for (int t = 0; t < T; ++t)
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) {
        double acc = hC[t * 64 + r * 8 + c];
        for (int k = 0; k < 4; ++k) acc = fma(hA[t * 32 + r * 4 + k], hB[t * 32 + c * 4 + k], acc);
        double acc2 = hC[t * 64 + r * 8 + c];
        for (int k = 3; k >= 0; --k) acc2 = fma(hA[t * 32 + r * 4 + k], hB[t * 32 + c * 4 + k], acc2);
        double d = hD[t * 64 + r * 8 + c];
        seq_fwd += (d == acc); seq_rev += (d == acc2); total++;
      }
  printf("dmma m8n8k4 semantics: equal to ascending fma chain %d/%d, descending %d/%d\n", seq_fwd, total, seq_rev, total);
  FILE* f = fopen("gpurun_out/dmma_semantics.bin", "wb");
  if (f) { fwrite(hA, 8, T * 32, f); fwrite(hB, 8, T * 32, f); fwrite(hC, 8, T * 64, f); fwrite(hD, 8, T * 64, f); fclose(f); }
  return 0;
}
