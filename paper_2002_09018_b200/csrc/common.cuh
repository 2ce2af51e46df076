// common.cuh -- shared device helpers for libshampoo (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "shampoo.h"

#define SHP_DEV __device__ __forceinline__

namespace shp {

constexpr int kWarp = 32;

// ----------------------------------------------------------------- DMMA
// mma.sync.m8n8k4.row.col.f64 -> SASS DMMA.8x8x4 on the FP64 tensor pipe.
// Measured on B200 (tools/microbench/fp64_pipes.cu, profiles/r01_fp64_pipes.txt):
// d = fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c)))) bit for bit, i.e. the
// ascending-k sequential fp64 chain; peak 37.1 TFLOP/s (= DFMA peak).
// Fragments: A(8x4 row) lane holds A[lane>>2][lane&3]; B(4x8 col) lane holds
// B[lane&3][lane>>2]; C(8x8) lane holds C[lane>>2][2*(lane&3)+{0,1}].
SHP_DEV void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------- shared memory tile
// Operand tiles are stored as fp64 [kTileM rows][kTileK k] (128 B per row);
// the 16-byte chunk c of row r lives at chunk c ^ X(r), X(r) = 2*(r&3) + ((r>>2)&1).
// * DMMA fragment reads (LDS.64, 8 rows x 4 consecutive k) are served per
//   half-warp: rows q = 0..3 XOR with 0,2,4,6 and rows 4..7 with 1,3,5,7, so the
//   8 (row, chunk) pairs of each half-warp hit 8 distinct chunk positions
//   (1 wavefront per half, the minimum for 256 B).
// * Row-wise stores (8 consecutive rows, same logical chunk) see 8 distinct
//   X values: conflict-free as well.
constexpr int kTileM = 128;
constexpr int kTileK = 16;
constexpr int kTileElems = kTileM * kTileK;  // doubles per operand tile

SHP_DEV int swx(int r) { return ((r & 3) << 1) | ((r >> 2) & 1); }
SHP_DEV int swz(int r, int k) { return r * kTileK + ((((k >> 1) ^ swx(r)) << 1) | (k & 1)); }
// element offset of 16-byte chunk c of row r
SHP_DEV int swc(int r, int c) { return r * kTileK + ((c ^ swx(r)) << 1); }

// ------------------------------------------------------------ misc helpers
SHP_DEV unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }

// atomic max of a non-negative double (or NaN, which sorts above +inf as bits)
SHP_DEV void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), dbits(v));
}

SHP_DEV double fmax_nan(double a, double b) {
  return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000LL) : (b > a ? b : a);
}

SHP_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(0xffffffffu, v, o);
    // NaN-propagating max (NaN compares false)
    v = (v != v || w != w) ? __longlong_as_double(0x7ff8000000000000LL) : (w > v ? w : v);
  }
  return v;
}

SHP_DEV double warp_sum_fixed(double v) {
  // fixed xor-butterfly order: deterministic for a given lane assignment
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
SHP_DEV T ld_nc(const T* p) { return __ldg(p); }

}  // namespace shp
