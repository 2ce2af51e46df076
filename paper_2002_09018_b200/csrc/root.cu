// root.cu -- batched epsilon-regularised inverse p-th roots by the coupled
// Newton iteration (rows a3-a6), one cooperative persistent kernel per batch.
//
// Method ("Schur-Newton ... a sequence of matrix-vector and
// matrix-matrix products", double precision; iteration of S:131; readings
// #1-#4, #16, #18 of DESIGN.md):
//   lambda_hat : power_iters power steps from the splitmix64 start vector
//   A_hat = A + eps_rel*lambda_hat*I ; c = lambda_hat*(1+eps_rel)
//   M_0 = A_hat / c ; X_0 = c^{-1/p} I
//   k = 0, 1, ...: err_k = max|M_k - I| ; stop on err_k <= tol, stagnation
//                  (err_k >= err_{k-1} < 1e-2 -> X_{k-1}) or k == max_iter
//                  T_k = ((p+1)I - M_k)/p ; X_{k+1} = X_k T_k ; M_{k+1} = T_k^p M_k
//   T^p by the left-to-right binary chain (squarings, multiplications by T),
//   any integer p in [1, 16] (reading #22); optionally X <- X^r before the
//   fp32 write (rational exponent -r/p, f4; reading #23).
//
// B200 design:
//  * All iterates are symmetric polynomials in A_hat, so every product computes
//    only the upper-triangle 128x128 tiles and mirror-stores them.
//  * Products run on the FP64 tensor pipe (DMMA.8x8x4) through dmma_gemm.cuh.
//  * One cooperative launch runs power iteration, setup, all iterations and
//    the final fp32 write; grid.sync separates dependent products.  Each CTA
//    keeps an identical copy of the active-matrix list (derived from the err
//    history in global memory), so converged matrices stop issuing tiles with
//    no host round trip.
//  * The M-update epilogue fuses T_{k+1} = ((p+1)I - M_{k+1})/p and the
//    max|M_{k+1} - I| reduction (warp max + one 64-bit atomicMax per warp).
#include <cooperative_groups.h>

#include "dmma_gemm.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace shp {

constexpr int kBufs = 7;  // X0, X1, M0, M1, T, S0, S1
constexpr int kRT = kNThreads;  // threads per root-kernel CTA (2 CTAs per SM)
enum { BX0 = 0, BX1 = 1, BM0 = 2, BM1 = 3, BT = 4, BS0 = 5, BS1 = 6 };
constexpr double kStagnationGate = 1e-2;
constexpr int kMaxBatchPerLaunch = 2048;

struct RootArgs {
  const float* A;
  int64_t lda, stride_a;
  float* X;
  int64_t ldx, stride_x;
  int batch, n, np, p, r, max_iter, power_iters;
  int k_sw;  // hybrid: matrices still iterating at check k_sw are handed to the 3xTF32 tail (> max_iter: off)
  int handoff_fp64;  // ozaki: hand off at k_sw = 0 with the fp64 buffers left as they are
  double eps_rel, tol;
  shampoo_root_info_t* info;
  double* bufs;  // batch * kBufs * np * np
  double* lam;   // batch
  double* errh;  // batch * (max_iter + 1)
  int4* res;     // batch: {result buffer, iters, status, -}
  double* wpi;   // 2 * batch * n: power-iteration w vectors (split mode, ping-pong)
  int* tail_act;  // hybrid: batch (active list of the tail)
  int* tail_nact;
};

SHP_DEV double* buf(const RootArgs& a, int mat, int b) {
  return a.bufs + ((int64_t)mat * kBufs + b) * (int64_t)a.np * a.np;
}

// ------------------------------------------------------------ decisions
enum { D_CONTINUE = 0, D_CONVERGED = 1, D_STAGNATED = 2, D_MAXITER = 3, D_NONFINITE = 4 };

SHP_DEV int decide(const RootArgs& a, int mat, int k) {
  const double* e = a.errh + (int64_t)mat * (a.max_iter + 1);
  double ek = e[k];
  if (!isfinite(ek)) return D_NONFINITE;
  if (ek <= a.tol) return D_CONVERGED;
  if (k >= 1) {
    double ep = e[k - 1];
    if (ek >= ep && ep < kStagnationGate) return D_STAGNATED;
  }
  if (k == a.max_iter) return D_MAXITER;
  return D_CONTINUE;
}

// ------------------------------------------------------- power iteration
SHP_DEV uint64_t splitmix64(uint64_t i) {
  uint64_t z = i + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Deterministic block reduction (fixed lane/warp order); result broadcast.
SHP_DEV double block_sum(double v, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum_fixed(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kRT / 32; ++w) s = __dadd_rn(s, red[w]);
  return s;
}

// ---- power-iteration pieces.  Every w[r] is one warp's fixed-lane-order dot
// product and every scalar reduction runs the same 128-thread block_sum over
// the full vectors, so lambda_hat is bit-identical whether one CTA or several
// CTAs compute a matrix's rows (batch-size independent results).
SHP_DEV void pi_init(double* v, int n, double* red) {
  double part = 0.0;
  for (int i = threadIdx.x; i < n; i += kRT) {
    const double x = (double)(splitmix64((uint64_t)i) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    v[i] = x;
    part = fma(x, x, part);
  }
  const double nv = sqrt(block_sum(part, red));
  for (int i = threadIdx.x; i < n; i += kRT) v[i] = v[i] / nv;
  __syncthreads();
}

// w[r] = sum_c A[r][c] v[c] for r in [r0, r1)
SHP_DEV void pi_rows(const RootArgs& a, const float* A, const double* v, double* w, int r0, int r1) {
  const int n = a.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool vec4 = ((a.lda & 3) == 0) && ((n & 3) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  if (vec4) {
    // kPR rows per warp pass x 4 column chunks (128 floats each) per row: 4*kPR
    // float4 loads in flight per lane; each lane accumulates its columns in
    // ascending order.
    constexpr int kPR = 8;
    for (int rb = r0 + warp * kPR; rb < r1; rb += kPR * (kRT / 32)) {
      double acc[kPR];
      const float* rows[kPR];
#pragma unroll
      for (int q = 0; q < kPR; ++q) {
        acc[q] = 0.0;
        rows[q] = A + (int64_t)min(rb + q, r1 - 1) * a.lda;
      }
      int c = 4 * lane;
      for (; c + 3 * 128 < n; c += 4 * 128) {
        float4 f[kPR][4];
#pragma unroll
        for (int q = 0; q < kPR; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) f[q][u] = __ldg(reinterpret_cast<const float4*>(rows[q] + c + u * 128));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int cc = c + u * 128;
          const double v0 = v[cc], v1 = v[cc + 1], v2 = v[cc + 2], v3 = v[cc + 3];
#pragma unroll
          for (int q = 0; q < kPR; ++q) {
            acc[q] = fma((double)f[q][u].x, v0, acc[q]);
            acc[q] = fma((double)f[q][u].y, v1, acc[q]);
            acc[q] = fma((double)f[q][u].z, v2, acc[q]);
            acc[q] = fma((double)f[q][u].w, v3, acc[q]);
          }
        }
      }
      for (; c < n; c += 128) {
#pragma unroll
        for (int q = 0; q < kPR; ++q) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(rows[q] + c));
          acc[q] = fma((double)f.x, v[c], acc[q]);
          acc[q] = fma((double)f.y, v[c + 1], acc[q]);
          acc[q] = fma((double)f.z, v[c + 2], acc[q]);
          acc[q] = fma((double)f.w, v[c + 3], acc[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < kPR; ++q) {
        const double sum = warp_sum_fixed(acc[q]);
        if (lane == 0 && rb + q < r1) w[rb + q] = sum;
      }
    }
  } else {
    for (int r = r0 + warp; r < r1; r += kRT / 32) {
      const float* row = A + (int64_t)r * a.lda;
      double acc = 0.0;
#pragma unroll 4
      for (int c = lane; c < n; c += 32) acc = fma((double)__ldg(row + c), v[c], acc);
      acc = warp_sum_fixed(acc);
      if (lane == 0) w[r] = acc;
    }
  }
}

// lam = v.w, nw = |w|; v <- w/nw unless nw == 0 (or NaN-free zero).  Returns false
// when the iteration must stop (|w| == 0), as the oracle's `break`.
SHP_DEV bool pi_update(double* v, const double* w, int n, double* red, double& lam) {
  double pl = 0.0, pw = 0.0;
  for (int i = threadIdx.x; i < n; i += kRT) {
    pl = fma(v[i], w[i], pl);
    pw = fma(w[i], w[i], pw);
  }
  lam = block_sum(pl, red);
  const double nw = sqrt(block_sum(pw, red));
  if (!(nw != 0.0)) return false;  // also stops on NaN (lam is then NaN)
  for (int i = threadIdx.x; i < n; i += kRT) v[i] = w[i] / nw;
  __syncthreads();
  return true;
}

// One CTA: lambda_hat of matrix `mat` (smem: v[n], w[n], red[8]).
SHP_DEV double power_iteration(const RootArgs& a, int mat, double* smem) {
  const int n = a.n;
  double* v = smem;
  double* w = smem + n;
  double* red = smem + 2 * n;
  const float* A = a.A + (int64_t)mat * a.stride_a;
  pi_init(v, n, red);
  double lam = 0.0;
  for (int it = 0; it < a.power_iters; ++it) {
    pi_rows(a, A, v, w, 0, n);
    __syncthreads();
    if (!pi_update(v, w, n, red, lam)) break;
  }
  __syncthreads();
  return lam;
}

// Split mode (batch < grid): `k` CTAs share each matrix's rows; w goes through
// global memory (ping-pong) with one grid.sync per power step; every CTA of a
// matrix then runs the same pi_update on the full vectors.
SHP_DEV void power_iteration_split(const RootArgs& a, double* smem, cg::grid_group& grid) {
  const int n = a.n, k = gridDim.x / a.batch;
  const int mat = blockIdx.x / k, part = blockIdx.x % k;
  const bool active = mat < a.batch;
  double* v = smem;
  double* w = smem + n;
  double* red = smem + 2 * n;
  const int rows_per = ((n + k - 1) / k + 7) / 8 * 8;
  const int r0 = min(n, part * rows_per), r1 = min(n, r0 + rows_per);
  const float* A = active ? a.A + (int64_t)mat * a.stride_a : nullptr;
  if (active) pi_init(v, n, red);
  double lam = 0.0;
  bool running = true;
  for (int it = 0; it < a.power_iters; ++it) {
    double* wg = a.wpi + ((int64_t)(it & 1) * a.batch + (active ? mat : 0)) * n;
    if (active && running) pi_rows(a, A, v, wg, r0, r1);
    grid.sync();
    if (active && running) {
      for (int i = threadIdx.x; i < n; i += kRT) w[i] = wg[i];
      __syncthreads();
      running = pi_update(v, w, n, red, lam);
    }
  }
  if (active && part == 0 && threadIdx.x == 0) a.lam[mat] = lam;
}

// c^{-1/p}: sqrt chains for p = 2^j (exact scale equivariance), pow otherwise
SHP_DEV double c_pow_neg_inv_p(double c, int p) {
  if ((p & (p - 1)) == 0) {
    double x = c;
    for (int q = p; q > 1; q >>= 1) x = sqrt(x);
    return 1.0 / x;
  }
  return pow(c, -1.0 / (double)p);
}

SHP_DEV int lead_bit(int p) { return 31 - __clz(p); }

SHP_DEV bool lam_ok(double lam) { return isfinite(lam) && lam > 0.0; }

// ------------------------------------------------------------ epilogues
enum { EPI_STORE = 0, EPI_MUPDATE = 1 };

template <int MODE>
SHP_DEV void epilogue(const RootArgs& a, const AccN& acc, int mat, int ti, int tj, double* dst, double* tdst,
                      double* err_slot) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = a.np, n = a.n;
  const bool mirror = ti != tj;
  const double inv_p = 1.0 / (double)a.p;
  const double pp1 = (double)(a.p + 1);
  double emax = 0.0;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int i = ti * kNT + accn_row(warp, lane, mt);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int j = tj * kNT + accn_col(warp, lane, nt, 0);
      const double c0 = acc.c[mt][nt][0], c1 = acc.c[mt][nt][1];
      *reinterpret_cast<double2*>(dst + (int64_t)i * np + j) = make_double2(c0, c1);
      if (mirror) {
        dst[(int64_t)j * np + i] = c0;
        dst[(int64_t)(j + 1) * np + i] = c1;
      }
      if (MODE == EPI_MUPDATE) {
        const bool iv = i < n;
        const bool v0 = iv && j < n, v1 = iv && j + 1 < n;
        const double d0 = (i == j) ? 1.0 : 0.0, d1 = (i == j + 1) ? 1.0 : 0.0;
        const double t0 = v0 ? (pp1 * d0 - c0) * inv_p : 0.0;
        const double t1 = v1 ? (pp1 * d1 - c1) * inv_p : 0.0;
        *reinterpret_cast<double2*>(tdst + (int64_t)i * np + j) = make_double2(t0, t1);
        if (mirror) {
          tdst[(int64_t)j * np + i] = t0;
          tdst[(int64_t)(j + 1) * np + i] = t1;
        }
        if (v0) emax = fmax_nan(emax, fabs(c0 - d0));
        if (v1) emax = fmax_nan(emax, fabs(c1 - d1));
      }
    }
  }
  if (MODE == EPI_MUPDATE) {
    emax = warp_max(emax);
    if (lane == 0) atomic_max_nonneg(err_slot, emax);
  }
}

// Ordered compaction of the active list: keep act[pos] iff the matrix may
// continue at check k.  Every CTA computes the same result from global state.
SHP_DEV int compact(const RootArgs& a, int* act, int nact, int k, int* cnt, bool first) {
  const int per = (nact + kRT - 1) / kRT;
  const int b0 = threadIdx.x * per;
  int mine[kMaxBatchPerLaunch / kRT];
  int nm = 0;
  for (int q = 0; q < per; ++q) {
    const int pos = b0 + q;
    if (pos < nact) {
      const int mat = act[pos];
      const bool keep = (!first || lam_ok(a.lam[mat])) && decide(a, mat, k) == D_CONTINUE && k < a.k_sw;
      if (keep) mine[nm++] = mat;
    }
  }
  cnt[threadIdx.x] = nm;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int i = 0; i < kRT; ++i) {
      const int c = cnt[i];
      cnt[i] = s;
      s += c;
    }
    cnt[kRT] = s;
  }
  __syncthreads();
  const int out = cnt[threadIdx.x];
  for (int q = 0; q < nm; ++q) act[out + q] = mine[q];
  const int total = cnt[kRT];
  __syncthreads();
  return total;
}

// One symmetric product stage over the active matrices: D = A_op * B_op
// (upper 64x64 tiles, mirror-stored).  An operand index < 0 selects the
// matrix's returned iterate (a.res[mat].x).
SHP_DEV void product_stage(const RootArgs& a, const int* act, int nact, int ab, int bb, int db, double* smem,
                           AccN& acc) {
  const int np = a.np, T = np / kNT, tiles = T * (T + 1) / 2;
  const int items = nact * tiles;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int pos = it / tiles, t = it - pos * tiles;
    const int mat = act[pos];
    int ti, tj;
    upper_tile(t, T, ti, tj);
    const int ra = ab < 0 ? a.res[mat].x : ab, rb = bb < 0 ? a.res[mat].x : bb;
    gemm_tile_f64(acc, buf(a, mat, ra) + (int64_t)ti * kNT * np, buf(a, mat, rb) + (int64_t)tj * kNT * np, np,
                  np / kAsyncK, smem);
    epilogue<EPI_STORE>(a, acc, mat, ti, tj, buf(a, mat, db), nullptr, nullptr);
  }
}

SHP_DEV void write_output(const RootArgs& a, int pbuf);
SHP_DEV void tail_handoff(const RootArgs& a);

// ---------------------------------------------------------------- kernel
// kOz: the Ozaki root's prologue (power iteration, setup, the k = 0 decision and
// handoff) without the FP64-DMMA iteration code, so it needs far fewer registers
// and no GEMM shared memory: more CTAs per SM for the latency-bound power sweeps.
template <bool kOz>
__global__ void __launch_bounds__(kRT, kOz ? 4 : 2) root_kernel(RootArgs a) {
  extern __shared__ __align__(16) double smem[];
  cg::grid_group grid = cg::this_grid();
  const int np = a.np, T = np / kNT, tiles = T * (T + 1) / 2;

  // ---- phase 0: power iteration + err history reset
  for (int mat = blockIdx.x; mat < a.batch; mat += gridDim.x) {
    double* e = a.errh + (int64_t)mat * (a.max_iter + 1);
    for (int k = threadIdx.x; k <= a.max_iter; k += kRT) e[k] = 0.0;
  }
  if (2 * a.batch <= (int)gridDim.x) {
    power_iteration_split(a, smem, grid);  // small batch: several CTAs per matrix
  } else {
    for (int mat = blockIdx.x; mat < a.batch; mat += gridDim.x) {
      const double lam = power_iteration(a, mat, smem);
      if (threadIdx.x == 0) a.lam[mat] = lam;
    }
  }
  grid.sync();

  // ---- phase 1: setup M_0, T_0, X_0 and err_0 (one warp per padded row)
  {
    const int lane = threadIdx.x & 31, gw = blockIdx.x * (kRT / 32) + (threadIdx.x >> 5);
    const int nw = gridDim.x * (kRT / 32);
    const int64_t rows = (int64_t)a.batch * np;
    for (int64_t rid = gw; rid < rows; rid += nw) {
      const int mat = (int)(rid / np), i = (int)(rid - (int64_t)mat * np);
      const double lam = a.lam[mat];
      if (!lam_ok(lam)) continue;  // warp-uniform
      const double c = lam * (1.0 + a.eps_rel);
      const double xd = c_pow_neg_inv_p(c, a.p), inv_p = 1.0 / (double)a.p;
      const float* arow = a.A + (int64_t)mat * a.stride_a + (int64_t)i * a.lda;
      double* mrow = buf(a, mat, BM0) + (int64_t)i * np;
      double* trow = buf(a, mat, BT) + (int64_t)i * np;
      double* xrow = buf(a, mat, BX0) + (int64_t)i * np;
      double e = 0.0;
      for (int j = lane; j < np; j += 32) {
        double m = 0.0, t = 0.0, x = 0.0;
        if (i < a.n && j < a.n) {
          double av = (double)arow[j];
          if (i == j) av = __dadd_rn(av, __dmul_rn(a.eps_rel, lam));  // (eps*lam) rounded, then added
          m = av / c;
          const double d = (i == j) ? 1.0 : 0.0;
          t = ((double)(a.p + 1) * d - m) * inv_p;
          x = (i == j) ? xd : 0.0;
          e = fmax_nan(e, fabs(m - d));
        }
        mrow[j] = m;
        trow[j] = t;
        xrow[j] = x;
      }
      e = warp_max(e);
      if (lane == 0) atomic_max_nonneg(a.errh + (int64_t)mat * (a.max_iter + 1), e);
    }
  }
  grid.sync();

  // ---- iterations
  if constexpr (!kOz) {
  int* act = reinterpret_cast<int*>(smem + kAsyncSmemDoubles);
  int* cnt = act + kMaxBatchPerLaunch;  // 257 ints scratch
  __shared__ int s_nact;
  // initial active list: lam ok and decide(k=0) == continue
  for (int i = threadIdx.x; i < a.batch; i += kRT) act[i] = i;
  __syncthreads();
  s_nact = compact(a, act, a.batch, 0, cnt, /*first=*/true);
  int nact = s_nact;
  AccN acc;
  for (int k = 0; nact > 0; ++k) {
    const int xs = k & 1;  // X_k in BX0 + xs, M_k in BM0 + xs
    const int tb = (a.p == 1) ? ((k & 1) ? BS0 : BT) : BT;
    const int tb_next = (a.p == 1) ? ((k & 1) ? BT : BS0) : BT;
    // P1: X_{k+1} = X_k T ; S0 = T T (p >= 2)
    {
      const int jobs = (a.p >= 2) ? 2 : 1;
      const int items = nact * tiles * jobs;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int pos = it / (tiles * jobs), rem = it - pos * tiles * jobs;
        const int t = rem / jobs, job = rem - t * jobs;
        const int mat = act[pos];
        int ti, tj;
        upper_tile(t, T, ti, tj);
        const double* Aop = (job == 0) ? buf(a, mat, BX0 + xs) : buf(a, mat, tb);
        const double* Bop = buf(a, mat, tb);
        gemm_tile_f64(acc, Aop + (int64_t)ti * kNT * np, Bop + (int64_t)tj * kNT * np, np, np / kAsyncK, smem);
        double* dst = (job == 0) ? buf(a, mat, BX0 + (xs ^ 1)) : buf(a, mat, BS0);
        epilogue<EPI_STORE>(a, acc, mat, ti, tj, dst, nullptr, nullptr);
      }
      grid.sync();
    }
    // rest of the left-to-right binary chain for T^p (S0 = T^2 from P1):
    // per remaining bit, square (except the first, fused above) and, if the
    // bit is set, multiply by T; ping-pong S0 / S1
    int rbuf = BS0;
    if (a.p >= 2) {
      const int nb = lead_bit(a.p);
      for (int bit = nb - 1; bit >= 0; --bit) {
        if (bit != nb - 1) {
          const int d = (rbuf == BS0) ? BS1 : BS0;
          product_stage(a, act, nact, rbuf, rbuf, d, smem, acc);
          rbuf = d;
          grid.sync();
        }
        if ((a.p >> bit) & 1) {
          const int d = (rbuf == BS0) ? BS1 : BS0;
          product_stage(a, act, nact, rbuf, BT, d, smem, acc);
          rbuf = d;
          grid.sync();
        }
      }
    }
    // P3: M_{k+1} = T^p M_k ; T_{k+1} ; err_{k+1}
    {
      const int tp = (a.p == 1) ? tb : rbuf;
      const int items = nact * tiles;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int pos = it / tiles, t = it - pos * tiles;
        const int mat = act[pos];
        int ti, tj;
        upper_tile(t, T, ti, tj);
        gemm_tile_f64(acc, buf(a, mat, tp) + (int64_t)ti * kNT * np,
                      buf(a, mat, BM0 + xs) + (int64_t)tj * kNT * np, np, np / kAsyncK, smem);
        epilogue<EPI_MUPDATE>(a, acc, mat, ti, tj, buf(a, mat, BM0 + (xs ^ 1)), buf(a, mat, tb_next),
                              a.errh + (int64_t)mat * (a.max_iter + 1) + (k + 1));
      }
      grid.sync();
    }
    // next active list (ordered compaction; identical in every CTA)
    nact = compact(a, act, nact, k + 1, cnt, false);
  }
  }  // !kOz

  // ---- finalize: per-matrix decision, then fp32 output
  for (int mat = blockIdx.x; mat < a.batch; mat += gridDim.x) {
    if (threadIdx.x == 0) {
      const double lam = a.lam[mat];
      int status, iters = 0, rbuf = -1;
      double err = __longlong_as_double(0x7ff8000000000000LL);
      if (!isfinite(lam)) {
        status = 2;
      } else if (!(lam > 0.0)) {
        status = 3;
      } else {
        int k = 0;
        for (;; ++k) {
          int d = decide(a, mat, k);
          if (d == D_CONTINUE) {
            if (k < a.k_sw) continue;
            status = -1;  // handed off to the 3xTF32 tail at check k_sw (root_tail.cu)
            iters = k;
            rbuf = -3;
            err = a.errh[(int64_t)mat * (a.max_iter + 1) + k];
            break;
          }
          const double* e = a.errh + (int64_t)mat * (a.max_iter + 1);
          if (d == D_CONVERGED) { status = 0; iters = k; rbuf = BX0 + (k & 1); err = e[k]; }
          else if (d == D_STAGNATED) { status = 1; iters = k - 1; rbuf = BX0 + ((k - 1) & 1); err = e[k - 1]; }
          else if (d == D_MAXITER) { status = 1; iters = k; rbuf = BX0 + (k & 1); err = e[k]; }
          else { status = 2; iters = k; rbuf = -1; err = e[k]; }
          break;
        }
      }
      a.res[mat] = make_int4(rbuf, iters, status, 0);
      shampoo_root_info_t inf;
      inf.iters = iters;
      inf.status = status;
      inf.lambda_max = lam;
      inf.err = err;
      a.info[mat] = inf;
    }
  }
  grid.sync();
  if (a.k_sw <= a.max_iter) tail_handoff(a);
  if (a.r == 1) write_output(a, -1);
  // r >= 2: root_power_kernel raises the returned iterates to the power r and
  // writes the output (a separate launch: keeping its product code out of this
  // kernel keeps the Newton loops' instruction footprint, measured 12% faster)
}

// Hybrid handoff (rows of every matrix handed off at check k_sw): X_k, M_k and
// T_k -> fp32 (hi, lo = hi - trunc_tf32(hi)) pairs in dead regions, the layout
// root_tail.cu iterates on (tail_region()).  Block 0 also writes the tail's
// initial active list.
SHP_DEV void tail_handoff(const RootArgs& a) {
  const int np = a.np, xs = a.k_sw & 1;
  const int tsrc = (a.p == 1 && (a.k_sw & 1)) ? BS0 : BT;
  const int lane = threadIdx.x & 31, gw = blockIdx.x * (kRT / 32) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (kRT / 32);
  const int64_t rows = (int64_t)a.batch * a.n;
  const int64_t half = (int64_t)np * np;  // floats per hi (or lo) half of a region
  for (int64_t rid = gw; rid < rows && !a.handoff_fp64; rid += nw) {
    const int mat = (int)(rid / a.n), i = (int)(rid - (int64_t)mat * a.n);
    if (a.res[mat].x != -3) continue;  // warp-uniform
    const int src[3] = {BX0 + xs, BM0 + xs, tsrc};
    const int dst[3] = {BX0 + (xs ^ 1), BM0 + (xs ^ 1), BS1};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double* s = buf(a, mat, src[q]) + (int64_t)i * np;
      float* h = reinterpret_cast<float*>(buf(a, mat, dst[q])) + (int64_t)i * np;
      for (int j = lane; j < a.n; j += 32) {
        const float v = __double2float_rn(s[j]);
        h[j] = v;
        h[half + j] = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int c = 0;
    for (int mat = 0; mat < a.batch; ++mat)
      if (a.res[mat].x == -3) a.tail_act[c++] = mat;
    *a.tail_nact = c;
  }
}

// Final fp32 write: X_i (or its power in buffer `pbuf`), I for degenerate
// matrices, nothing for non-finite ones.
SHP_DEV void write_output(const RootArgs& a, int pbuf) {
  const int np = a.np;
  const int lane = threadIdx.x & 31, gw = blockIdx.x * (kRT / 32) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (kRT / 32);
  const int64_t rows = (int64_t)a.batch * a.n;
  for (int64_t rid = gw; rid < rows; rid += nw) {
    const int mat = (int)(rid / a.n), i = (int)(rid - (int64_t)mat * a.n);
    const int4 r = a.res[mat];
    float* out = a.X + (int64_t)mat * a.stride_x + (int64_t)i * a.ldx;
    if (r.z == 3) {
      for (int j = lane; j < a.n; j += 32) out[j] = (i == j) ? 1.0f : 0.0f;
    } else if (r.x >= 0) {
      const double* src = buf(a, mat, pbuf >= 0 ? pbuf : r.x) + (int64_t)i * np;
      for (int j = lane; j < a.n; j += 32) out[j] = (float)src[j];
    }
  }
}

// ---- rational exponent (f4): X <- X^r for every returned iterate, by the
// left-to-right binary chain over the freed M0 / M1 buffers, then the output.
__global__ void __launch_bounds__(kRT, 2) root_power_kernel(RootArgs a) {
  extern __shared__ __align__(16) double smem[];
  cg::grid_group grid = cg::this_grid();
  int* act = reinterpret_cast<int*>(smem + kAsyncSmemDoubles);
  __shared__ int s_n;
  if (threadIdx.x == 0) {
    int c = 0;
    for (int mat = 0; mat < a.batch; ++mat)
      if (a.res[mat].x >= 0) act[c++] = mat;
    s_n = c;
  }
  __syncthreads();
  const int npow = s_n;
  AccN acc;
  int pbuf = -1;
  const int nb = lead_bit(a.r);
  for (int bit = nb - 1; bit >= 0; --bit) {
    const int d0 = (pbuf == BM0) ? BM1 : BM0;
    product_stage(a, act, npow, pbuf, pbuf, d0, smem, acc);  // square (pbuf -1 = X)
    pbuf = d0;
    grid.sync();
    if ((a.r >> bit) & 1) {
      const int d1 = (pbuf == BM0) ? BM1 : BM0;
      product_stage(a, act, npow, pbuf, -1, d1, smem, acc);  // times X
      pbuf = d1;
      grid.sync();
    }
  }
  write_output(a, pbuf);
}

// ---------------------------------------------------------------- host side
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int padded(int n) { return (n + kNT - 1) / kNT * kNT; }

size_t root_workspace_bytes(int batch, int n, int max_iter, int precision) {
  const size_t np = (size_t)padded(n);
  const int chunk = batch < kMaxBatchPerLaunch ? batch : kMaxBatchPerLaunch;
  return align256((size_t)batch * kBufs * np * np * sizeof(double)) + align256((size_t)batch * sizeof(double)) +
         align256((size_t)batch * (max_iter + 1) * sizeof(double)) + align256((size_t)batch * sizeof(int4)) +
         align256((size_t)2 * batch * n * sizeof(double)) + root_tail_ws_bytes(chunk) +
         (precision == 2 ? align256(root_ozaki_ws_bytes(chunk, n)) : 0);
}

size_t root_smem_bytes(int n) {
  size_t gemm = (size_t)kAsyncSmemDoubles * sizeof(double) + (kMaxBatchPerLaunch + kRT + 1) * sizeof(int);
  size_t pi = (2 * (size_t)n + 8) * sizeof(double);
  return gemm > pi ? gemm : pi;
}

int root_launch(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx, int64_t stride_x, int batch,
                int n, int p, int r, int k_sw, int precision, int slices, double slice_budget, double eps_rel,
                double tol, int max_iter, int power_iters, shampoo_root_info_t* info, void* ws, cudaStream_t stream,
                int64_t* launches) {
  const bool oz = (precision == 2);
  const size_t smem = oz ? (2 * (size_t)n + 8) * sizeof(double) : root_smem_bytes(n);
  if (oz) {
    if (ensure_smem((const void*)root_kernel<true>, smem) != cudaSuccess)
      return set_cuda_error("cudaFuncSetAttribute(root_kernel<ozaki>)");
  } else if (ensure_smem((const void*)root_kernel<false>, smem) != cudaSuccess ||
             ensure_smem((const void*)root_power_kernel, smem) != cudaSuccess) {
    return set_cuda_error("cudaFuncSetAttribute(root_kernel)");
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, oz ? root_kernel<true> : root_kernel<false>, kRT, smem) !=
          cudaSuccess ||
      per_sm < 1)
    return set_error(SHAMPOO_ERR_UNSUPPORTED, "root_kernel cannot be resident (smem %zu)", smem);
  const int np = padded(n);
  char* w = static_cast<char*>(ws);
  for (int b0 = 0; b0 < batch; b0 += kMaxBatchPerLaunch) {
    const int bc = (batch - b0 < kMaxBatchPerLaunch) ? batch - b0 : kMaxBatchPerLaunch;
    RootArgs a;
    a.A = A + (int64_t)b0 * stride_a;
    a.lda = lda;
    a.stride_a = stride_a;
    a.X = X + (int64_t)b0 * stride_x;
    a.ldx = ldx;
    a.stride_x = stride_x;
    a.batch = bc;
    a.n = n;
    a.np = np;
    a.p = p;
    a.r = r;
    a.max_iter = max_iter;
    a.k_sw = precision == 2 ? 0 : k_sw;
    a.handoff_fp64 = precision == 2 ? 1 : 0;
    a.power_iters = power_iters;
    a.eps_rel = eps_rel;
    a.tol = tol;
    a.info = info + b0;
    char* q = w;
    a.bufs = reinterpret_cast<double*>(q);
    q += align256((size_t)bc * kBufs * np * np * sizeof(double));
    a.lam = reinterpret_cast<double*>(q);
    q += align256((size_t)bc * sizeof(double));
    a.errh = reinterpret_cast<double*>(q);
    q += align256((size_t)bc * (max_iter + 1) * sizeof(double));
    a.res = reinterpret_cast<int4*>(q);
    q += align256((size_t)bc * sizeof(int4));
    a.wpi = reinterpret_cast<double*>(q);
    q += align256((size_t)2 * bc * n * sizeof(double));
    void* tail_maps = q;
    a.tail_act = reinterpret_cast<int*>(q + align256((size_t)2 * 7 * 128));
    a.tail_nact = a.tail_act + bc;
    q += root_tail_ws_bytes(bc);
    void* oz_ws = q;
    void* args[] = {&a};
    const int grid = num_sms() * per_sm;
    void* tok;
    prof_begin_launch("root_kernel", stream, &tok);
    cudaError_t e = cudaLaunchCooperativeKernel(oz ? (const void*)root_kernel<true> : (const void*)root_kernel<false>,
                                                dim3(grid), dim3(kRT), args, smem, stream);
    prof_end_launch(tok, stream);
    if (e != cudaSuccess) return set_cuda_error("cudaLaunchCooperativeKernel(root_kernel)", e);
    ++*launches;
    if (r >= 2) {
      e = cudaLaunchCooperativeKernel((const void*)root_power_kernel, dim3(grid), dim3(kRT), args, smem, stream);
      if (e != cudaSuccess) return set_cuda_error("cudaLaunchCooperativeKernel(root_power_kernel)", e);
      ++*launches;
    }
    if (precision == 2) {
      int rc = root_ozaki_launch(a.bufs, bc, n, np, p, max_iter, tol, a.errh, a.res, a.info, a.X, ldx, stride_x,
                                 a.tail_act, a.tail_nact, oz_ws, slices, eps_rel, slice_budget, stream, launches);
      if (rc) return rc;
    } else if (k_sw <= max_iter) {
      int rc = root_tail_launch(a.bufs, bc, n, np, p, max_iter, k_sw, tol, a.errh, a.res, a.info, a.X, ldx, stride_x,
                                a.tail_act, a.tail_nact, tail_maps, stream, launches);
      if (rc) return rc;
    }
  }
  return SHAMPOO_OK;
}

// ======================================================= residual check
// residual_i = || X_i^p (A_i + eps*lambda_i I) - I ||_F in fp64 (config 2's
// "residual check"; the north star's invariant).  Cooperative kernel:
// convert -> log2(p) symmetric squarings -> full product with A_hat -> sums.
constexpr int kResBufs = 4;  // Y0 (X), Y1, Y2, Ahat

struct ResArgs {
  const float* A;
  int64_t lda, stride_a;
  const float* X;
  int64_t ldx, stride_x;
  int batch, n, np, p;
  double eps_rel;
  const shampoo_root_info_t* info;
  double* out;
  double* bufs;  // batch * 4 * np^2
  double* part;  // batch * T^2
};

SHP_DEV double* rbuf(const ResArgs& a, int mat, int b) {
  return a.bufs + ((int64_t)mat * kResBufs + b) * (int64_t)a.np * a.np;
}

__global__ void __launch_bounds__(kRT, 2) residual_kernel(ResArgs a) {
  extern __shared__ __align__(16) double smem[];
  cg::grid_group grid = cg::this_grid();
  const int np = a.np, n = a.n, T = np / kNT, tiles = T * (T + 1) / 2;
  const int64_t np2 = (int64_t)np * np, total = (int64_t)a.batch * np2;
  for (int64_t idx = (int64_t)blockIdx.x * kRT + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * kRT) {
    const int mat = (int)(idx / np2);
    const int64_t rem = idx - (int64_t)mat * np2;
    const int i = (int)(rem / np), j = (int)(rem - (int64_t)i * np);
    const bool valid = i < n && j < n;
    double x = 0.0, ah = 0.0;
    if (valid) {
      const int r = i < j ? i : j, q = i < j ? j : i;  // upper triangles (symmetric by contract)
      x = (double)a.X[(int64_t)mat * a.stride_x + (int64_t)r * a.ldx + q];
      ah = (double)a.A[(int64_t)mat * a.stride_a + (int64_t)r * a.lda + q];
      if (i == j) ah = __dadd_rn(ah, __dmul_rn(a.eps_rel, a.info[mat].lambda_max));
    }
    rbuf(a, mat, 0)[rem] = x;
    rbuf(a, mat, 3)[rem] = ah;
  }
  grid.sync();
  // X^p by the left-to-right binary chain: per bit after the leading one,
  // square, then multiply by X (Y0) if the bit is set; ping-pong Y1 / Y2
  int src = 0;
  AccN acc;
  const int nsteps = 2 * (31 - __clz(a.p));
  for (int step = 0; step < nsteps; ++step) {
    const int bit = (31 - __clz(a.p)) - 1 - step / 2;
    const bool square = (step & 1) == 0;
    if (!square && !((a.p >> bit) & 1)) continue;  // uniform across the grid
    const int dst = (src == 1) ? 2 : 1;
    for (int it = blockIdx.x; it < a.batch * tiles; it += gridDim.x) {
      const int mat = it / tiles, t = it - mat * tiles;
      int ti, tj;
      upper_tile(t, T, ti, tj);
      const double* S = rbuf(a, mat, src);
      const double* S2 = square ? S : rbuf(a, mat, 0);
      gemm_tile_f64(acc, S + (int64_t)ti * kNT * np, S2 + (int64_t)tj * kNT * np, np, np / kAsyncK, smem);
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      double* D = rbuf(a, mat, dst);
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int i = ti * kNT + accn_row(warp, lane, mt);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int j = tj * kNT + accn_col(warp, lane, nt, 0);
          *reinterpret_cast<double2*>(D + (int64_t)i * np + j) = make_double2(acc.c[mt][nt][0], acc.c[mt][nt][1]);
          if (ti != tj) {
            D[(int64_t)j * np + i] = acc.c[mt][nt][0];
            D[(int64_t)(j + 1) * np + i] = acc.c[mt][nt][1];
          }
        }
      }
    }
    grid.sync();
    src = dst;
  }
  __shared__ double red[kRT / 32];
  for (int it = blockIdx.x; it < a.batch * T * T; it += gridDim.x) {
    const int mat = it / (T * T), t = it - mat * T * T;
    const int ti = t / T, tj = t - ti * T;
    gemm_tile_f64(acc, rbuf(a, mat, src) + (int64_t)ti * kNT * np, rbuf(a, mat, 3) + (int64_t)tj * kNT * np,
                  np, np / kAsyncK, smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double s = 0.0;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int i = ti * kNT + accn_row(warp, lane, mt);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = tj * kNT + accn_col(warp, lane, nt, e);
          if (i < n && j < n) {
            const double d = acc.c[mt][nt][e] - ((i == j) ? 1.0 : 0.0);
            s = fma(d, d, s);
          }
        }
    }
    s = warp_sum_fixed(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t2 = 0.0;
      for (int w = 0; w < kRT / 32; ++w) t2 = __dadd_rn(t2, red[w]);
      a.part[(int64_t)mat * T * T + t] = t2;
    }
    __syncthreads();
  }
  grid.sync();
  for (int mat = blockIdx.x * kRT + threadIdx.x; mat < a.batch; mat += gridDim.x * kRT) {
    double s = 0.0;
    for (int t = 0; t < T * T; ++t) s = __dadd_rn(s, a.part[(int64_t)mat * T * T + t]);
    a.out[mat] = sqrt(s);
  }
}

size_t residual_workspace_bytes(int batch, int n) {
  const size_t np = (size_t)padded(n), T = np / kNT;
  return align256((size_t)batch * kResBufs * np * np * sizeof(double)) + align256((size_t)batch * T * T * sizeof(double));
}

int residual_launch(const float* A, int64_t lda, int64_t stride_a, const float* X, int64_t ldx, int64_t stride_x,
                    int batch, int n, int p, double eps_rel, const shampoo_root_info_t* info, double* residual,
                    void* ws, cudaStream_t stream, int64_t* launches) {
  const size_t smem = (size_t)kAsyncSmemDoubles * sizeof(double);
  if (ensure_smem((const void*)residual_kernel, smem) != cudaSuccess)
    return set_cuda_error("cudaFuncSetAttribute(residual_kernel)");
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, residual_kernel, kRT, smem) != cudaSuccess || per_sm < 1)
    return set_error(SHAMPOO_ERR_UNSUPPORTED, "residual_kernel cannot be resident");
  ResArgs a;
  a.A = A;
  a.lda = lda;
  a.stride_a = stride_a;
  a.X = X;
  a.ldx = ldx;
  a.stride_x = stride_x;
  a.batch = batch;
  a.n = n;
  a.np = padded(n);
  a.p = p;
  a.eps_rel = eps_rel;
  a.info = info;
  a.out = residual;
  const size_t np = (size_t)a.np;
  char* q = static_cast<char*>(ws);
  a.bufs = reinterpret_cast<double*>(q);
  q += align256((size_t)batch * kResBufs * np * np * sizeof(double));
  a.part = reinterpret_cast<double*>(q);
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)residual_kernel, dim3(num_sms() * per_sm), dim3(kRT),
                                              args, smem, stream);
  if (e != cudaSuccess) return set_cuda_error("cudaLaunchCooperativeKernel(residual_kernel)", e);
  ++*launches;
  return SHAMPOO_OK;
}

}  // namespace shp
