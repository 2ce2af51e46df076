/* Oracle: Shampoo statistics, diagonal accumulator and graft numerator (row a2).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain C, fp64, no BLAS,
 * compiled with -O2 -ffp-contract=off.  Shares nothing with the CUDA path.
 *
 * Follows Alg. 1 of the paper:
 *     L_t <- beta2 L_{t-1} + (1-beta2) G G^T   (beta2 < 1)   else L_{t-1} + G G^T
 *     R_t <- beta2 R_{t-1} + (1-beta2) G^T G
 *     D_t <- D_{t-1} + G o G                    (always a sum)
 * written as (decay, weight) = (beta2, 1-beta2) or (1, 1), reading #6.
 *
 * Arithmetic contract (reading #15; bit-exact target for the GPU):
 *   acc = 0.0; for k ascending: acc = acc + (double)a_k * (double)b_k
 *     (each product of two floats is exact in double, so fused and unfused
 *      multiply-add give the same bits)
 *   t1 = weight*acc; t2 = decay*(double)S_ij; S_ij = S_ji = (float)(t1 + t2)
 *   D_ij = (float)((double)D_ij + (double)g_ij*(double)g_ij)
 * Graft numerator of a block (floor 1e-30 of S:437 = reading #11):
 *   num_b = sum_ij g_ij^2 / max((double)D_new_ij, 1e-30)  (row-major order)
 */
#include <math.h>
#include <stdint.h>

/* 1 if every G entry of the block is finite, else 0 ("non-finite gradient
 * entries -> rejected, state unchanged"). */
int oracle_block_finite(const float* G, int64_t ldg, int64_t row0, int64_t col0, int rows, int cols) {
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j)
      if (!isfinite(G[(row0 + i) * ldg + col0 + j])) return 0;
  return 1;
}

/* L_b (rows x rows, leading dim ldl) <- decay*L_b + weight * G_b G_b^T. */
void oracle_stats_left(const float* G, int64_t ldg, int64_t row0, int64_t col0, int rows, int cols,
                       float* L, int64_t ldl, double decay, double weight) {
  for (int i = 0; i < rows; ++i) {
    const float* gi = G + (row0 + i) * ldg + col0;
    for (int j = i; j < rows; ++j) {
      const float* gj = G + (row0 + j) * ldg + col0;
      double acc = 0.0;
      for (int k = 0; k < cols; ++k) acc = acc + (double)gi[k] * (double)gj[k];
      double t1 = weight * acc;
      double t2 = decay * (double)L[(int64_t)i * ldl + j];
      float r = (float)(t1 + t2);
      L[(int64_t)i * ldl + j] = r;
      L[(int64_t)j * ldl + i] = r;
    }
  }
}

/* R_b (cols x cols, leading dim ldr) <- decay*R_b + weight * G_b^T G_b. */
void oracle_stats_right(const float* G, int64_t ldg, int64_t row0, int64_t col0, int rows, int cols,
                        float* R, int64_t ldr, double decay, double weight) {
  for (int i = 0; i < cols; ++i) {
    for (int j = i; j < cols; ++j) {
      double acc = 0.0;
      for (int k = 0; k < rows; ++k) {
        const float* gk = G + (row0 + k) * ldg + col0;
        acc = acc + (double)gk[i] * (double)gk[j];
      }
      double t1 = weight * acc;
      double t2 = decay * (double)R[(int64_t)i * ldr + j];
      float r = (float)(t1 + t2);
      R[(int64_t)i * ldr + j] = r;
      R[(int64_t)j * ldr + i] = r;
    }
  }
}

/* D_b <- D_b + G_b o G_b; returns the block's graft numerator. */
double oracle_diag_update(const float* G, int64_t ldg, int64_t row0, int64_t col0, int rows, int cols,
                          float* D, int64_t ldd) {
  double num = 0.0;
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) {
      double g = (double)G[(row0 + i) * ldg + col0 + j];
      float* d = D + (row0 + i) * ldd + col0 + j;
      float dn = (float)((double)*d + g * g);
      *d = dn;
      double den = (double)dn > 1e-30 ? (double)dn : 1e-30;
      num = num + (g * g) / den;
    }
  return num;
}

/* ---------------------------------------------------------------- f3: tensors
 * Mode statistic of one block of an order-k tensor (the paper's method "holds
 * for tensors of arbitrary order"; per-mode statistics of
 * the mode-i unfolding, DESIGN.md §6.5 / reading #24):
 *   U  : rows x K row-major fp32, the mode-i unfolding of the block (row a =
 *        index a of mode i; columns = the remaining block indices in row-major
 *        order)
 *   S  : rows x rows (leading dim lds) <- decay*S + weight * U U^T
 * Chunked sequential contract (reading #25): for chunk c = [c*C, min(K, (c+1)*C)),
 *   s_c = 0.0; for k ascending in the chunk: s_c = s_c + (double)u_a[k]*(double)u_b[k]
 *   acc = 0.0; for c ascending: acc = acc + s_c
 *   t1 = weight*acc; t2 = decay*(double)S_ab; S_ab = S_ba = (float)(t1 + t2)
 * For K <= C this is exactly the matrix contract above. */
void oracle_mode_stat(const float* U, int rows, int64_t K, int64_t chunk, float* S, int64_t lds, double decay,
                      double weight) {
  for (int a = 0; a < rows; ++a) {
    const float* ua = U + (int64_t)a * K;
    for (int b = a; b < rows; ++b) {
      const float* ub = U + (int64_t)b * K;
      double acc = 0.0;
      for (int64_t c0 = 0; c0 < K; c0 += chunk) {
        const int64_t c1 = c0 + chunk < K ? c0 + chunk : K;
        double s = 0.0;
        for (int64_t k = c0; k < c1; ++k) s = s + (double)ua[k] * (double)ub[k];
        acc = acc + s;
      }
      double t1 = weight * acc;
      double t2 = decay * (double)S[(int64_t)a * lds + b];
      float r = (float)(t1 + t2);
      S[(int64_t)a * lds + b] = r;
      S[(int64_t)b * lds + a] = r;
    }
  }
}
