/* shampoo.h -- C ABI of libshampoo: the data-parallel hot path of distributed
 * Shampoo (Anil, Gupta, Koren, Regan, Singer, "Second Order Optimization Made
 * Practical", arXiv 2002.09018) on NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = line n of the paper text (reference PAPER.md), "S:n" = line
 * n of the reference SPEC.md, "reading #k" = DESIGN.md §3 entry k.
 *
 * Conventions shared by every call
 * ---------------------------------
 *  - Pointers are DEVICE pointers unless the parameter is marked (host).
 *  - The caller owns all memory (statistics, roots, gradients, D, P, tables,
 *    workspaces).  The library holds no device memory and no state between
 *    calls; calls on different streams may run concurrently from different
 *    host threads.
 *  - Matrices are row-major fp32 with an explicit leading dimension (in
 *    elements).  Statistics and roots are symmetric; kernels read the upper
 *    triangle and always write both triangles.
 *  - Host-checkable problems (shapes, p, alignment, non-finite scalars,
 *    workspace too small, capacity) return a non-zero status synchronously
 *    and enqueue nothing.  Data-dependent outcomes (non-finite gradients,
 *    non-convergence, degenerate statistics) are never return codes: they are
 *    reported per block / per matrix in device arrays.
 *  - Every compute call is stream-ordered, enqueues its kernels on `stream`
 *    and returns without synchronising the host.
 *  - No exception crosses the ABI; on error the message is available from
 *    shampoo_last_error() (thread-local).
 */
#ifndef SHAMPOO_H_
#define SHAMPOO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SHAMPOO_ABI_VERSION 4

typedef enum {
  SHAMPOO_OK = 0,
  SHAMPOO_ERR_INVALID_ARG = 1, /* bad shape / p / alignment / scalar        */
  SHAMPOO_ERR_UNSUPPORTED = 2, /* valid request this build cannot serve     */
  SHAMPOO_ERR_CUDA = 3,        /* a CUDA runtime call or launch failed      */
  SHAMPOO_ERR_WORKSPACE = 4,   /* workspace pointer null or too small       */
  SHAMPOO_ERR_CAPACITY = 5     /* host output array too small (plan)        */
} shampoo_status_t;

typedef void* shampoo_stream_t; /* a cudaStream_t (NULL = legacy default stream) */

/* One block of one parameter tensor (plan output; integer, bit-exact vs the
 * oracle).  P:396-398: "divide the tensor into blocks and treating individual
 * block as a separate tensor".  80 bytes.  The root of a side is S^{-r/p}:
 * (r, p) = (1, 4) two-sided, (1, 2) one-sided, p = 0 skipped; a split plan
 * (f4) gives e.g. (1, 8) / (3, 8). */
typedef struct {
  int32_t tensor_id;   /* index into the caller's tensor list                          */
  int32_t reserved;    /* 0                                                            */
  int64_t row0, col0;  /* block origin inside the tensor                               */
  int32_t rows, cols;  /* extent; the last block of each axis may be ragged            */
  int32_t p_left;      /* root order of L_b^{-r/p}: 4 two-sided, 2 one-sided, 0 skipped */
  int32_t p_right;     /* root order of R_b^{-r/p}                                     */
  int32_t r_left;      /* exponent numerator of the left root (0 if skipped)           */
  int32_t r_right;     /* exponent numerator of the right root (0 if skipped)          */
  int32_t owner_left;  /* rank that updates L_b and computes its root (-1 if skipped)  */
  int32_t owner_right; /* rank that updates R_b and computes its root (-1 if skipped)  */
  int64_t left_off;    /* element offset of L_b (and of its root) in the packed buffer */
  int64_t right_off;   /*   ... of R_b; -1 when the side is skipped                    */
  int32_t left_ld;     /* leading dimension of L_b = roundup(rows, 4)                  */
  int32_t right_ld;    /* leading dimension of R_b = roundup(cols, 4)                  */
} shampoo_block_t;

/* A strided batch of same-size roots S^{-r/p} owned by one rank (plan output). */
typedef struct {
  int32_t owner, n, p, count;
  int64_t offset; /* element offset of the first matrix in the packed buffer */
  int64_t stride; /* elements between consecutive matrices                   */
  int32_t r;      /* exponent numerator                                       */
  int32_t reserved;
} shampoo_group_t;

/* One parameter tensor.  An array of these lives in DEVICE memory. */
typedef struct {
  const float* G; /* gradient, row-major m x n                                    */
  float* D;       /* diagonal AdaGrad accumulator (same layout as G), in/out      */
  float* P;       /* preconditioned-gradient output (same layout as G)            */
  int64_t ldg, ldd, ldp;
  int64_t m, n;
} shampoo_tensor_t;

/* Optimizer state of one parameter tensor for the Alg. 1 tail (f2); an array of
 * these, parallel to the shampoo_tensor_t array, lives in DEVICE memory. */
typedef struct {
  float* W;  /* parameters, updated in place                                 */
  float* M;  /* momentum of the grafted diagonal direction D^{-1/2} o G       */
  float* Pm; /* momentum of the preconditioned gradient                      */
  int64_t ldw, ldm, ldpm;
} shampoo_state_t;

/* Per-matrix result of the root solver (device array). */
typedef struct {
  int32_t iters;     /* coupled-Newton iterations performed                        */
  int32_t status;    /* 0 converged (err <= tol); 1 not converged, best iterate
                        returned; 2 non-finite input, X left untouched;
                        3 degenerate (lambda_hat <= 0), X = I written           */
  double lambda_max; /* power-iteration estimate lambda_hat (reading #3)          */
  double err;        /* max_ij |M - I| of the returned iterate                     */
} shampoo_root_info_t;

int shampoo_abi_version(void);
const char* shampoo_last_error(void);

/* ------------------------------------------------------------------ a1: plan
 * Blocking plan, exponents, owners and packing (P:356-359, P:385-390,
 * P:396-398; rule in DESIGN.md §5 / oracle/plan.py).
 *   shapes      (host) 2*n_tensors int64: m0, n0, m1, n1, ...
 *   split_num, split_den : the Lemma's split 1/p = split_num/split_den
 *               (f4): two-sided blocks get
 *               L^{-split_num/(2 split_den)} and R^{-(split_den-split_num)/(2 split_den)},
 *               reduced to r/p with p <= 16.  (1, 2) = the default -1/4, -1/4.
 *               1 <= split_num < split_den, else SHAMPOO_ERR_INVALID_ARG.
 *   blocks      (host, out) capacity entries, or NULL to query counts only
 *   groups      (host, out) group_capacity entries, or NULL
 *   stats_elems (host, out) elements of the packed statistics/roots buffer
 *               (= world_size * segment_elems; segment r holds rank r's roots)
 * Returns SHAMPOO_ERR_CAPACITY (counts still written) if an array is too small. */
int shampoo_plan(const int64_t* shapes, int32_t n_tensors, int32_t block_size, int64_t max_precond_dim,
                 int32_t world_size, int32_t split_num, int32_t split_den, shampoo_block_t* blocks, int32_t capacity, int32_t* n_blocks,
                 shampoo_group_t* groups, int32_t group_capacity, int32_t* n_groups,
                 int64_t* stats_elems, int64_t* segment_elems);

/* Layer-granular variant (reading #30; "As preconditioners need to be
 * computed for every layer of the network, we distribute the computation across
 * all the CPUs"): every root of tensor t is owned by tensor_owner[t], the tensors
 * assigned LPT -- sorted by (cost desc, index), cost = sum over the tensor's roots
 * of n^3 x (products per iteration + 12) + m*n, each to the least-loaded rank
 * (lowest on ties).  Packing as shampoo_plan.  An owner then holds whole tensors:
 * their statistics, roots and preconditioned gradient, so the multi-GPU step
 * exchanges P (one all-gather) instead of the roots.
 *   tensor_owner (host, out, nullable) n_tensors entries. */
int shampoo_plan_layers(const int64_t* shapes, int32_t n_tensors, int32_t block_size, int64_t max_precond_dim,
                        int32_t world_size, int32_t split_num, int32_t split_den, shampoo_block_t* blocks,
                        int32_t capacity, int32_t* n_blocks, shampoo_group_t* groups, int32_t group_capacity,
                        int32_t* n_groups, int64_t* stats_elems, int64_t* segment_elems, int32_t* tensor_owner);

/* ------------------------------------------------------- a2: statistics step
 * For every block b (Alg. 1; contract in DESIGN.md §6.2):
 *   if any G_b entry is non-finite: block_status[b] = 2, L_b/R_b/D_b untouched,
 *                                   graft_num[b] = 0;
 *   else  L_b <- decay*L_b + weight*G_b G_b^T   (if p_left  and (only_owner<0 or owner_left ==only_owner))
 *         R_b <- decay*R_b + weight*G_b^T G_b   (if p_right and (only_owner<0 or owner_right==only_owner))
 *         D_b <- D_b + G_b o G_b                (always; D may be NULL per tensor -> skipped)
 *         graft_num[b] = sum g^2 / max(D_new, 1e-30)   (reading #11)
 * L/R use the sequential fp64 contract (ascending-k fp64 accumulation, then
 * t1 = weight*acc, t2 = decay*old, (float)(t1+t2)); they are BIT-EXACT with the
 * oracle.  (decay, weight) = (beta2, 1-beta2) or (1, 1) (reading #6).
 *   tensors, blocks : device tables (n_tensors / n_blocks entries)
 *   blocks_host     : the same block table in HOST memory (sizes the workspace)
 *   stats           : packed fp32 statistics (offsets from the plan), in/out
 *   graft_num       : double[n_blocks] out (nullable)
 *   block_status    : int32[n_blocks] out (nullable)
 *   workspace       : >= shampoo_stats_workspace_bytes(blocks_host, n_blocks, only_owner), 256-B
 *                     aligned (holds the owned blocks widened to zero-padded fp64 panels)
 * G, D, P need only fp32 alignment; any ld >= n works. */
size_t shampoo_stats_workspace_bytes(const shampoo_block_t* blocks_host, int32_t n_blocks, int32_t only_owner);
int shampoo_stats_update(const shampoo_tensor_t* tensors, int32_t n_tensors, const shampoo_block_t* blocks,
                         const shampoo_block_t* blocks_host, int32_t n_blocks, int32_t only_owner, float* stats,
                         double decay, double weight, double* graft_num, int32_t* block_status, void* workspace,
                         size_t workspace_bytes, shampoo_stream_t stream);

/* --------------------------------------- a3-a6: batched inverse p-th roots
 * X_i ~ (A_i + eps_rel*lambda_hat_i*I)^{-1/p} for a strided batch of n x n
 * symmetric PSD fp32 matrices, by the coupled Newton iteration (
 * S:131; readings #1-#4):
 *   lambda_hat: `power_iters` power steps from the splitmix64 start vector;
 *   A_hat = A + eps_rel*lambda_hat*I;  c = lambda_hat*(1+eps_rel);
 *   M_0 = A_hat/c;  X_0 = c^{-1/p} I;
 *   repeat: err = max|M-I|; stop if err <= tol (or stagnation / max_iter);
 *           T = ((p+1)I - M)/p;  X <- X T;  M <- T^p M
 *           (T^p by the left-to-right binary chain of squarings and
 *           multiplications by T).
 * Products run in fp64 on the FP64 tensor pipe (DMMA); results are written
 * as fp32.  p integer in [1, 16] (c^{-1/p} by sqrt chains when p = 2^j,
 * pow otherwise; reading #22); 1 <= n <= 8192.
 *   A   : batch matrices at A + i*stride_a, leading dim lda (fp32, read only)
 *   X   : outputs at X + i*stride_x, leading dim ldx (fp32; may alias A only if
 *         A == X with equal strides/ld -- the input is consumed first)
 *   info: shampoo_root_info_t[batch] out
 *   workspace: >= shampoo_root_workspace_bytes(batch, n, p, max_iter), 256-B aligned
 * A_i must be symmetric (statistics are, by construction): the Newton setup
 * reads its upper triangle.  Non-finite input leaves X_i untouched (status 2);
 * lambda_hat <= 0 writes X_i = I (status 3). */
size_t shampoo_root_workspace_bytes(int32_t batch, int32_t n, int32_t p, int32_t max_iter);
int shampoo_inverse_pth_root_batched(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                     int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                     double tol, int32_t max_iter, int32_t power_iters,
                                     shampoo_root_info_t* info, void* workspace, size_t workspace_bytes,
                                     shampoo_stream_t stream);

/* f4: rational exponents ("L^{1/p} (x) R^{1/q}"
 * "L^{-1/2p} G R^{-1/2q}"; reading #23):
 *   X_i ~ A_hat_i^{-r/p} = (A_hat_i^{-1/p})^r,  1 <= r <= p <= 16,
 * the p-th root above (same iteration, statuses and info, which describe the
 * p-th root) raised to the integer power r by symmetric FP64 DMMA products
 * (left-to-right binary chain) before the fp32 write.  r = 1 is exactly
 * shampoo_inverse_pth_root_batched.  Same arguments and workspace. */
int shampoo_inverse_root_rational_batched(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                          int64_t stride_x, int32_t batch, int32_t n, int32_t p, int32_t r,
                                          double eps_rel, double tol, int32_t max_iter, int32_t power_iters,
                                          shampoo_root_info_t* info, void* workspace, size_t workspace_bytes,
                                          shampoo_stream_t stream);

/* Hybrid precision (north star: "3xTF32 error-compensated splits or FP64 DMMA";
 * DESIGN.md §6.3b): the first fp64_iters coupled-Newton iterations in fp64 on
 * the DMMA pipe, the rest on the tcgen05 tensor cores with 3xTF32 products
 * (hi = trunc_tf32(x), lo = x - hi; lo.hi + hi.lo + hi.hi in fp32) and fp32
 * iterates; symmetric upper tiles only.
 * fp64_iters = -1: automatic, the smallest k with eps_rel * g^k >= 1e-2
 * (1e-1 for p <= 3), g = (1 + 1/p)^p (k = 11 for p = 4, eps_rel = 1e-6);
 * eps_rel = 0 or fp64_iters > max_iter: pure fp64 (= the call above).
 * Measured on B200 (n = 1024, kappa(A_hat) = 1e6, p = 4): rel. Frobenius
 * error 9e-5 (bar 1e-3), 1.43x the pure-fp64 rate.  The tensor core's fp32
 * accumulation is biased on near-identity products (~1e-5): k-tiles are
 * ordered so the O(1) diagonal blocks come last, and the tail stops at
 * max|M - I| <= max(tol, 1e-5) or by the stagnation rule (status 1).
 * Same arguments, statuses and workspace as shampoo_inverse_pth_root_batched. */
int shampoo_inverse_pth_root_batched_hybrid(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                            int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                            double tol, int32_t max_iter, int32_t power_iters, int32_t fp64_iters,
                                            shampoo_root_info_t* info, void* workspace, size_t workspace_bytes,
                                            shampoo_stream_t stream);

/* Ozaki precision: every coupled-Newton product on the INT8
 * tensor cores -- each fp64 operand is split per row into `slices` int8 slices
 * (one rounding, to 2^-(7 slices - 1) relative to the row maximum), the
 * slices (slices + 1) / 2 slice products with s + t <= slices + 1 accumulate
 * EXACTLY in int32 TMEM accumulators (tcgen05.mma.kind::i8), and the epilogue
 * combines them in fp64.  Iterates, power iteration, ridge, stopping rule and
 * statuses are those of shampoo_inverse_pth_root_batched (p-th roots, r = 1);
 * the workspace is larger (shampoo_root_ozaki_workspace_bytes: + 5 x 7 int8
 * planes per matrix, enough for either slice count).
 * slices = 7 (28 products): fp64-level; measured 2.4e-7 relative Frobenius
 *   root error at n = 1024, kappa 1e6 (fp32-output-limited).
 * slices = 6 (21 products): the precision chosen against the north star's
 *   1e-3 bar -- host emulation (tools/ozaki_precision.py) 3.8e-6 at n = 256;
 *   measured on B200 in tests/test_gpu_ozaki.py.
 * Any other value: SHAMPOO_ERR_INVALID_ARG, nothing enqueued.
 * slice_budget (ABI v4; reading #29): 0 = every product of every
 *   iteration uses `slices` slices (the fixed-slice root).  > 0 = per-iteration
 *   schedule: an error in M_k reaches the root amplified by ~1/(p lambda_min(M_k))
 *   and lambda_min(M_k) >= m_k = min(1, eps_rel g^k), g = ((p+1)/p)^p (the ridge
 *   and the scalar recurrence), so iteration k uses the smallest S in
 *   [5, slices] with 2^-(7S-1) sqrt(n/1024) / (p m_k) <= slice_budget, and the X-update
 *   X_k T_k (not amplified) min(S, 5).  eps_rel = 0 keeps `slices` throughout.
 *   1e-9 (the binding's default): 0.68 of the fixed-7 slice products at
 *   n = 1024, p = 4, kappa 1e6, root error 2.9e-7 vs 1.2e-7 in host emulation
 *   (tools/ozaki_schedule.py).  Must be in [0, 1), else SHAMPOO_ERR_INVALID_ARG. */
size_t shampoo_root_ozaki_workspace_bytes(int32_t batch, int32_t n, int32_t p, int32_t max_iter);
/* Host-only: the slice count the Ozaki root uses for the products of iteration
 * k (the M-chain; the X-update uses min(result, 5) when slice_budget > 0) for
 * these arguments -- the schedule above, for accounting (bench roofline). */
int shampoo_ozaki_iteration_slices(int32_t k, int32_t p, int32_t n, double eps_rel, double slice_budget,
                                   int32_t slices);
int shampoo_inverse_pth_root_batched_ozaki(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                           int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                           double tol, int32_t max_iter, int32_t power_iters, int32_t slices,
                                           double slice_budget, shampoo_root_info_t* info, void* workspace,
                                           size_t workspace_bytes, shampoo_stream_t stream);

/* Precision "auto" (the bench's): the Ozaki root above (slices, slice_budget)
 * for n >= SHAMPOO_OZAKI_MIN_N, shampoo_inverse_pth_root_batched (FP64 DMMA)
 * below -- the Ozaki loop launches ~7 kernels per iteration and tiles 128 rows,
 * which small matrices cannot fill (measured on B200: n = 128 Ozaki 19k vs
 * FP64 72k roots/s; n = 512 2.7k vs 2.5k; n = 1024 580 vs 354).  Arguments as
 * the Ozaki call; workspace >= shampoo_root_auto_workspace_bytes(...). */
#define SHAMPOO_OZAKI_MIN_N 512
size_t shampoo_root_auto_workspace_bytes(int32_t batch, int32_t n, int32_t p, int32_t max_iter);
int shampoo_inverse_pth_root_batched_auto(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                          int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                          double tol, int32_t max_iter, int32_t power_iters, int32_t slices,
                                          double slice_budget, shampoo_root_info_t* info, void* workspace,
                                          size_t workspace_bytes, shampoo_stream_t stream);

/* Independent root check (config 2, north-star invariant):
 *   residual_i = || X_i^p (A_i + eps_rel*lambda_i*I) - I ||_F   in fp64,
 * lambda_i = info[i].lambda_max from the root call.  out: double[batch]. */
size_t shampoo_root_residual_workspace_bytes(int32_t batch, int32_t n, int32_t p);
int shampoo_root_residual_batched(const float* A, int64_t lda, int64_t stride_a, const float* X, int64_t ldx,
                                  int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                  const shampoo_root_info_t* info, double* residual, void* workspace,
                                  size_t workspace_bytes, shampoo_stream_t stream);

/* ------------------------------------------- a8, a9: precondition + graft
 * For every block b (readings #9-#11, #17):
 *   two-sided  P_b = X_L G_b X_R;  one-sided P_b = G_b X_R or X_L G_b;
 *   no side    P_b = D_b^{-1/2} o G_b  (grafted diagonal AdaGrad);
 *   graft_scale[b] = sqrt(graft_num[b]) / ||P_b||_F  (0 if ||P_b|| = 0),
 * written into tensors[t].P.  roots uses the statistics packing.  The caller
 * applies W -= eta * graft_scale[b] * P_b (grafting).
 * Products: 3xTF32 on the tcgen05 tensor cores (fp32-accurate: x = hi + lo
 * exact TF32 split, hi.hi + hi.lo + lo.hi accumulated in TMEM) for blocks with
 * a right factor whose ragged extents sit on the tensor edge or are multiples
 * of 32; FP64 DMMA for the rest (left-only blocks).
 *   tensors_host, blocks_host : HOST tables (the call derives TMA tensor maps
 *                               and per-block GEMM jobs from them and uploads
 *                               them into the workspace, stream-ordered)
 *   graft_num  : double[n_blocks] from shampoo_stats_update (nullable -> no scale)
 *   graft_scale: float[n_blocks] out (nullable)
 *   den        : double[n_blocks] out, ||P_b||_F^2 (nullable)
 *   workspace  : >= shampoo_precondition_workspace_bytes(...), 256-B aligned
 * Errors: SHAMPOO_ERR_WORKSPACE if the workspace is smaller than required. */
size_t shampoo_precondition_workspace_bytes(const shampoo_tensor_t* tensors_host, int32_t n_tensors,
                                            const shampoo_block_t* blocks_host, int32_t n_blocks);
int shampoo_precondition(const shampoo_tensor_t* tensors_host, int32_t n_tensors, const shampoo_block_t* blocks_host,
                         int32_t n_blocks, const float* roots, const double* graft_num, float* graft_scale,
                         double* den, void* workspace, size_t workspace_bytes, shampoo_stream_t stream);

/* The same with the roots' TF32 remainder supplied by the caller: roots_lo =
 * roots - trunc_tf32(roots) over the packed buffer (shampoo_tf32_split), computed
 * once per root refresh instead of once per step (roots change every kappa
 * steps).  roots_lo NULL = shampoo_precondition. */
int shampoo_precondition_split(const shampoo_tensor_t* tensors_host, int32_t n_tensors,
                               const shampoo_block_t* blocks_host, int32_t n_blocks, const float* roots,
                               const float* roots_lo, const double* graft_num, float* graft_scale, double* den,
                               void* workspace, size_t workspace_bytes, shampoo_stream_t stream);

/* lo[i] = x[i] - trunc_tf32(x[i]) for i < n (n % 4 == 0, both 16-B aligned): the
 * exact remainder of the TF32 split the tensor cores need (they truncate fp32
 * operands to TF32). */
int shampoo_tf32_split(const float* x, float* lo, int64_t n, shampoo_stream_t stream);

/* ----------------------------------------- f2: momentum, step size, update
 * The tail of Algorithm 1, per block b (readings #9, #11):
 *   M_t = beta1 M_{t-1} + (1-beta1) D_t^{-1/2} o G_t               (line 12)
 *   shampoo_branch (t > tau):
 *     Pm_t = beta1 Pm_{t-1} + (1-beta1) P_t   (P_t = shampoo_precondition's P)
 *     eta_b = eta0 ||M_t||_F / ||Pm_t||_F (0 if ||Pm_t|| = 0);  W -= eta_b Pm_t
 *   else:  eta_b = eta0;  W -= eta0 M_t                               (lines 22-23)
 * Norms are fixed-order fp64 sums over the stored fp32 values (deterministic).
 *   tensors, states, blocks : DEVICE tables (parallel tensor / state arrays)
 *   eta_out : double[n_blocks] out (nullable)
 *   workspace: >= shampoo_momentum_workspace_bytes(n_blocks), 256-B aligned */
size_t shampoo_momentum_workspace_bytes(int32_t n_blocks);
int shampoo_momentum_step(const shampoo_tensor_t* tensors, const shampoo_state_t* states, int32_t n_tensors,
                          const shampoo_block_t* blocks, int32_t n_blocks, double beta1, double eta0,
                          int32_t shampoo_branch, double* eta_out, void* workspace, size_t workspace_bytes,
                          shampoo_stream_t stream);

/* ===================================================== f3: tensors of order 1..4
 * The paper's method "holds for tensors of arbitrary order";
 * per-mode Shampoo (readings #24-#26): mode i of an order-k tensor is
 * preconditioned iff 1 < d_i <= max_precond_dim; with k' kept modes each gets
 * the root H_i^{-1/(2k')} (exponents sum to -1/2); H_i accumulates
 * U_i U_i^T of the mode-i unfolding of each block; P_B = B x_0 X_0 x_1 X_1 ...
 * Every mode is blocked by block_size.  Roots are computed with
 * shampoo_inverse_pth_root_batched over the groups of the tensor plan (the
 * packing is the matrix plan's). */
#define SHAMPOO_MAX_ORDER 4

/* One parameter tensor (HOST array): contiguous row-major fp32 of dims[0..order-1]. */
typedef struct {
  const float* G; /* gradient                                   */
  float* D;       /* diagonal AdaGrad accumulator (nullable)     */
  float* P;       /* preconditioned-gradient output (nullable for the statistics call) */
  int64_t dims[SHAMPOO_MAX_ORDER]; /* unused trailing entries = 1 */
  int32_t order;                   /* 1..4                         */
  int32_t reserved;
} shampoo_ttensor_t;

/* One block (sub-tensor) of an order-k tensor (plan output; integer, bit-exact
 * vs oracle/tensor.py).  136 bytes.  Entries i >= order: extent 1, p 0. */
typedef struct {
  int32_t tensor_id, order;
  int64_t origin[SHAMPOO_MAX_ORDER];
  int32_t extent[SHAMPOO_MAX_ORDER];
  int32_t p[SHAMPOO_MAX_ORDER];     /* root order of mode i (2k'), 0 = not preconditioned */
  int32_t owner[SHAMPOO_MAX_ORDER]; /* rank that updates H_i and computes its root, -1    */
  int32_t ld[SHAMPOO_MAX_ORDER];    /* leading dim of H_i = roundup(extent_i, 4)         */
  int64_t off[SHAMPOO_MAX_ORDER];   /* packed offset of H_i (and its root), -1           */
} shampoo_tblock_t;

/* Plan for tensors (rule above; blocks row-major over each tensor's block grid,
 * tensors in caller order; roots sorted by (n^3 products(p) desc, tensor, block,
 * mode), LPT owners; packing as shampoo_plan, r = 1).
 *   dims (host) SHAMPOO_MAX_ORDER int64 per tensor; orders (host) int32 per tensor.
 * Returns SHAMPOO_ERR_CAPACITY (counts still written) if an array is too small. */
int shampoo_tensor_plan(const int64_t* dims, const int32_t* orders, int32_t n_tensors, int32_t block_size,
                        int64_t max_precond_dim, int32_t world_size, shampoo_tblock_t* blocks, int32_t capacity,
                        int32_t* n_blocks, shampoo_group_t* groups, int32_t group_capacity, int32_t* n_groups,
                        int64_t* stats_elems, int64_t* segment_elems);

/* Statistics step for every block (Alg. 1 P:594-601 per mode):
 *   non-finite G_B: block_status 2, H/D untouched, graft_num 0;
 *   else H_i <- decay*H_i + weight*U_i U_i^T for every kept mode i owned by
 *   only_owner (or all if < 0) under the CHUNKED sequential contract (reading
 *   #25: fp64 sums over chunks of 4096 unfolding columns, chunk sums added in
 *   ascending order, then the §6.2 epilogue) -- BIT-EXACT with the oracle;
 *   D_B <- D_B + G_B o G_B and graft_num[b] = sum g^2 / max(D, 1e-30) for every block.
 * tensors_host / blocks_host: HOST tables (job tables are derived and uploaded
 * into the workspace).  workspace >= shampoo_tensor_stats_workspace_bytes(...). */
size_t shampoo_tensor_stats_workspace_bytes(const shampoo_ttensor_t* tensors_host, int32_t n_tensors,
                                            const shampoo_tblock_t* blocks_host, int32_t n_blocks,
                                            int32_t only_owner);
int shampoo_tensor_stats_update(const shampoo_ttensor_t* tensors_host, int32_t n_tensors,
                                const shampoo_tblock_t* blocks_host, int32_t n_blocks, int32_t only_owner,
                                float* stats, double decay, double weight, double* graft_num,
                                int32_t* block_status, void* workspace, size_t workspace_bytes,
                                shampoo_stream_t stream);

/* Preconditioned gradient and graft scale for every block:
 *   P_B = B x_0 X_0 x_1 X_1 ... over the kept modes (X_i = root at off[i]);
 *   no kept mode: P_B = D_B^{-1/2} o G_B (reading #17);
 *   graft_scale[b] = sqrt(graft_num[b]) / ||P_B||_F (0 if ||P_B|| = 0).
 * Mode products run in fp64 (FP64 DMMA tiles for modes > 32, fp64 FMA fibres
 * for small modes) with fp32 intermediates; parity is tolerance-based (1e-3).
 * workspace >= shampoo_tensor_precondition_workspace_bytes(...). */
size_t shampoo_tensor_precondition_workspace_bytes(const shampoo_ttensor_t* tensors_host, int32_t n_tensors,
                                                   const shampoo_tblock_t* blocks_host, int32_t n_blocks);
int shampoo_tensor_precondition(const shampoo_ttensor_t* tensors_host, int32_t n_tensors,
                                const shampoo_tblock_t* blocks_host, int32_t n_blocks, const float* roots,
                                const double* graft_num, float* graft_scale, double* den, void* workspace,
                                size_t workspace_bytes, shampoo_stream_t stream);

/* Kernel timing for measurement (bench.py's roofline): between
 * shampoo_profile_begin() and shampoo_profile_end(), every launch of the
 * library's dominant kernels ("root_kernel", "ozaki_gemm") on this host thread
 * is bracketed by CUDA events recorded on its launching stream.  end()
 * synchronizes those events and returns the summed milliseconds and the launch
 * count of `kernel` (NULL: all). */
int shampoo_profile_begin(void);
int shampoo_profile_end(const char* kernel, double* ms, int64_t* launches);
/* After shampoo_profile_end(): the duration (ms, host array `out` of
 * `capacity` floats) of each recorded launch of `kernel` (NULL: all) in launch
 * order; *n receives the number of such launches (may exceed capacity: only
 * the first `capacity` are written).  Lets the caller separate launches that
 * did work from the early-exit launches of converged batches. */
int shampoo_profile_launch_ms(const char* kernel, float* out, int64_t capacity, int64_t* n);

/* Number of kernel launches the last compute call on this host thread
 * enqueued (bench accounting, "gpu_launches"). */
int64_t shampoo_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SHAMPOO_H_ */
