// abi.cpp -- the extern "C" entry points of libshampoo (include/shampoo.h):
// host-side validation, error reporting and dispatch to the CUDA launchers.
#include <atomic>
#include <map>
#include <mutex>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "internal.h"

namespace shp {

static thread_local char g_err[512] = "";
static thread_local int64_t g_launches = 0;

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

int set_cuda_error(const char* what, cudaError_t e) {
  return set_error(SHAMPOO_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ------------------------------------------------------------- profiling
// Event pairs around launches of named kernels (bench.py's roofline timing).
struct ProfRec {
  const char* name;
  cudaEvent_t e0, e1;
};
static thread_local bool g_prof = false;
static thread_local std::vector<ProfRec>* g_prof_recs = nullptr;

void prof_begin_launch(const char* name, cudaStream_t stream, void** token) {
  *token = nullptr;
  if (!g_prof) return;
  ProfRec r{name, nullptr, nullptr};
  cudaEventCreate(&r.e0);
  cudaEventCreate(&r.e1);
  cudaEventRecord(r.e0, stream);
  g_prof_recs->push_back(r);
  *token = reinterpret_cast<void*>(g_prof_recs->size());
}

void prof_end_launch(void* token, cudaStream_t stream) {
  if (!g_prof || !token) return;
  cudaEventRecord((*g_prof_recs)[reinterpret_cast<size_t>(token) - 1].e1, stream);
}

// Per-device caches (a process may drive several GPUs, e.g. tests on cuda:1 after cuda:0): the SM count and the
// dynamic shared-memory opt-in are properties of the current device's context, not of the process.
static constexpr int kMaxDevices = 64;

int num_sms() {
  static std::atomic<int> n[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int v = n[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    n[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

cudaError_t ensure_smem(const void* func, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(dev, func);
  auto it = done.find(key);
  if (it != done.end() && it->second >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done[key] = smem;
  return e;
}

int plan_impl(const int64_t* shapes, int32_t n_tensors, int32_t block_size, int64_t max_precond_dim,
              int32_t world_size, int32_t split_num, int32_t split_den, shampoo_block_t* out_blocks, int32_t capacity, int32_t* n_blocks_out,
              shampoo_group_t* out_groups, int32_t group_capacity, int32_t* n_groups_out, int64_t* stats_elems,
              int64_t* segment_elems, int32_t layer_owners, int32_t* tensor_owner_out);

int tensor_plan_impl(const int64_t* dims, const int32_t* orders, int32_t n_tensors, int32_t block_size,
                     int64_t max_precond_dim, int32_t world_size, shampoo_tblock_t* out_blocks, int32_t capacity,
                     int32_t* n_blocks_out, shampoo_group_t* out_groups, int32_t group_capacity,
                     int32_t* n_groups_out, int64_t* stats_elems, int64_t* segment_elems);

// host tables of the tensor path: orders, extents inside the tensor, pointers
static int check_tensor_tables(const shampoo_ttensor_t* T, int32_t n_tensors, const shampoo_tblock_t* B,
                               int32_t n_blocks, bool need_p) {
  if (!T || !B) return set_error(SHAMPOO_ERR_INVALID_ARG, "null tensor/block table");
  for (int32_t t = 0; t < n_tensors; ++t) {
    if (T[t].order < 1 || T[t].order > SHAMPOO_MAX_ORDER)
      return set_error(SHAMPOO_ERR_INVALID_ARG, "tensor %d: order %d", t, T[t].order);
    if (!T[t].G || (need_p && !T[t].P)) return set_error(SHAMPOO_ERR_INVALID_ARG, "tensor %d: null G or P", t);
    for (int i = 0; i < T[t].order; ++i)
      if (T[t].dims[i] < 1) return set_error(SHAMPOO_ERR_INVALID_ARG, "tensor %d: dim %d < 1", t, i);
  }
  for (int32_t b = 0; b < n_blocks; ++b) {
    const shampoo_tblock_t& k = B[b];
    if (k.tensor_id < 0 || k.tensor_id >= n_tensors)
      return set_error(SHAMPOO_ERR_INVALID_ARG, "block %d: tensor_id out of range", b);
    const shampoo_ttensor_t& t = T[k.tensor_id];
    if (k.order != t.order) return set_error(SHAMPOO_ERR_INVALID_ARG, "block %d: order mismatch", b);
    bool any = false;
    for (int i = 0; i < k.order; ++i) {
      if (k.extent[i] < 1 || k.origin[i] < 0 || k.origin[i] + k.extent[i] > t.dims[i])
        return set_error(SHAMPOO_ERR_INVALID_ARG, "block %d: mode %d outside the tensor", b, i);
      if (k.p[i] && (k.p[i] > 16 || k.off[i] < 0 || k.ld[i] < k.extent[i]))
        return set_error(SHAMPOO_ERR_INVALID_ARG, "block %d: mode %d has a bad root entry", b, i);
      any |= k.p[i] != 0;
    }
    if (need_p && !any && !t.D)
      return set_error(SHAMPOO_ERR_INVALID_ARG, "block %d: diagonal-only block needs D", b);
  }
  return SHAMPOO_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static int check_ws(const void* ws, size_t have, size_t need) {
  if (need == 0) return SHAMPOO_OK;
  if (!ws || have < need)
    return set_error(SHAMPOO_ERR_WORKSPACE, "workspace too small: have %zu bytes, need %zu", have, need);
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return set_error(SHAMPOO_ERR_WORKSPACE, "workspace not 256-B aligned");
  return SHAMPOO_OK;
}

static bool valid_p(int p) { return p >= 1 && p <= 16; }

}  // namespace shp

using namespace shp;

extern "C" {

int shampoo_abi_version(void) { return SHAMPOO_ABI_VERSION; }

int shampoo_profile_begin(void) {
  if (!g_prof_recs) g_prof_recs = new std::vector<ProfRec>();
  for (auto& r : *g_prof_recs) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  g_prof_recs->clear();
  g_prof = true;
  return SHAMPOO_OK;
}

int shampoo_profile_end(const char* kernel, double* ms, int64_t* launches) {
  g_prof = false;
  double total = 0.0;
  int64_t count = 0;
  if (g_prof_recs) {
    for (auto& r : *g_prof_recs) {
      if (kernel && std::strcmp(kernel, r.name) != 0) continue;
      float t = 0.0f;
      if (cudaEventSynchronize(r.e1) != cudaSuccess || cudaEventElapsedTime(&t, r.e0, r.e1) != cudaSuccess)
        return set_cuda_error("shampoo_profile_end");
      total += t;
      ++count;
    }
  }
  if (ms) *ms = total;
  if (launches) *launches = count;
  return SHAMPOO_OK;
}

int shampoo_profile_launch_ms(const char* kernel, float* out, int64_t capacity, int64_t* n) {
  int64_t count = 0;
  if (g_prof_recs) {
    for (auto& r : *g_prof_recs) {
      if (kernel && std::strcmp(kernel, r.name) != 0) continue;
      if (out && count < capacity) {
        float t = 0.0f;
        if (cudaEventSynchronize(r.e1) != cudaSuccess || cudaEventElapsedTime(&t, r.e0, r.e1) != cudaSuccess)
          return set_cuda_error("shampoo_profile_launch_ms");
        out[count] = t;
      }
      ++count;
    }
  }
  if (n) *n = count;
  return SHAMPOO_OK;
}

const char* shampoo_last_error(void) { return g_err; }

int64_t shampoo_last_launch_count(void) { return g_launches; }

int shampoo_plan(const int64_t* shapes, int32_t n_tensors, int32_t block_size, int64_t max_precond_dim,
                 int32_t world_size, int32_t split_num, int32_t split_den, shampoo_block_t* blocks, int32_t capacity, int32_t* n_blocks,
                 shampoo_group_t* groups, int32_t group_capacity, int32_t* n_groups, int64_t* stats_elems,
                 int64_t* segment_elems) {
  g_err[0] = 0;
  return plan_impl(shapes, n_tensors, block_size, max_precond_dim, world_size, split_num, split_den, blocks, capacity, n_blocks, groups,
                   group_capacity, n_groups, stats_elems, segment_elems, 0, nullptr);
}

int shampoo_plan_layers(const int64_t* shapes, int32_t n_tensors, int32_t block_size, int64_t max_precond_dim,
                        int32_t world_size, int32_t split_num, int32_t split_den, shampoo_block_t* blocks,
                        int32_t capacity, int32_t* n_blocks, shampoo_group_t* groups, int32_t group_capacity,
                        int32_t* n_groups, int64_t* stats_elems, int64_t* segment_elems, int32_t* tensor_owner) {
  g_err[0] = 0;
  return plan_impl(shapes, n_tensors, block_size, max_precond_dim, world_size, split_num, split_den, blocks, capacity,
                   n_blocks, groups, group_capacity, n_groups, stats_elems, segment_elems, 1, tensor_owner);
}

size_t shampoo_stats_workspace_bytes(const shampoo_block_t* blocks_host, int32_t n_blocks, int32_t only_owner) {
  return (n_blocks > 0 && blocks_host) ? stats_workspace_bytes(blocks_host, n_blocks, only_owner) : 0;
}

int shampoo_stats_update(const shampoo_tensor_t* tensors, int32_t n_tensors, const shampoo_block_t* blocks,
                         const shampoo_block_t* blocks_host, int32_t n_blocks, int32_t only_owner, float* stats,
                         double decay, double weight, double* graft_num, int32_t* block_status, void* workspace,
                         size_t workspace_bytes, shampoo_stream_t stream) {
  g_err[0] = 0;
  g_launches = 0;
  if (n_blocks < 0 || n_tensors < 0) return set_error(SHAMPOO_ERR_INVALID_ARG, "negative counts");
  if (n_blocks == 0) return SHAMPOO_OK;
  if (!tensors || !blocks || !blocks_host) return set_error(SHAMPOO_ERR_INVALID_ARG, "null tensor/block table");
  if (!std::isfinite(decay) || !std::isfinite(weight))
    return set_error(SHAMPOO_ERR_INVALID_ARG, "decay/weight must be finite");
  if (!stats) return set_error(SHAMPOO_ERR_INVALID_ARG, "null statistics buffer");
  if (!aligned16(stats)) return set_error(SHAMPOO_ERR_INVALID_ARG, "statistics buffer not 16-B aligned");
  int rc = check_ws(workspace, workspace_bytes, stats_workspace_bytes(blocks_host, n_blocks, only_owner));
  if (rc) return rc;
  return stats_launch(tensors, n_tensors, blocks, n_blocks, only_owner, stats, decay, weight, graft_num, block_status,
                      workspace, static_cast<cudaStream_t>(stream), &g_launches);
}

size_t shampoo_root_workspace_bytes(int32_t batch, int32_t n, int32_t p, int32_t max_iter) {
  (void)p;
  if (batch <= 0 || n <= 0 || max_iter < 0) return 0;
  return root_workspace_bytes(batch, n, max_iter, 0);
}

int shampoo_inverse_pth_root_batched(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                     int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                     double tol, int32_t max_iter, int32_t power_iters,
                                     shampoo_root_info_t* info, void* workspace, size_t workspace_bytes,
                                     shampoo_stream_t stream) {
  return shampoo_inverse_root_rational_batched(A, lda, stride_a, X, ldx, stride_x, batch, n, p, 1, eps_rel, tol,
                                               max_iter, power_iters, info, workspace, workspace_bytes, stream);
}

static int root_entry(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx, int64_t stride_x,
                      int32_t batch, int32_t n, int32_t p, int32_t r, int32_t k_sw, double eps_rel, double tol,
                      int32_t max_iter, int32_t power_iters, shampoo_root_info_t* info, void* workspace,
                      size_t workspace_bytes, shampoo_stream_t stream, int precision = 0, int slices = 7,
                      double slice_budget = 0.0);

int shampoo_ozaki_iteration_slices(int32_t k, int32_t p, int32_t n, double eps_rel, double slice_budget,
                                   int32_t slices) {
  return ozaki_iteration_slices(k, p, n, eps_rel, slice_budget, slices);
}

size_t shampoo_root_ozaki_workspace_bytes(int32_t batch, int32_t n, int32_t p, int32_t max_iter) {
  (void)p;
  if (batch <= 0 || n <= 0 || max_iter < 0) return 0;
  return root_workspace_bytes(batch, n, max_iter, 2);
}

int shampoo_inverse_pth_root_batched_ozaki(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                           int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                           double tol, int32_t max_iter, int32_t power_iters, int32_t slices,
                                           double slice_budget, shampoo_root_info_t* info, void* workspace,
                                           size_t workspace_bytes, shampoo_stream_t stream) {
  return root_entry(A, lda, stride_a, X, ldx, stride_x, batch, n, p, 1, 0, eps_rel, tol, max_iter, power_iters, info,
                    workspace, workspace_bytes, stream, 2, slices, slice_budget);
}

size_t shampoo_root_auto_workspace_bytes(int32_t batch, int32_t n, int32_t p, int32_t max_iter) {
  return n >= SHAMPOO_OZAKI_MIN_N ? shampoo_root_ozaki_workspace_bytes(batch, n, p, max_iter)
                                  : shampoo_root_workspace_bytes(batch, n, p, max_iter);
}

int shampoo_inverse_pth_root_batched_auto(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                          int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                          double tol, int32_t max_iter, int32_t power_iters, int32_t slices,
                                          double slice_budget, shampoo_root_info_t* info, void* workspace,
                                          size_t workspace_bytes, shampoo_stream_t stream) {
  if (n >= SHAMPOO_OZAKI_MIN_N)
    return shampoo_inverse_pth_root_batched_ozaki(A, lda, stride_a, X, ldx, stride_x, batch, n, p, eps_rel, tol,
                                                  max_iter, power_iters, slices, slice_budget, info, workspace,
                                                  workspace_bytes, stream);
  return shampoo_inverse_pth_root_batched(A, lda, stride_a, X, ldx, stride_x, batch, n, p, eps_rel, tol, max_iter,
                                          power_iters, info, workspace, workspace_bytes, stream);
}

int shampoo_inverse_root_rational_batched(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                          int64_t stride_x, int32_t batch, int32_t n, int32_t p, int32_t r,
                                          double eps_rel, double tol, int32_t max_iter, int32_t power_iters,
                                          shampoo_root_info_t* info, void* workspace, size_t workspace_bytes,
                                          shampoo_stream_t stream) {
  return root_entry(A, lda, stride_a, X, ldx, stride_x, batch, n, p, r, max_iter + 1, eps_rel, tol, max_iter,
                    power_iters, info, workspace, workspace_bytes, stream);
}

// a-priori switch of the hybrid root: after k fp64 iterations
// the smallest eigenvalue of M is at least eps_rel * g^k, g = (1 + 1/p)^p;
// switch once that reaches 1e-2 (measured on B200, n = 1024, kappa 1e6: a
// switch at 1e-3 (k = 8) leaves a 1.3e-3 root error -- the tensor core's fp32
// accumulation is biased on near-identity products -- at 1e-2 (k = 11) ~1e-4;
// p = 1 at 1e-2 measured 3.1e-4, hence 1e-1 for p <= 3)
static int auto_fp64_iters(int p, double eps_rel) {
  if (!(eps_rel > 0.0)) return -1;
  const double g = std::pow(1.0 + 1.0 / p, (double)p);
  // low orders amplify product errors more (X ~ A_hat^{-1/p}): p <= 3 switches at 1e-1
  const double thr = p <= 3 ? 1e-1 : 1e-2;
  int k = (int)std::ceil(std::log(thr / eps_rel) / std::log(g));
  return k < 1 ? 1 : k;
}

int shampoo_inverse_pth_root_batched_hybrid(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx,
                                            int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                            double tol, int32_t max_iter, int32_t power_iters, int32_t fp64_iters,
                                            shampoo_root_info_t* info, void* workspace, size_t workspace_bytes,
                                            shampoo_stream_t stream) {
  int k_sw = fp64_iters;
  if (k_sw < 0) {
    k_sw = auto_fp64_iters(p, eps_rel);
    if (k_sw < 0) k_sw = max_iter + 1;  // no ridge: no a-priori bound, stay in fp64
  }
  if (k_sw == 0) {
    g_err[0] = 0;
    return set_error(SHAMPOO_ERR_INVALID_ARG, "fp64_iters must be >= 1 (or -1 for automatic)");
  }
  if (k_sw > max_iter) k_sw = max_iter + 1;
  return root_entry(A, lda, stride_a, X, ldx, stride_x, batch, n, p, 1, k_sw, eps_rel, tol, max_iter, power_iters,
                    info, workspace, workspace_bytes, stream);
}

static int root_entry(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx, int64_t stride_x,
                      int32_t batch, int32_t n, int32_t p, int32_t r, int32_t k_sw, double eps_rel, double tol,
                      int32_t max_iter, int32_t power_iters, shampoo_root_info_t* info, void* workspace,
                      size_t workspace_bytes, shampoo_stream_t stream, int precision, int slices,
                      double slice_budget) {
  g_err[0] = 0;
  g_launches = 0;
  if (batch < 0) return set_error(SHAMPOO_ERR_INVALID_ARG, "batch < 0");
  if (batch == 0) return SHAMPOO_OK;
  if (n < 1 || n > 8192) return set_error(SHAMPOO_ERR_INVALID_ARG, "n = %d outside [1, 8192]", n);
  if (!valid_p(p)) return set_error(SHAMPOO_ERR_INVALID_ARG, "p = %d not in [1, 16]", p);
  if (r < 1 || r > p) return set_error(SHAMPOO_ERR_INVALID_ARG, "r = %d not in [1, p = %d]", r, p);
  if (!A || !X || !info) return set_error(SHAMPOO_ERR_INVALID_ARG, "null A, X or info");
  if (lda < n || ldx < n) return set_error(SHAMPOO_ERR_INVALID_ARG, "leading dimension < n");
  if (batch > 1 && (stride_a < lda * (int64_t)(n - 1) + n || stride_x < ldx * (int64_t)(n - 1) + n))
    return set_error(SHAMPOO_ERR_INVALID_ARG, "batch stride too small");
  if (!std::isfinite(eps_rel) || eps_rel < 0 || !std::isfinite(tol) || tol < 0)
    return set_error(SHAMPOO_ERR_INVALID_ARG, "eps_rel / tol must be finite and >= 0");
  if (max_iter < 0 || max_iter > 1000 || power_iters < 1)
    return set_error(SHAMPOO_ERR_INVALID_ARG, "max_iter in [0, 1000], power_iters >= 1");
  if (precision == 2 && slices != 6 && slices != 7)
    return set_error(SHAMPOO_ERR_INVALID_ARG, "slices = %d not in {6, 7}", slices);
  if (precision == 2 && !(slice_budget >= 0.0 && slice_budget < 1.0))
    return set_error(SHAMPOO_ERR_INVALID_ARG, "slice_budget must be in [0, 1)");
  if (precision == 2 && max_iter < 1) precision = 0;  // nothing to iterate: the fp64 kernel decides at k = 0
  const int mode = precision ? precision : (k_sw <= max_iter ? 1 : 0);
  int rc = check_ws(workspace, workspace_bytes, root_workspace_bytes(batch, n, max_iter, mode));
  if (rc) return rc;
  return root_launch(A, lda, stride_a, X, ldx, stride_x, batch, n, p, r, k_sw, precision, slices, slice_budget,
                     eps_rel, tol,
                     max_iter,
                     power_iters, info,
                     workspace, static_cast<cudaStream_t>(stream), &g_launches);
}

size_t shampoo_root_residual_workspace_bytes(int32_t batch, int32_t n, int32_t p) {
  (void)p;
  if (batch <= 0 || n <= 0) return 0;
  return residual_workspace_bytes(batch, n);
}

int shampoo_root_residual_batched(const float* A, int64_t lda, int64_t stride_a, const float* X, int64_t ldx,
                                  int64_t stride_x, int32_t batch, int32_t n, int32_t p, double eps_rel,
                                  const shampoo_root_info_t* info, double* residual, void* workspace,
                                  size_t workspace_bytes, shampoo_stream_t stream) {
  g_err[0] = 0;
  g_launches = 0;
  if (batch < 0) return set_error(SHAMPOO_ERR_INVALID_ARG, "batch < 0");
  if (batch == 0) return SHAMPOO_OK;
  if (n < 1 || n > 8192) return set_error(SHAMPOO_ERR_INVALID_ARG, "n = %d outside [1, 8192]", n);
  if (!valid_p(p)) return set_error(SHAMPOO_ERR_INVALID_ARG, "p = %d not in [1, 16]", p);
  if (!A || !X || !info || !residual) return set_error(SHAMPOO_ERR_INVALID_ARG, "null argument");
  if (lda < n || ldx < n) return set_error(SHAMPOO_ERR_INVALID_ARG, "leading dimension < n");
  if (!std::isfinite(eps_rel) || eps_rel < 0) return set_error(SHAMPOO_ERR_INVALID_ARG, "eps_rel");
  int rc = check_ws(workspace, workspace_bytes, residual_workspace_bytes(batch, n));
  if (rc) return rc;
  return residual_launch(A, lda, stride_a, X, ldx, stride_x, batch, n, p, eps_rel, info, residual, workspace,
                         static_cast<cudaStream_t>(stream), &g_launches);
}

size_t shampoo_precondition_workspace_bytes(const shampoo_tensor_t* tensors_host, int32_t n_tensors,
                                            const shampoo_block_t* blocks_host, int32_t n_blocks) {
  if (!tensors_host || !blocks_host || n_blocks <= 0 || n_tensors <= 0) return 0;
  return precondition_workspace_bytes(tensors_host, n_tensors, blocks_host, n_blocks);
}

int shampoo_precondition(const shampoo_tensor_t* tensors_host, int32_t n_tensors, const shampoo_block_t* blocks_host,
                         int32_t n_blocks, const float* roots, const double* graft_num, float* graft_scale,
                         double* den, void* workspace, size_t workspace_bytes, shampoo_stream_t stream) {
  return shampoo_precondition_split(tensors_host, n_tensors, blocks_host, n_blocks, roots, nullptr, graft_num,
                                    graft_scale, den, workspace, workspace_bytes, stream);
}

int shampoo_tf32_split(const float* x, float* lo, int64_t n, shampoo_stream_t stream) {
  g_err[0] = 0;
  g_launches = 0;
  if (n < 0 || (n & 3)) return set_error(SHAMPOO_ERR_INVALID_ARG, "n must be a non-negative multiple of 4");
  if (n == 0) return SHAMPOO_OK;
  if (!x || !lo || !aligned16(x) || !aligned16(lo)) return set_error(SHAMPOO_ERR_INVALID_ARG, "x / lo not 16-B aligned");
  return split_flat_launch(x, lo, n, static_cast<cudaStream_t>(stream), &g_launches);
}

int shampoo_precondition_split(const shampoo_tensor_t* tensors_host, int32_t n_tensors,
                               const shampoo_block_t* blocks_host, int32_t n_blocks, const float* roots,
                               const float* roots_lo, const double* graft_num, float* graft_scale, double* den,
                               void* workspace, size_t workspace_bytes, shampoo_stream_t stream) {
  g_err[0] = 0;
  g_launches = 0;
  if (n_blocks < 0 || n_tensors < 0) return set_error(SHAMPOO_ERR_INVALID_ARG, "negative counts");
  if (n_blocks == 0) return SHAMPOO_OK;
  if (!tensors_host || !blocks_host || !roots) return set_error(SHAMPOO_ERR_INVALID_ARG, "null tensor/block/roots");
  for (int32_t b = 0; b < n_blocks; ++b)
    if (blocks_host[b].tensor_id < 0 || blocks_host[b].tensor_id >= n_tensors)
      return set_error(SHAMPOO_ERR_INVALID_ARG, "block %d: tensor_id out of range", b);
  for (int32_t t = 0; t < n_tensors; ++t)
    if (!tensors_host[t].G || !tensors_host[t].P) return set_error(SHAMPOO_ERR_INVALID_ARG, "tensor %d: null G or P", t);
  if (!workspace) return set_error(SHAMPOO_ERR_WORKSPACE, "null workspace");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return set_error(SHAMPOO_ERR_WORKSPACE, "workspace not 256-B aligned");
  if (roots_lo && !aligned16(roots_lo)) return set_error(SHAMPOO_ERR_INVALID_ARG, "roots_lo not 16-B aligned");
  return precondition_launch(tensors_host, n_tensors, blocks_host, n_blocks, roots, roots_lo, graft_num, graft_scale,
                             den, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), &g_launches);
}

int shampoo_tensor_plan(const int64_t* dims, const int32_t* orders, int32_t n_tensors, int32_t block_size,
                        int64_t max_precond_dim, int32_t world_size, shampoo_tblock_t* blocks, int32_t capacity,
                        int32_t* n_blocks, shampoo_group_t* groups, int32_t group_capacity, int32_t* n_groups,
                        int64_t* stats_elems, int64_t* segment_elems) {
  g_err[0] = 0;
  return tensor_plan_impl(dims, orders, n_tensors, block_size, max_precond_dim, world_size, blocks, capacity,
                          n_blocks, groups, group_capacity, n_groups, stats_elems, segment_elems);
}

size_t shampoo_tensor_stats_workspace_bytes(const shampoo_ttensor_t* tensors_host, int32_t n_tensors,
                                            const shampoo_tblock_t* blocks_host, int32_t n_blocks,
                                            int32_t only_owner) {
  if (n_blocks <= 0 || check_tensor_tables(tensors_host, n_tensors, blocks_host, n_blocks, false)) return 0;
  return tensor_stats_workspace_bytes(tensors_host, blocks_host, n_blocks, only_owner);
}

int shampoo_tensor_stats_update(const shampoo_ttensor_t* tensors_host, int32_t n_tensors,
                                const shampoo_tblock_t* blocks_host, int32_t n_blocks, int32_t only_owner,
                                float* stats, double decay, double weight, double* graft_num,
                                int32_t* block_status, void* workspace, size_t workspace_bytes,
                                shampoo_stream_t stream) {
  g_err[0] = 0;
  g_launches = 0;
  if (n_blocks < 0 || n_tensors < 0) return set_error(SHAMPOO_ERR_INVALID_ARG, "negative counts");
  if (n_blocks == 0) return SHAMPOO_OK;
  int rc = check_tensor_tables(tensors_host, n_tensors, blocks_host, n_blocks, false);
  if (rc) return rc;
  if (!std::isfinite(decay) || !std::isfinite(weight))
    return set_error(SHAMPOO_ERR_INVALID_ARG, "decay/weight must be finite");
  if (!stats) return set_error(SHAMPOO_ERR_INVALID_ARG, "null statistics buffer");
  if (!workspace) return set_error(SHAMPOO_ERR_WORKSPACE, "null workspace");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return set_error(SHAMPOO_ERR_WORKSPACE, "workspace not 256-B aligned");
  return tensor_stats_launch(tensors_host, blocks_host, n_blocks, only_owner, stats, decay, weight, graft_num,
                             block_status, workspace, workspace_bytes, static_cast<cudaStream_t>(stream),
                             &g_launches);
}

size_t shampoo_tensor_precondition_workspace_bytes(const shampoo_ttensor_t* tensors_host, int32_t n_tensors,
                                                   const shampoo_tblock_t* blocks_host, int32_t n_blocks) {
  if (n_blocks <= 0 || check_tensor_tables(tensors_host, n_tensors, blocks_host, n_blocks, false)) return 0;
  return tensor_precondition_workspace_bytes(tensors_host, blocks_host, n_blocks);
}

int shampoo_tensor_precondition(const shampoo_ttensor_t* tensors_host, int32_t n_tensors,
                                const shampoo_tblock_t* blocks_host, int32_t n_blocks, const float* roots,
                                const double* graft_num, float* graft_scale, double* den, void* workspace,
                                size_t workspace_bytes, shampoo_stream_t stream) {
  g_err[0] = 0;
  g_launches = 0;
  if (n_blocks < 0 || n_tensors < 0) return set_error(SHAMPOO_ERR_INVALID_ARG, "negative counts");
  if (n_blocks == 0) return SHAMPOO_OK;
  int rc = check_tensor_tables(tensors_host, n_tensors, blocks_host, n_blocks, true);
  if (rc) return rc;
  if (!roots) return set_error(SHAMPOO_ERR_INVALID_ARG, "null roots");
  if (!workspace) return set_error(SHAMPOO_ERR_WORKSPACE, "null workspace");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return set_error(SHAMPOO_ERR_WORKSPACE, "workspace not 256-B aligned");
  return tensor_precondition_launch(tensors_host, blocks_host, n_blocks, roots, graft_num, graft_scale, den,
                                    workspace, workspace_bytes, static_cast<cudaStream_t>(stream), &g_launches);
}

size_t shampoo_momentum_workspace_bytes(int32_t n_blocks) { return n_blocks > 0 ? momentum_workspace_bytes(n_blocks) : 0; }

int shampoo_momentum_step(const shampoo_tensor_t* tensors, const shampoo_state_t* states, int32_t n_tensors,
                          const shampoo_block_t* blocks, int32_t n_blocks, double beta1, double eta0,
                          int32_t shampoo_branch, double* eta_out, void* workspace, size_t workspace_bytes,
                          shampoo_stream_t stream) {
  g_err[0] = 0;
  g_launches = 0;
  if (n_blocks < 0 || n_tensors < 0) return set_error(SHAMPOO_ERR_INVALID_ARG, "negative counts");
  if (n_blocks == 0) return SHAMPOO_OK;
  if (!tensors || !states || !blocks) return set_error(SHAMPOO_ERR_INVALID_ARG, "null table");
  if (!std::isfinite(beta1) || beta1 < 0.0 || beta1 >= 1.0 || !std::isfinite(eta0))
    return set_error(SHAMPOO_ERR_INVALID_ARG, "beta1 must be in [0, 1) and eta0 finite");
  int rc = check_ws(workspace, workspace_bytes, momentum_workspace_bytes(n_blocks));
  if (rc) return rc;
  return momentum_launch(tensors, states, blocks, n_blocks, beta1, eta0, shampoo_branch ? 1 : 0, eta_out, workspace,
                         static_cast<cudaStream_t>(stream), &g_launches);
}

}  // extern "C"
