// internal.h -- host-side helpers shared by the libshampoo translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stddef.h>
#include <stdint.h>

#include "shampoo.h"

namespace shp {

int set_error(int code, const char* fmt, ...);
int set_cuda_error(const char* what, cudaError_t e = cudaGetLastError());

// root.cu
size_t root_workspace_bytes(int batch, int n, int max_iter, int precision);  // 0 fp64, 1 hybrid, 2 ozaki
int root_launch(const float* A, int64_t lda, int64_t stride_a, float* X, int64_t ldx, int64_t stride_x, int batch,
                int n, int p, int r, int k_sw, int precision, int slices, double slice_budget, double eps_rel,
                double tol, int max_iter, int power_iters,
                shampoo_root_info_t* info, void* ws, cudaStream_t stream, int64_t* launches);
// root_tail.cu (hybrid 3xTF32 tail)
size_t root_tail_ws_bytes(int batch);
size_t root_ozaki_ws_bytes(int batch, int n);
int root_ozaki_launch(double* bufs, int batch, int n, int np, int p, int max_iter, double tol, double* errh,
                      const int4* res, shampoo_root_info_t* info, float* X, int64_t ldx, int64_t stride_x, int* act,
                      int* nact, void* oz_ws, int slices, double eps_rel, double slice_budget, cudaStream_t stream,
                      int64_t* launches);
// slice count of Ozaki iteration k (reading #29; root_tail.cu)
int ozaki_iteration_slices(int k, int p, int n, double eps_rel, double budget, int s_max);
int root_tail_launch(double* bufs, int batch, int n, int np, int p, int max_iter, int k_sw, double tol, double* errh,
                     const int4* res, shampoo_root_info_t* info, float* X, int64_t ldx, int64_t stride_x, int* act,
                     int* nact, void* maps_ws, cudaStream_t stream, int64_t* launches);
size_t residual_workspace_bytes(int batch, int n);
int residual_launch(const float* A, int64_t lda, int64_t stride_a, const float* X, int64_t ldx, int64_t stride_x,
                    int batch, int n, int p, double eps_rel, const shampoo_root_info_t* info, double* residual,
                    void* ws, cudaStream_t stream, int64_t* launches);

// stats.cu
size_t stats_workspace_bytes(const shampoo_block_t* blocks_host, int n_blocks, int only_owner);
int stats_launch(const shampoo_tensor_t* tensors, int n_tensors, const shampoo_block_t* blocks, int n_blocks,
                 int only_owner, float* stats, double decay, double weight, double* graft_num, int32_t* block_status,
                 void* ws, cudaStream_t stream, int64_t* launches);

// precondition.cu
size_t precondition_workspace_bytes(const shampoo_tensor_t* tensors_host, int n_tensors,
                                    const shampoo_block_t* blocks_host, int n_blocks);
int precondition_launch(const shampoo_tensor_t* tensors_host, int n_tensors, const shampoo_block_t* blocks_host,
                        int n_blocks, const float* roots, const float* roots_lo, const double* graft_num,
                        float* graft_scale, double* den, void* ws, size_t ws_bytes, cudaStream_t stream,
                        int64_t* launches);
int split_flat_launch(const float* x, float* lo, int64_t n, cudaStream_t stream, int64_t* launches);

// momentum.cu
size_t momentum_workspace_bytes(int n_blocks);
int momentum_launch(const shampoo_tensor_t* tensors, const shampoo_state_t* states, const shampoo_block_t* blocks,
                    int n_blocks, double beta1, double eta0, int shampoo_branch, double* eta_out, void* ws,
                    cudaStream_t stream, int64_t* launches);

// tensor.cu (f3)
size_t tensor_stats_workspace_bytes(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks,
                                    int only_owner);
int tensor_stats_launch(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks, int only_owner,
                        float* stats, double decay, double weight, double* graft_num, int32_t* block_status,
                        void* ws, size_t ws_bytes, cudaStream_t stream, int64_t* launches);
size_t tensor_precondition_workspace_bytes(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks);
int tensor_precondition_launch(const shampoo_ttensor_t* T, const shampoo_tblock_t* B, int n_blocks,
                               const float* roots, const double* graft_num, float* graft_scale, double* den,
                               void* ws, size_t ws_bytes, cudaStream_t stream, int64_t* launches);

int num_sms();  // of the current device (cached per device)
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (current device, kernel, larger size); thread-safe
cudaError_t ensure_smem(const void* func, size_t smem);
// profiling hooks (shampoo_profile_begin/end): bracket a launch with events
void prof_begin_launch(const char* name, cudaStream_t stream, void** token);
void prof_end_launch(void* token, cudaStream_t stream);

}  // namespace shp
