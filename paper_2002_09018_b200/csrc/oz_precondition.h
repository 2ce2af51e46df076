// oz_precondition.h -- one-sided preconditioned gradient on the INT8 tensor cores (oz_precondition.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "shampoo.h"

namespace shp {

// an fp32 row source of the slicer: element (i, j) at src[i * ld + j]; rows >= rows, cols >= cols read as 0
struct OzSliceJob {
  const float* src;
  int64_t ld;
  int32_t rows, cols;
};

bool oz_precondition_eligible(const shampoo_block_t& b);
// flags[b] == 2 marks the blocks served here (host array)
size_t oz_precondition_bytes(const shampoo_block_t* blocks_host, int n_blocks, const int* flags);
int oz_precondition_launch(const shampoo_tensor_t* tensors_host, const shampoo_block_t* blocks_host, int n_blocks,
                           const int* flags, const float* roots, void* ws, cudaStream_t stream, int64_t* launches);

}  // namespace shp
