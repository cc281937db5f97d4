// rowops.cuh -- per-token row traversal shared by the combine pass (layout.cu) and the
// standalone residual + RMSNorm (router.cu): one CTA per token, thread t owns the
// 8-element chunks t, t + nthreads, ... of the row. Both kernels use this exact
// traversal and reduction tree, so the unfused expert-parallel step reproduces the
// fused single-GPU step bit for bit.
#pragma once
#include <cuda_runtime.h>

namespace sere {

constexpr int kRowVec = 8;

__host__ __device__ inline int row_threads(int d_h) {
  int t = ((d_h + kRowVec - 1) / kRowVec + 31) / 32 * 32;
  return t < 32 ? 32 : (t > 256 ? 256 : t);
}

// sum over the block (warp xor tree, then warps in index order); s_red >= 8 floats
__device__ __forceinline__ float block_sum(float v, float* s_red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < (blockDim.x + 31) / 32; ++i) tot += s_red[i];
  __syncthreads();
  return tot;
}

}  // namespace sere
