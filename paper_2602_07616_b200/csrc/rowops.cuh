// rowops.cuh -- per-token row traversal shared by the combine pass (layout.cu) and the
// standalone residual + RMSNorm (router.cu): one CTA per token; the row is walked in
// blocks of nthreads * 8 elements, and inside a block thread t owns the two 4-element
// chunks starting at 4*t and 4*(nthreads + t) -- every warp-wide 16-B access covers 512
// contiguous bytes (full sectors). Both kernels use this exact traversal and reduction
// tree, so the unfused expert-parallel step reproduces the fused single-GPU step bit
// for bit.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace sere {

#ifndef SERE_ROW_CHUNKS
#define SERE_ROW_CHUNKS 2
#endif
constexpr int kRowChunks = SERE_ROW_CHUNKS;  // 4-element chunks per thread per row block
constexpr int kRowVec = 4 * kRowChunks;
constexpr int kRowMaxThreads = 512;

__host__ __device__ inline int row_threads(int d_h) {
  int t = ((d_h + kRowVec - 1) / kRowVec + 31) / 32 * 32;
  return t < 32 ? 32 : (t > kRowMaxThreads ? kRowMaxThreads : t);
}

// element offset of chunk c (0/1) of thread tid in the row block starting at `base`
__device__ __forceinline__ int row_chunk(int base, int c) { return base + (c * blockDim.x + threadIdx.x) * 4; }

__device__ __forceinline__ void store_bf16x4(__nv_bfloat16* dst, const float (&v)[4]) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(dst) = u;
}

// sum over the block (warp xor tree, then warps in index order); s_red >= 16 floats
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
