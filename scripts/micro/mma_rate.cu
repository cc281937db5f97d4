// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, SS operands, 128B swizzle) issue
// rate for M=128 and several N, 4 MMAs (K=64) per commit -- the inner loop of moe_ffn_kernel.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_07616_b200/csrc/ptx.cuh"
using namespace sere;

// MMA issued by the whole converged warp; elect.sync inside the asm picks the issuing lane
__device__ __forceinline__ void umma_bf16_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
               : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_rate2(int n, int iters, int mw, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    const uint32_t idesc = umma_idesc_bf16(128, n);
    const uint32_t b_addr = smem_u32(smem);
    const uint64_t bdesc0 = umma_desc_sw128(b_addr);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < mw; ++j) {
        const uint64_t adesc0 = umma_desc_sw128(b_addr + 32768 + j * 16384);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16_elect(tbase + j * n, adesc0 + 2 * k, bdesc0 + 2 * k, idesc, (it > 0 || k > 0) ? 1u : 0u);
      }
      if ((it + 1) % MODE == 0) umma_commit_elect(&bar);
    }
    long long t1 = clock64();
    mbar_wait(&bar, (iters / MODE - 1) & 1);
    long long t2 = clock64();
    if (lane == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_order(int n, int iters, int mw, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    const uint32_t idesc = umma_idesc_bf16(128, n);
    const uint32_t b_addr = smem_u32(smem);
    const uint64_t bdesc0 = umma_desc_sw128(b_addr);
    const uint64_t adesc0 = umma_desc_sw128(b_addr + 32768);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE == 10) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          for (int j = 0; j < mw; ++j)
            umma_bf16_elect(tbase + j * n, adesc0 + 1024 * j + 2 * k, bdesc0 + 2 * k, idesc, (it > 0 || k > 0) ? 1u : 0u);
      } else {  // 2 alternating accumulators per A tile
#pragma unroll
        for (int k = 0; k < 4; ++k)
          for (int j = 0; j < mw; ++j)
            umma_bf16_elect(tbase + (2 * j + (k & 1)) * n, adesc0 + 1024 * j + 2 * k, bdesc0 + 2 * k, idesc,
                            (it > 0 || k > 1) ? 1u : 0u);
      }
      umma_commit_elect(&bar);
    }
    long long t1 = clock64();
    mbar_wait(&bar, (iters - 1) & 1);
    long long t2 = clock64();
    if (lane == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

__global__ void __launch_bounds__(128, 1) mma_two_issuers(int n, int iters, int mw, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if ((warp == 1 || warp == 2) && lane == 0) {
    const int w = warp - 1;
    const uint32_t idesc = umma_idesc_bf16(128, n);
    const uint32_t b_addr = smem_u32(smem);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < mw; ++j) {
        const uint32_t a_addr = b_addr + 32768 + (w * mw + j) * 16384;
        for (int k = 0; k < 4; ++k)
          umma_bf16(tbase + (w * mw + j) * n, umma_desc_sw128(a_addr + 32 * k), umma_desc_sw128(b_addr + 32 * k),
                    idesc, (it > 0 || k > 0) ? 1u : 0u);
      }
      umma_commit(&bar[w]);
    }
    mbar_wait(&bar[w], (iters - 1) & 1);
    long long t2 = clock64();
    if (w == 0) out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

__global__ void __launch_bounds__(128, 1) mma_rate(int n, int iters, int mw, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, n);
    const uint32_t b_addr = smem_u32(smem);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < mw; ++j) {
        const uint32_t a_addr = b_addr + 32768 + j * 16384;
        for (int k = 0; k < 4; ++k)
          umma_bf16(tbase + j * n, umma_desc_sw128(a_addr + 32 * k), umma_desc_sw128(b_addr + 32 * k), idesc,
                    (it > 0 || k > 0) ? 1u : 0u);
      }
      umma_commit(&bar);
    }
    long long t1 = clock64();
    mbar_wait(&bar, (iters - 1) & 1);
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(mma_two_issuers, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int ns[] = {16, 32, 64, 96, 128, 192, 256};
  for (int mw : {1, 2, 4}) {
    for (int n : ns) {
      if (mw * n > 512) continue;
      const int iters = 2000;
      mma_rate<<<148, 128, 200 * 1024>>>(n, iters, mw, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long h[2];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      const double per = double(h[1]) / (iters * mw * 4);
      double r[3];
      int ci = 0;
      for (int c : {1, 2, 4}) {
        if (c == 1) mma_rate2<1><<<148, 128, 200 * 1024>>>(n, iters, mw, d);
        if (c == 2) mma_rate2<2><<<148, 128, 200 * 1024>>>(n, iters, mw, d);
        if (c == 4) mma_rate2<4><<<148, 128, 200 * 1024>>>(n, iters, mw, d);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err2 %s\n", cudaGetErrorString(e)); return 1; }
        long long h2[2];
        cudaMemcpy(h2, d, sizeof(h2), cudaMemcpyDeviceToHost);
        r[ci++] = double(h2[1]) / (iters * mw * 4);
      }
      double q[2] = {0, 0};
      mma_order<10><<<148, 128, 200 * 1024>>>(n, iters, mw, d);
      cudaDeviceSynchronize();
      long long h3[2];
      cudaMemcpy(h3, d, sizeof(h3), cudaMemcpyDeviceToHost);
      q[0] = double(h3[1]) / (iters * mw * 4);
      if (2 * mw * n <= 512) {
        mma_order<11><<<148, 128, 200 * 1024>>>(n, iters, mw, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h3, d, sizeof(h3), cudaMemcpyDeviceToHost);
        q[1] = double(h3[1]) / (iters * mw * 4);
      }
      double two = 0;
      if (2 * mw * n <= 512 && 2 * mw <= 8) {
        mma_two_issuers<<<148, 128, 200 * 1024>>>(n, iters, mw, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h3, d, sizeof(h3), cudaMemcpyDeviceToHost);
        two = double(h3[1]) / (iters * mw * 4 * 2);
      }
      printf("mw=%d N=%3d: j-major %.1f | k-major %.1f | 2-acc %.1f | 2 issuers %.1f cyc/mma (floor %.1f)\n", mw, n,
             r[0], q[0], q[1], two, 128.0 * n / 256.0);
    }
  }
  return 0;
}
