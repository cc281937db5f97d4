// Cold-code fetch cost: one CTA runs N straight-line FFMAs once (8 independent chains, so
// issue-bound at ~1 instr/cycle when the instructions are resident). Cycles per KB of SASS
// above that floor = the instruction-fetch cost a run-once kernel (re-route/align) pays.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o icache icache.cu && ./icache
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void straight(float* out, long long* cyc, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x[i & 7] = fmaf(x[i & 7], a, b);
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int N>
void run(int threads) {
  float* out; long long* cyc;
  cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 8 * 8);
  long long h[3];
  for (int r = 0; r < 3; ++r) {
    straight<N><<<1, threads>>>(out, cyc, 1.0001f, 0.5f);
    cudaMemcpy(&h[r], cyc, 8, cudaMemcpyDeviceToHost);
  }
  printf("N=%6d (%4d KB SASS) threads=%4d: cycles first %7lld  second %7lld  third %7lld  -> %.0f cyc/KB cold\n", N,
         N * 16 / 1024, threads, h[0], h[1], h[2], (double)h[0] / (N * 16 / 1024.0));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int th : {32, 1024}) {
    run<1024>(th);
    run<4096>(th);
    run<8192>(th);
  }
  return 0;
}
