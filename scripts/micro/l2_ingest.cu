// Microbenchmark: per-SM bulk-copy ingest when the source is L2-resident vs HBM, and the
// cost of cp.async.bulk.prefetch.L2 issue. Question it answers: can the FFN's first k-steps
// run faster than HBM pace if their weights were prefetched into L2?
//   stream(ctas, region): each CTA streams `total` bytes by 32 KB bulk copies into a 6-slot
//   smem ring, cycling over its own `region` bytes (region small => L2 hits).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_07616_b200/csrc/ptx.cuh"
using namespace sere;

__global__ void __launch_bounds__(64, 1) stream(const uint8_t* __restrict__ w, size_t region, size_t total,
                                                int copy_bytes, int slots) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const size_t steps = total / copy_bytes, per_region = region / copy_bytes;
  const uint8_t* base = w + blockIdx.x * region;
  const uint64_t pol = policy_evict_last();
  if (warp == 0 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (size_t i = 0; i < steps; ++i) {
      mbar_wait(&empty[s], ph ^ 1u);
      mbar_arrive_expect_tx(&full[s], copy_bytes);
      bulk_g2s(smem + s * copy_bytes, base + (i % per_region) * copy_bytes, copy_bytes, &full[s], pol);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
  } else if (warp == 1 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (size_t i = 0; i < steps; ++i) {
      mbar_wait(&full[s], ph);
      mbar_arrive(&empty[s]);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
  }
}

__global__ void prefetch_issue(const uint8_t* w, size_t per_cta, uint32_t run, long long* cyc) {
  const long long t0 = clock64();
  const uint8_t* base = w + blockIdx.x * per_cta;
  for (size_t o = threadIdx.x * (size_t)run; o < per_cta; o += (size_t)blockDim.x * run)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"(run) : "memory");
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const int sms = 148;
  uint8_t* w; long long* cyc;
  const size_t big = size_t(8) << 30;
  cudaMalloc(&w, big);
  cudaMemset(w, 1, big);
  cudaMalloc(&cyc, 1024 * sizeof(long long));
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  struct Cfg { int ctas; size_t region; size_t total; int copy; const char* what; };
  Cfg cfgs[] = {
      {148, size_t(48) << 20, size_t(48) << 20, 32768, "HBM (distinct 48 MB per CTA)"},
      {148, size_t(256) << 10, size_t(48) << 20, 32768, "L2 (256 KB per CTA, 37 MB total)"},
      {32, size_t(256) << 10, size_t(48) << 20, 32768, "L2, 32 CTAs"},
      {8, size_t(256) << 10, size_t(32) << 20, 32768, "L2, 8 CTAs"},
      {148, size_t(256) << 10, size_t(48) << 20, 16384, "L2, 16 KB copies"},
  };
  for (const Cfg& c : cfgs) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      stream<<<c.ctas, 64, 6 * c.copy + 1024>>>(w, c.region, c.total, c.copy, 6);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = double(c.total) * c.ctas / (ms * 1e-3) / 1e9;
    printf("%-40s ctas=%3d copy=%5d: %8.1f GB/s total, %6.1f GB/s per SM (%.3f ms)\n", c.what, c.ctas, c.copy, gbs,
           gbs / c.ctas, ms);
  }
  // prefetch issue cost: 128 CTAs x 384 KB (48 MB) in runs of 128 KB / 32 KB / 4 KB
  const uint32_t runs[] = {131072, 32768, 4096};
  for (uint32_t run : runs) {
    for (int threads : {1, 32, 256}) {
      cudaMemset(w + (size_t(1) << 30), 2, size_t(256) << 20);  // evict: touch 256 MB elsewhere
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      prefetch_issue<<<128, threads>>>(w + (size_t(4) << 30), size_t(384) << 10, run, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      long long h[128];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (long long v : h) mx = v > mx ? v : mx;
      // then read the prefetched data back: L2 hits if the prefetch landed
      cudaEventRecord(e0);
      stream<<<128, 64, 6 * 32768 + 1024>>>(w + (size_t(4) << 30), size_t(384) << 10, size_t(384) << 10, 32768, 6);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms2;
      cudaEventElapsedTime(&ms2, e0, e1);
      // and the same read without a prefetch (cold)
      cudaMemset(w + (size_t(1) << 30), 3, size_t(256) << 20);
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      stream<<<128, 64, 6 * 32768 + 1024>>>(w + (size_t(4) << 30), size_t(384) << 10, size_t(384) << 10, 32768, 6);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms3;
      cudaEventElapsedTime(&ms3, e0, e1);
      printf("prefetch 48 MB run=%6u threads=%3d: kernel %.1f us, max issue %lld cyc | read after: %.1f us, cold read %.1f us\n",
             run, threads, ms * 1e3, mx, ms2 * 1e3, ms3 * 1e3);
    }
  }
  return 0;
}
