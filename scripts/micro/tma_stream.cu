// Microbenchmark: per-SM bulk-async-copy (cp.async.bulk) streaming from HBM into a smem
// ring -- the producer side of moe_ffn_kernel without MMAs. One CTA per SM, one
// producer lane; a consumer lane releases slots as soon as they land. Reports the
// aggregate HBM read bandwidth for several ring depths, copy sizes and with an extra
// L2-resident "activation" copy per step.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_07616_b200/csrc/ptx.cuh"
using namespace sere;

__global__ void __launch_bounds__(64, 1) stream(const uint8_t* __restrict__ w, size_t per_cta, int slots,
                                                int copy_bytes, int copies_per_slot, const uint8_t* act,
                                                int act_bytes, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[32], empty[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int slot_bytes = copy_bytes * copies_per_slot + act_bytes;
  const size_t steps = per_cta / (static_cast<size_t>(copy_bytes) * copies_per_slot);
  const uint8_t* base = w + blockIdx.x * per_cta;
  const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (size_t i = 0; i < steps; ++i) {
      mbar_wait(&empty[s], ph ^ 1u);
      uint8_t* dst = smem + s * slot_bytes;
      mbar_arrive_expect_tx(&full[s], copy_bytes * copies_per_slot + act_bytes);
      if (act_bytes) bulk_g2s(dst + copy_bytes * copies_per_slot, act + (i % 64) * act_bytes, act_bytes, &full[s], pol_x);
      for (int c = 0; c < copies_per_slot; ++c)
        bulk_g2s(dst + c * copy_bytes, base + (i * copies_per_slot + c) * copy_bytes, copy_bytes, &full[s], pol_w);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
  } else if (warp == 1 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (size_t i = 0; i < steps; ++i) {
      mbar_wait(&full[s], ph);
      mbar_arrive(&empty[s]);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  const int sms = 148;
  const size_t per_cta = size_t(64) << 20;  // 64 MB per CTA -> 9.5 GB total
  uint8_t* w; uint8_t* act; long long* d;
  cudaMalloc(&w, per_cta * sms);
  cudaMalloc(&act, 64 << 20);
  cudaMemset(w, 1, per_cta * sms);
  cudaMemset(act, 1, 64 << 20);
  cudaMalloc(&d, sms * sizeof(long long));
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int slots, copy, cps, act; };
  Cfg cfgs[] = {{4, 16384, 1, 0},  {6, 16384, 1, 0},  {8, 16384, 1, 0},  {12, 16384, 1, 0}, {13, 16384, 1, 0},
                {6, 32768, 1, 0},  {6, 16384, 2, 0},  {3, 16384, 4, 0},  {2, 16384, 4, 0},
                {6, 16384, 1, 12288}, {6, 16384, 1, 16384}, {4, 16384, 2, 16384}, {3, 16384, 4, 16384},
                {2, 16384, 4, 16384}, {12, 16384, 1, 2048}};
  for (const Cfg& c : cfgs) {
    const int smem = c.slots * (c.copy * c.cps + c.act) + 1024;
    if (smem > 220 * 1024) continue;
    const size_t per = per_cta / (c.copy * c.cps) * (c.copy * c.cps) / 4;  // 16 MB per CTA per run
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      stream<<<sms, 64, smem>>>(w, per, c.slots, c.copy, c.cps, act, c.act, d);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1)
        printf("slots %2d x (%d x %5d B + act %5d B) = %3d KB weights in flight: %.0f GB/s HBM\n", c.slots, c.cps,
               c.copy, c.act, c.slots * c.copy * c.cps / 1024, per * sms / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
