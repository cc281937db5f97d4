// router.cu -- router GEMM + top-K softmax (moe.py:248-277, `route_topk`).
//
// logits[t,e] = sum_k x[t,k] * W_r[k,e] in fp32 with a fixed reduction order,
// then per token the K largest logits (descending, ties to the LOWER index, the
// stable argsort of moe.py:260) and a softmax over exactly those K (moe.py:261-264).
// One CTA handles kTok tokens; its M*KS threads split d_h into KS contiguous
// chunks (so every W_r row is read coalesced across experts), partial sums meet
// in shared memory in a fixed order, and one warp per token selects the top K.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "params.cuh"

namespace sere {

constexpr int kTok = 4;

__global__ void __launch_bounds__(1024) route_topk_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ wr,
                                                          const float* __restrict__ bias, int T, int d_h,
                                                          int M, int K, int KS, int32_t* __restrict__ ids,
                                                          float* __restrict__ weights, float* __restrict__ logits_out) {
  extern __shared__ float sm[];
  float* s_part = sm;                          // [KS][kTok][M]
  float* s_logit = s_part + KS * kTok * M;     // [kTok][M]
  __nv_bfloat16* s_x = reinterpret_cast<__nv_bfloat16*>(s_logit + kTok * M);  // [kTok][d_h]
  const int t0 = blockIdx.x * kTok;
  const int nt = min(kTok, T - t0);
  for (int i = threadIdx.x; i < kTok * d_h; i += blockDim.x) {
    const int j = i / d_h, k = i % d_h;
    s_x[i] = j < nt ? x[static_cast<size_t>(t0 + j) * d_h + k] : __float2bfloat16(0.f);
  }
  __syncthreads();
  const int e = threadIdx.x % M, ks = threadIdx.x / M;
  if (ks < KS) {
    const int chunk = (d_h + KS - 1) / KS;
    const int k0 = ks * chunk, k1 = min(d_h, k0 + chunk);
    float acc[kTok];
#pragma unroll
    for (int j = 0; j < kTok; ++j) acc[j] = 0.f;
    for (int k = k0; k < k1; ++k) {
      const float w = __bfloat162float(wr[static_cast<size_t>(k) * M + e]);
#pragma unroll
      for (int j = 0; j < kTok; ++j) acc[j] = fmaf(__bfloat162float(s_x[j * d_h + k]), w, acc[j]);
    }
#pragma unroll
    for (int j = 0; j < kTok; ++j) s_part[(ks * kTok + j) * M + e] = acc[j];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kTok * M; i += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < KS; ++q) s += s_part[q * kTok * M + i];
    if (bias) s += bias[i % M];
    s_logit[i] = s;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < nt) {
    const int t = t0 + warp;
    float* lg = s_logit + warp * M;
    if (logits_out)
      for (int v = lane; v < M; v += 32) logits_out[static_cast<size_t>(t) * M + v] = lg[v];
    float sel_val[32];
    float top = 0.f;
    for (int r = 0; r < K; ++r) {
      float bv = -CUDART_INF_F;
      int bi = -1;
      for (int v = lane; v < M; v += 32) {
        const float l = lg[v];
        if (bi < 0 || l > bv) { bv = l; bi = v; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
      }
      if (r == 0) top = bv;
      sel_val[r] = bv;
      if (lane == 0) ids[static_cast<size_t>(t) * K + r] = bi;
      __syncwarp();
      if (lane == (bi & 31)) lg[bi] = -CUDART_INF_F;  // remove the pick (ties resolved on index above)
      __syncwarp();
    }
    if (lane == 0) {
      float den = 0.f;
      for (int r = 0; r < K; ++r) { sel_val[r] = expf(sel_val[r] - top); den += sel_val[r]; }
      for (int r = 0; r < K; ++r) weights[static_cast<size_t>(t) * K + r] = sel_val[r] / den;
    }
  }
}

cudaError_t launch_route_topk(const __nv_bfloat16* x, const __nv_bfloat16* w_router, const float* bias, int T,
                              int d_h, int M, int K, int32_t* ids, float* weights, float* logits_out,
                              cudaStream_t stream) {
  int KS = 1024 / M;
  if (KS < 1) KS = 1;
  if (KS > 64) KS = 64;
  int threads = ((M * KS + 31) / 32) * 32;
  if (threads < 32 * kTok) threads = 32 * kTok;
  if (threads > 1024) threads = 1024;
  const size_t smem = static_cast<size_t>(KS) * kTok * M * 4 + static_cast<size_t>(kTok) * M * 4 +
                      static_cast<size_t>(kTok) * d_h * 2;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(route_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int blocks = (T + kTok - 1) / kTok;
  route_topk_kernel<<<blocks, threads, smem, stream>>>(x, w_router, bias, T, d_h, M, K, KS, ids, weights,
                                                        logits_out);
  return cudaGetLastError();
}

// ------------------------------------------------------------ residual + RMSNorm
// x += y (if y), h = bf16(x * rsqrt(mean(x^2) + eps)); one CTA per token, fixed-order tree reduction
__global__ void __launch_bounds__(256) residual_rmsnorm_kernel(float* __restrict__ x, const float* __restrict__ y,
                                                               __nv_bfloat16* __restrict__ h, int d_h, float eps) {
  __shared__ float s_red[8];
  const int t = blockIdx.x;
  float* xr = x + static_cast<size_t>(t) * d_h;
  const float* yr = y ? y + static_cast<size_t>(t) * d_h : nullptr;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d_h; i += blockDim.x) {
    float v = xr[i];
    if (yr) { v += yr[i]; xr[i] = v; }
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < (blockDim.x + 31) / 32; ++w) tot += s_red[w];
  const float r = rsqrtf(tot / static_cast<float>(d_h) + eps);
  for (int i = threadIdx.x; i < d_h; i += blockDim.x)
    h[static_cast<size_t>(t) * d_h + i] = __float2bfloat16_rn(xr[i] * r);
}

cudaError_t launch_residual_rmsnorm(float* x, const float* y, __nv_bfloat16* h_out, int T, int d_h, float eps,
                                    cudaStream_t stream) {
  residual_rmsnorm_kernel<<<T, 256, 0, stream>>>(x, y, h_out, d_h, eps);
  return cudaGetLastError();
}

}  // namespace sere
