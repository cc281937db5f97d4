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
      const float w = __bfloat162float(wr[static_cast<size_t>(e) * d_h + k]);  // W_r^T [M, d_h]
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

// ------------------------------------------------------------------ fast path
// Tensor-core router for M <= 256, M % 8 == 0, K <= 32: grid (T/32 token tiles, d_h/256
// K-splits); each CTA stages a 32 x 256 slice of x and the transposed 256 x M slice of
// W_r in shared memory and issues bf16 mma.sync m16n8k16 (fp32 accumulate): the router
// GEMM is 0.27 GFLOP/layer and purely latency-bound, so it needs many small CTAs, not
// TMEM. Partial logits go to the workspace; the LAST CTA of each token tile (atomic
// ticket) sums the splits in split order (deterministic), adds the bias and runs the
// warp top-K + softmax, then resets its ticket for the next launch.
constexpr int kRtTok = 32, kRtKC = 256, kRtPad = 8;

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(256) route_mma_kernel(const __nv_bfloat16* __restrict__ x,
                                                        const __nv_bfloat16* __restrict__ wr,
                                                        const float* __restrict__ bias, int T, int d_h, int M, int K,
                                                        int nsplit, float* __restrict__ part,
                                                        int32_t* __restrict__ tickets, int32_t* __restrict__ ids,
                                                        float* __restrict__ weights, float* __restrict__ logits_out) {
  extern __shared__ __align__(16) uint8_t rsm[];
  constexpr int LD = kRtKC + kRtPad;  // padded row (bank-conflict-free fragment loads)
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(rsm);        // [32][LD]
  __nv_bfloat16* wt = xs + kRtTok * LD;                             // [M][LD]  (W_r transposed)
  __shared__ int s_last;
  const int t0 = blockIdx.x * kRtTok, split = blockIdx.y, k0 = split * kRtKC;
  const int kn = min(kRtKC, d_h - k0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int CPR = kRtKC / 8;  // 16-B chunks per staged row (d_h % 8 == 0 on this path)
  for (int i = tid; i < kRtTok * CPR; i += blockDim.x) {
    const int t = i / CPR, k = (i % CPR) * 8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (t0 + t < T && k < kn) v = *reinterpret_cast<const uint4*>(x + static_cast<size_t>(t0 + t) * d_h + k0 + k);
    *reinterpret_cast<uint4*>(xs + t * LD + k) = v;
  }
  for (int i = tid; i < M * CPR; i += blockDim.x) {  // W_r^T rows: expert-major, K contiguous
    const int e = i / CPR, k = (i % CPR) * 8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (k < kn) v = *reinterpret_cast<const uint4*>(wr + static_cast<size_t>(e) * d_h + k0 + k);
    *reinterpret_cast<uint4*>(wt + e * LD + k) = v;
  }
  __syncthreads();
  const int g = lane >> 2, tg = lane & 3;
  const int th = warp & 1;                 // token half: rows 16*th .. +16
  const int n_tiles = M / 8;
  float acc[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  const __nv_bfloat16* xa = xs + (16 * th + g) * LD + tg * 2;
  for (int kk = 0; kk < kRtKC; kk += 16) {
    const uint32_t a0 = *reinterpret_cast<const uint32_t*>(xa + kk);
    const uint32_t a1 = *reinterpret_cast<const uint32_t*>(xa + 8 * LD + kk);
    const uint32_t a2 = *reinterpret_cast<const uint32_t*>(xa + kk + 8);
    const uint32_t a3 = *reinterpret_cast<const uint32_t*>(xa + 8 * LD + kk + 8);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int nt = (warp >> 1) + 4 * j;
      if (nt < n_tiles) {
        const __nv_bfloat16* wb = wt + (nt * 8 + g) * LD + tg * 2 + kk;
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(wb);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(wb + 8);
        mma_bf16_16816(acc[j], a0, a1, a2, a3, b0, b1);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int nt = (warp >> 1) + 4 * j;
    if (nt < n_tiles) {
      const int e = nt * 8 + tg * 2;
      const int ta = t0 + 16 * th + g, tb = ta + 8;
      float* pp = part + static_cast<size_t>(split) * T * M;
      if (ta < T) { pp[static_cast<size_t>(ta) * M + e] = acc[j][0]; pp[static_cast<size_t>(ta) * M + e + 1] = acc[j][1]; }
      if (tb < T) { pp[static_cast<size_t>(tb) * M + e] = acc[j][2]; pp[static_cast<size_t>(tb) * M + e + 1] = acc[j][3]; }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&tickets[blockIdx.x], 1) == nsplit - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int tl = warp; tl < kRtTok; tl += blockDim.x / 32) {
    const int t = t0 + tl;
    if (t >= T) break;
    float lg[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int v = lane + 32 * j;
      float s = -CUDART_INF_F;
      if (v < M) {
        s = 0.f;
        for (int q = 0; q < nsplit; ++q) s += __ldcg(part + (static_cast<size_t>(q) * T + t) * M + v);
        if (bias) s += bias[v];
        if (logits_out) logits_out[static_cast<size_t>(t) * M + v] = s;
      }
      lg[j] = s;
    }
    float top = 0.f, den = 0.f, my_w = 0.f;
    int my_id = 0;
    for (int r = 0; r < K; ++r) {
      float bv = -CUDART_INF_F;
      int bi = -1;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int v = lane + 32 * j;
        if (v < M && (bi < 0 || lg[j] > bv)) { bv = lg[j]; bi = v; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
      }
      if (r == 0) top = bv;
      const float ex = expf(bv - top);
      den += ex;
      if (lane == r) { my_id = bi; my_w = ex; }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (lane + 32 * j == bi) lg[j] = -CUDART_INF_F;
    }
    if (lane < K) {
      ids[static_cast<size_t>(t) * K + lane] = my_id;
      weights[static_cast<size_t>(t) * K + lane] = my_w / den;
    }
  }
  if (tid == 0) tickets[blockIdx.x] = 0;
}

size_t route_workspace_bytes(int T, int d_h, int M) {
  const int nsplit = (d_h + kRtKC - 1) / kRtKC;
  const int tiles = (T + kRtTok - 1) / kRtTok;
  return 256 + static_cast<size_t>(tiles) * 4 + static_cast<size_t>(nsplit) * T * M * 4;
}

bool route_fast_path(int M, int K, int d_h) { return M % 8 == 0 && M <= 256 && K <= 32 && d_h % 8 == 0; }

cudaError_t launch_route_mma(const __nv_bfloat16* x, const __nv_bfloat16* w_router, const float* bias, int T,
                             int d_h, int M, int K, int32_t* ids, float* weights, float* logits_out, void* ws,
                             cudaStream_t stream) {
  const int nsplit = (d_h + kRtKC - 1) / kRtKC;
  const int tiles = (T + kRtTok - 1) / kRtTok;
  int32_t* tickets = reinterpret_cast<int32_t*>(ws);
  float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + ((tiles * 4 + 255) / 256) * 256);
  const size_t smem = static_cast<size_t>(kRtTok + M) * (kRtKC + kRtPad) * 2;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(route_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  route_mma_kernel<<<dim3(tiles, nsplit), 256, smem, stream>>>(x, w_router, bias, T, d_h, M, K, nsplit, part,
                                                               tickets, ids, weights, logits_out);
  return cudaGetLastError();
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
// x += y (if y), h = bf16(x * rsqrt(mean(x^2) + eps)); one CTA per token. The traversal
// (4-element chunks per thread, same block size) and the reduction tree are exactly those
// of the combine kernel's fused epilogue (layout.cu), so the unfused expert-parallel step
// reproduces the fused single-GPU step bit for bit.
__global__ void __launch_bounds__(256) residual_rmsnorm_kernel(float* __restrict__ x, const float* __restrict__ y,
                                                               __nv_bfloat16* __restrict__ h, int d_h, float eps) {
  __shared__ float s_red[8];
  const int t = blockIdx.x;
  float ss = 0.f;
  for (int f0 = threadIdx.x * 4; f0 < d_h; f0 += blockDim.x * 4) {
    const size_t o = static_cast<size_t>(t) * d_h + f0;
    for (int q = 0; q < 4 && f0 + q < d_h; ++q) {
      float v = x[o + q];
      if (y) {
        v = v + y[o + q];
        x[o + q] = v;
      }
      ss = fmaf(v, v, ss);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < (blockDim.x + 31) / 32; ++i) tot += s_red[i];
  const float r = rsqrtf(tot / static_cast<float>(d_h) + eps);
  for (int f0 = threadIdx.x * 4; f0 < d_h; f0 += blockDim.x * 4) {
    const size_t o = static_cast<size_t>(t) * d_h + f0;
    for (int q = 0; q < 4 && f0 + q < d_h; ++q) h[o + q] = __float2bfloat16_rn(x[o + q] * r);
  }
}

cudaError_t launch_residual_rmsnorm(float* x, const float* y, __nv_bfloat16* h_out, int T, int d_h, float eps,
                                    cudaStream_t stream) {
  int threads = d_h / 4 >= 256 ? 256 : ((d_h / 4 + 31) / 32) * 32;  // == launch_combine
  if (threads < 32) threads = 32;
  residual_rmsnorm_kernel<<<T, threads, 0, stream>>>(x, y, h_out, d_h, eps);
  return cudaGetLastError();
}

}  // namespace sere
