// layout.cu -- data movement around the grouped FFN:
//   * pack/unpack of expert weights between the reference orientation
//     (ExpertWeights, moe.py:70-77: x @ W, W [d_h,d_m] / [d_m,d_h]) and the
//     tcgen05 tile layout of the bank: K-major 128x64 bf16 tiles,
//     128-B swizzled, each tile one contiguous 16 KB block so a single bulk
//     async copy streams it at full DRAM burst length;
//   * permute: gather token rows into the per-expert grouped, swizzled,
//     K-tiled activation buffer the GEMM's B operand reads (moe.py:303-307's
//     `x[rows]`), zero-filling padding rows;
//   * combine: deterministic fixed-order weighted sum (moe.py:302-309): slot 0..K-1
//     then shared experts, no atomics, fp32 out.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "params.cuh"
#include "plan.cuh"
#include "ptx.cuh"

namespace sere {

// ------------------------------------------------------------------ packing
// A bank tile is 128 output features x 64 input features of a weight W[K][F] kept in
// the reference's x @ W orientation (row-major, ExpertWeights moe.py:70-77): tile
// row r = feature f0 + r, column c = input k0 + c, bf16, 128-B rows with the 16-B
// chunk swizzle of the UMMA SW128 K-major layout. Out-of-range entries are zero.
__device__ __forceinline__ void tile_xfer(const __nv_bfloat16* __restrict__ W, int K, int F, int f0, int k0,
                                          uint8_t* __restrict__ dst, int unpack, __nv_bfloat16 (*sd)[130]) {
  if (!unpack) {
    for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) {
      const int kk = i / 128, ff = i % 128;
      const int k = k0 + kk, f = f0 + ff;
      sd[kk][ff] = (k < K && f < F) ? W[static_cast<size_t>(k) * F + f] : __float2bfloat16(0.f);
    }
    __syncthreads();
    for (int cid = threadIdx.x; cid < 128 * 8; cid += blockDim.x) {
      const int r = cid / 8, c = cid % 8;
      alignas(16) __nv_bfloat16 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = sd[c * 8 + q][r];
      *reinterpret_cast<uint4*>(dst + r * 128 + sw128_chunk(c, r) * 16) = *reinterpret_cast<uint4*>(v);
    }
  } else {
    for (int cid = threadIdx.x; cid < 128 * 8; cid += blockDim.x) {
      const int r = cid / 8, c = cid % 8;
      alignas(16) __nv_bfloat16 v[8];
      *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(dst + r * 128 + sw128_chunk(c, r) * 16);
#pragma unroll
      for (int q = 0; q < 8; ++q) sd[c * 8 + q][r] = v[q];
    }
    __syncthreads();
    __nv_bfloat16* out = const_cast<__nv_bfloat16*>(W);
    for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) {
      const int kk = i / 128, ff = i % 128;
      const int k = k0 + kk, f = f0 + ff;
      if (k < K && f < F) out[static_cast<size_t>(k) * F + f] = sd[kk][ff];
    }
  }
}

// W13 tile (e, fb, kt, s): s = 0 gate / 1 up, features 128*fb.., inputs 64*kt.. of
// w_gate / w_up [d_h, d_m]; the gate and up tiles of one (fb, kt) are adjacent (one
// 32 KB copy feeds both accumulators of the SwiGLU epilogue).
__global__ void __launch_bounds__(256) pack_w13_kernel(const __nv_bfloat16* __restrict__ wg,
                                                       const __nv_bfloat16* __restrict__ wu, int d_h, int d_m,
                                                       int tiles, int ktiles, uint8_t* __restrict__ w13,
                                                       int first, int unpack) {
  __shared__ __nv_bfloat16 sd[64][130];
  const int tile = blockIdx.x;
  const int s = tile & 1;
  const int kt = (tile >> 1) % ktiles;
  const int fb = ((tile >> 1) / ktiles) % tiles;
  const int e = (tile >> 1) / (ktiles * tiles);
  uint8_t* dst = w13 + ((static_cast<size_t>((first + e) * tiles + fb) * ktiles + kt) * 2 + s) * kTileBytes;
  const __nv_bfloat16* W = (s ? wu : wg) + static_cast<size_t>(e) * d_h * d_m;
  tile_xfer(W, d_h, d_m, fb * 128, kt * 64, dst, unpack, sd);
}

// W2 tile (e, mt, kt): output features 128*mt.., inputs 64*kt.. of w_down [d_m, d_h]
__global__ void __launch_bounds__(256) pack_w2_kernel(const __nv_bfloat16* __restrict__ wd, int d_h, int d_m,
                                                      int tiles, int ktiles, uint8_t* __restrict__ w2, int first,
                                                      int unpack) {
  __shared__ __nv_bfloat16 sd[64][130];
  const int tile = blockIdx.x;
  const int kt = tile % ktiles;
  const int mt = (tile / ktiles) % tiles;
  const int e = tile / (ktiles * tiles);
  uint8_t* dst = w2 + (static_cast<size_t>((first + e) * tiles + mt) * ktiles + kt) * kTileBytes;
  tile_xfer(wd + static_cast<size_t>(e) * d_m * d_h, d_m, d_h, mt * 128, kt * 64, dst, unpack, sd);
}

cudaError_t launch_pack(const __nv_bfloat16* wg, const __nv_bfloat16* wu, const __nv_bfloat16* wd, int count,
                        const Dims& d, int Et, int first, uint8_t* bank, int unpack, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  uint8_t* w13 = bank;
  uint8_t* w2 = bank + bank_w13_bytes(Et, d);
  const unsigned g13 = static_cast<unsigned>(count) * d.tiles_gu * d.ktiles_gu * 2;
  const unsigned g2 = static_cast<unsigned>(count) * d.tiles_dn * d.ktiles_dn;
  pack_w13_kernel<<<g13, 256, 0, stream>>>(wg, wu, d.d_h, d.d_m, d.tiles_gu, d.ktiles_gu, w13, first, unpack);
  pack_w2_kernel<<<g2, 256, 0, stream>>>(wd, d.d_h, d.d_m, d.tiles_dn, d.ktiles_dn, w2, first, unpack);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ permute
// x_pack[kt][row][64] (128-B rows, chunk-swizzled) <- x[row_token[row]][64*kt .. +64]
__global__ void __launch_bounds__(256) permute_kernel(const __nv_bfloat16* __restrict__ x, int d_h, int d_h_pad,
                                                      const int32_t* __restrict__ plan,
                                                      const int32_t* __restrict__ row_token, int r_max,
                                                      uint8_t* __restrict__ x_pack) {
  if (plan[P_STATUS] != 0) return;
  const int total_rows = plan[P_TOTAL_ROWS];
  const int cpr = d_h_pad / 8;  // 16-B chunks per row
  const long long n = static_cast<long long>(total_rows) * cpr;
  const bool vec = (d_h & 7) == 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / cpr), ch = static_cast<int>(i % cpr);
    const int t = row_token[r];
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    const int k0 = ch * 8;
    if (t >= 0 && k0 < d_h) {
      const __nv_bfloat16* src = x + static_cast<size_t>(t) * d_h + k0;
      if (vec) {
        v = *reinterpret_cast<const uint4*>(src);
      } else {
        alignas(16) __nv_bfloat16 tmp[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) tmp[q] = (k0 + q < d_h) ? src[q] : __float2bfloat16(0.f);
        v = *reinterpret_cast<uint4*>(tmp);
      }
    }
    const int kt = ch >> 3, c = ch & 7;
    *reinterpret_cast<uint4*>(x_pack + (static_cast<size_t>(kt) * r_max + r) * 128 + sw128_chunk(c, r) * 16) = v;
  }
}

cudaError_t launch_permute(const __nv_bfloat16* x, const Dims& d, const int32_t* plan, const int32_t* row_token,
                           int r_max, uint8_t* x_pack, int num_sms, cudaStream_t stream) {
  const long long work = static_cast<long long>(r_max) * (d.d_h_pad / 8);
  int blocks = static_cast<int>((work + 255) / 256);
  blocks = blocks < num_sms * 8 ? blocks : num_sms * 8;
  if (blocks < 1) blocks = 1;
  permute_kernel<<<blocks, 256, 0, stream>>>(x, d.d_h, d.d_h_pad, plan, row_token, r_max, x_pack);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ combine
// y[t] = sum_k w[t,k] * Y[slot_row[t,k]]  (k ascending)  + sum_s Y[shared row]   (moe.py:302-309)
// Y = sum over down-GEMM K splits in split order. Products and sums rounded
// separately (no FMA contraction), mirroring numpy's `y[rows] += w * E(x)`.
// Optional decode-block epilogue (x_res != null): x_res[t] += y[t], then
// h_next[t] = bf16(x_res[t] * rsqrt(mean(x_res[t]^2) + eps)) -- the residual add and the
// next layer's RMSNorm fused into the same pass over the token row (one CTA per token).
__device__ __forceinline__ float4 load_y_sum(const float* src, int ksplit, size_t split_stride) {
  float4 v = *reinterpret_cast<const float4*>(src);
  for (int s = 1; s < ksplit; ++s) {
    const float4 o = *reinterpret_cast<const float4*>(src + s * split_stride);
    v.x = __fadd_rn(v.x, o.x); v.y = __fadd_rn(v.y, o.y); v.z = __fadd_rn(v.z, o.z); v.w = __fadd_rn(v.w, o.w);
  }
  return v;
}

__global__ void __launch_bounds__(256) combine_kernel(const float* __restrict__ y_perm, int ksplit, int r_max,
                                                      int d_h, int d_h_pad, const int32_t* __restrict__ plan,
                                                      const int32_t* __restrict__ slot_row,
                                                      const float* __restrict__ w, int T, int K, int n_shared,
                                                      float* __restrict__ y, __nv_bfloat16* __restrict__ y_bf16,
                                                      float* __restrict__ x_res, __nv_bfloat16* __restrict__ h_next,
                                                      float eps) {
  __shared__ float s_red[8];
  if (plan[P_STATUS] != 0) return;
  const int TK = T * K;
  const size_t split_stride = static_cast<size_t>(r_max) * d_h_pad;
  const bool vec = (d_h & 3) == 0;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    float ss = 0.f;
    for (int f0 = threadIdx.x * 4; f0 < d_h; f0 += blockDim.x * 4) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int k = 0; k < K; ++k) {
        const int row = slot_row[t * K + k];
        if (row < 0) continue;  // expert owned by another rank (expert parallelism)
        const float wk = w[t * K + k];
        const float4 v = load_y_sum(y_perm + static_cast<size_t>(row) * d_h_pad + f0, ksplit, split_stride);
        acc[0] = __fadd_rn(acc[0], __fmul_rn(wk, v.x));
        acc[1] = __fadd_rn(acc[1], __fmul_rn(wk, v.y));
        acc[2] = __fadd_rn(acc[2], __fmul_rn(wk, v.z));
        acc[3] = __fadd_rn(acc[3], __fmul_rn(wk, v.w));
      }
      for (int s = 0; s < n_shared; ++s) {
        const int row = slot_row[TK + t * n_shared + s];
        const float4 v = load_y_sum(y_perm + static_cast<size_t>(row) * d_h_pad + f0, ksplit, split_stride);
        acc[0] = __fadd_rn(acc[0], v.x);
        acc[1] = __fadd_rn(acc[1], v.y);
        acc[2] = __fadd_rn(acc[2], v.z);
        acc[3] = __fadd_rn(acc[3], v.w);
      }
      const size_t o = static_cast<size_t>(t) * d_h + f0;
      if (y) {
        if (vec) *reinterpret_cast<float4*>(y + o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        else for (int q = 0; q < 4 && f0 + q < d_h; ++q) y[o + q] = acc[q];
      }
      if (y_bf16)
        for (int q = 0; q < 4 && f0 + q < d_h; ++q) y_bf16[o + q] = __float2bfloat16_rn(acc[q]);
      if (x_res) {
        for (int q = 0; q < 4 && f0 + q < d_h; ++q) {
          const float v = x_res[o + q] + acc[q];
          x_res[o + q] = v;
          ss = fmaf(v, v, ss);
        }
      }
    }
    if (x_res) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = ss;
      __syncthreads();
      float tot = 0.f;
      for (int i = 0; i < (blockDim.x + 31) / 32; ++i) tot += s_red[i];
      const float r = rsqrtf(tot / static_cast<float>(d_h) + eps);
      for (int f0 = threadIdx.x * 4; f0 < d_h; f0 += blockDim.x * 4) {
        const size_t o = static_cast<size_t>(t) * d_h + f0;
        for (int q = 0; q < 4 && f0 + q < d_h; ++q) h_next[o + q] = __float2bfloat16_rn(x_res[o + q] * r);
      }
      __syncthreads();
    }
  }
}

cudaError_t launch_combine(const float* y_perm, const Dims& d, int r_max, const int32_t* plan,
                           const int32_t* slot_row, const float* w, int T, int K, int n_shared, float* y,
                           __nv_bfloat16* y_bf16, float* x_res, __nv_bfloat16* h_next, float eps,
                           cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  int threads = d.d_h / 4 >= 256 ? 256 : ((d.d_h / 4 + 31) / 32) * 32;
  if (threads < 32) threads = 32;
  combine_kernel<<<T, threads, 0, stream>>>(y_perm, d.ksplit_dn, r_max, d.d_h, d.d_h_pad, plan, slot_row, w, T, K,
                                            n_shared, y, y_bf16, x_res, h_next, eps);
  return cudaGetLastError();
}

}  // namespace sere
