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
#include "rowops.cuh"

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
// x_pack[kt][row][64] (128-B rows, chunk-swizzled) <- x[row_token[row]][64*kt .. +64].
// One warp per permuted row: the source token is read once, then every lane keeps
// kPermVec independent 16-B loads in flight before storing (a latency-bound gather).
constexpr int kPermVec = 8;

__global__ void __launch_bounds__(256) permute_kernel(const __nv_bfloat16* __restrict__ x, int d_h, int d_h_pad,
                                                      const int32_t* __restrict__ plan,
                                                      const int32_t* __restrict__ row_token, int r_max,
                                                      uint8_t* __restrict__ x_pack) {
  if (plan[P_STATUS] != 0) return;
  const int total_rows = plan[P_TOTAL_ROWS];
  const int cpr = d_h_pad / 8;  // 16-B chunks per row
  const int lane = threadIdx.x & 31;
  const bool vec = (d_h & 7) == 0;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < total_rows; r += (gridDim.x * blockDim.x) >> 5) {
    const int t = row_token[r];
    for (int c0 = 0; c0 < cpr; c0 += 32 * kPermVec) {
      uint4 v[kPermVec];
#pragma unroll
      for (int i = 0; i < kPermVec; ++i) {
        const int ch = c0 + lane + 32 * i;
        const int k0 = ch * 8;
        v[i] = make_uint4(0u, 0u, 0u, 0u);
        if (t >= 0 && ch < cpr && k0 < d_h) {
          const __nv_bfloat16* src = x + static_cast<size_t>(t) * d_h + k0;
          if (vec) {
            v[i] = __ldg(reinterpret_cast<const uint4*>(src));
          } else {
            alignas(16) __nv_bfloat16 tmp[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) tmp[q] = (k0 + q < d_h) ? src[q] : __float2bfloat16(0.f);
            v[i] = *reinterpret_cast<uint4*>(tmp);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kPermVec; ++i) {
        const int ch = c0 + lane + 32 * i;
        if (ch < cpr) {
          const int kt = ch >> 3, c = ch & 7;
          *reinterpret_cast<uint4*>(x_pack + (static_cast<size_t>(kt) * r_max + r) * 128 + sw128_chunk(c, r) * 16) =
              v[i];
        }
      }
    }
  }
}

cudaError_t launch_permute(const __nv_bfloat16* x, const Dims& d, const int32_t* plan, const int32_t* row_token,
                           int r_max, uint8_t* x_pack, int num_sms, cudaStream_t stream) {
  int blocks = (r_max + 7) / 8;  // one warp per row, 8 warps per CTA
  if (blocks > num_sms * 8) blocks = num_sms * 8;
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
// next layer's RMSNorm fused into the same pass over the token row.
// One CTA per token (rowops.cuh traversal); each thread gathers its 8 features of up to
// kCombBatch slots at once so that many loads are in flight.
constexpr int kCombBatch = 4;

__device__ __forceinline__ void load_y8(const float* src, int ksplit, size_t split_stride, float (&v)[8]) {
  float4 a = *reinterpret_cast<const float4*>(src), b = *reinterpret_cast<const float4*>(src + 4);
  for (int s = 1; s < ksplit; ++s) {
    const float4 oa = *reinterpret_cast<const float4*>(src + s * split_stride);
    const float4 ob = *reinterpret_cast<const float4*>(src + s * split_stride + 4);
    a.x = __fadd_rn(a.x, oa.x); a.y = __fadd_rn(a.y, oa.y); a.z = __fadd_rn(a.z, oa.z); a.w = __fadd_rn(a.w, oa.w);
    b.x = __fadd_rn(b.x, ob.x); b.y = __fadd_rn(b.y, ob.y); b.z = __fadd_rn(b.z, ob.z); b.w = __fadd_rn(b.w, ob.w);
  }
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
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
  const int t = blockIdx.x;
  float ss = 0.f;
  for (int f0 = threadIdx.x * kRowVec; f0 < d_h; f0 += blockDim.x * kRowVec) {
    // y_perm rows are d_h_pad (multiple of 128) wide, so the 8-float read never leaves the row
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int k0 = 0; k0 < K + n_shared; k0 += kCombBatch) {
      int row[kCombBatch];
      float wk[kCombBatch];
      float v[kCombBatch][8];
#pragma unroll
      for (int b = 0; b < kCombBatch; ++b) {
        const int k = k0 + b;
        row[b] = -1;
        wk[b] = 1.f;
        if (k < K) {
          row[b] = slot_row[t * K + k];
          wk[b] = w[t * K + k];
        } else if (k < K + n_shared) {
          row[b] = slot_row[TK + t * n_shared + (k - K)];
        }
        if (row[b] >= 0) load_y8(y_perm + static_cast<size_t>(row[b]) * d_h_pad + f0, ksplit, split_stride, v[b]);
      }
#pragma unroll
      for (int b = 0; b < kCombBatch; ++b) {
        if (row[b] < 0) continue;  // padding of the batch, or an expert owned by another rank (EP)
        if (k0 + b < K) {
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(wk[b], v[b][q]));
        } else {  // shared experts: weight 1 (moe.py:308-309)
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], v[b][q]);
        }
      }
    }
    const size_t o = static_cast<size_t>(t) * d_h + f0;
    const bool full = f0 + 8 <= d_h && (d_h & 3) == 0;
    if (y) {
      if (full) {
        *reinterpret_cast<float4*>(y + o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        *reinterpret_cast<float4*>(y + o + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
      } else {
        for (int q = 0; q < 8 && f0 + q < d_h; ++q) y[o + q] = acc[q];
      }
    }
    if (y_bf16)
      for (int q = 0; q < 8 && f0 + q < d_h; ++q) y_bf16[o + q] = __float2bfloat16_rn(acc[q]);
    if (x_res) {
      for (int q = 0; q < 8 && f0 + q < d_h; ++q) {
        const float vv = x_res[o + q] + acc[q];
        x_res[o + q] = vv;
        ss = fmaf(vv, vv, ss);
      }
    }
  }
  if (x_res) {
    const float tot = block_sum(ss, s_red);
    const float r = rsqrtf(tot / static_cast<float>(d_h) + eps);
    for (int f0 = threadIdx.x * kRowVec; f0 < d_h; f0 += blockDim.x * kRowVec) {
      const size_t o = static_cast<size_t>(t) * d_h + f0;
      for (int q = 0; q < 8 && f0 + q < d_h; ++q) h_next[o + q] = __float2bfloat16_rn(x_res[o + q] * r);
    }
  }
}

cudaError_t launch_combine(const float* y_perm, const Dims& d, int r_max, const int32_t* plan,
                           const int32_t* slot_row, const float* w, int T, int K, int n_shared, float* y,
                           __nv_bfloat16* y_bf16, float* x_res, __nv_bfloat16* h_next, float eps,
                           cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  combine_kernel<<<T, row_threads(d.d_h), 0, stream>>>(y_perm, d.ksplit_dn, r_max, d.d_h, d.d_h_pad, plan, slot_row,
                                                        w, T, K, n_shared, y, y_bf16, x_res, h_next, eps);
  return cudaGetLastError();
}

}  // namespace sere
