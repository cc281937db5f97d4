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

// W2 tile (e, mt, kt): output features 128*mt.., inputs 64*kt.. of w_down [d_m, d_h]; placed by
// w2_tile_offset (m-tile pairs adjacent per k-tile)
__global__ void __launch_bounds__(256) pack_w2_kernel(const __nv_bfloat16* __restrict__ wd, int d_h, int d_m,
                                                      int tiles, int ktiles, uint8_t* __restrict__ w2, int first,
                                                      int unpack) {
  __shared__ __nv_bfloat16 sd[64][130];
  const int tile = blockIdx.x;
  const int kt = tile % ktiles;
  const int mt = (tile / ktiles) % tiles;
  const int e = tile / (ktiles * tiles);
  uint8_t* dst = w2 + w2_tile_offset(first + e, mt, kt, tiles, ktiles);
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
// The permutation and the gather of one layer (moe.py:303-307's per-expert `x[rows]`):
// CTA (tb, j) owns token block tb (32 tokens) and the j-th 512-B slice of every row.
//  1. the block's cells are ranked: the cells of bank expert e get consecutive rows
//     erow0[e] + blk_prefix[tb][e] + (cells of e earlier in the block, by slot then token) --
//     the group order (token block, slot, token) the align kernel's prefixes describe. All
//     slots at once: lane masks per (slot, expert) by shared-memory atomicOr, a prefix over
//     slots of their popcounts, then rank = prefix + popc(mask & lanes below);
//  2. slice j == 0 writes slot_row[t,k] (combine) and its inverse row_token;
//  3. every warp copies its tokens' slice once from x and stores it into each of the
//     token's rows of x_pack[kt][row][128 B] (SW128 chunk swizzle), so a token row is read
//     once per slice instead of once per slot.
// Padding rows are not written: their FFN columns never reach an output.
// (128 threads capped at 46 registers, so that the PDL-launched FFN could co-reside, measured
// 1.7% slower on the C4 step: the permute's own gather loses more than the FFN gains)
constexpr int kPermThreads = 256;
constexpr int kPermMaxSlots = 64;       // K + n_shared (K <= 32, n_shared <= 31)
constexpr int kPermTokPerWarp = kTokBlkPerm / (kPermThreads / 32);

__host__ __device__ inline size_t permute_smem_bytes(int K, int n_shared, int m_loc) {
  // rows [K + n_shared][32] int32, lane masks u32 + slot prefixes u16 [K][m_loc], then the
  // block's first row per expert int32 [m_loc + n_shared]
  return static_cast<size_t>(K + n_shared) * kTokBlkPerm * 4 + static_cast<size_t>(K) * m_loc * 4 +
         static_cast<size_t>(round_up(K * m_loc, 2)) * 2 + static_cast<size_t>(m_loc + n_shared) * 4;
}

__global__ void __launch_bounds__(kPermThreads) permute_kernel(
    const __nv_bfloat16* __restrict__ x, int d_h, int d_h_pad, const int32_t* __restrict__ plan, int Et, int m_loc,
    int e_lo, const int32_t* __restrict__ ids_final, const uint16_t* __restrict__ blk_prefix, int T, int K,
    int n_shared, int32_t* __restrict__ slot_row, int32_t* __restrict__ row_token, int r_max,
    uint8_t* __restrict__ x_pack, const float* __restrict__ y_dead, long long y_lines, int x_early) {
  extern __shared__ __align__(16) uint8_t perm_smem[];
  int (*s_row)[kTokBlkPerm] = reinterpret_cast<int (*)[kTokBlkPerm]>(perm_smem);  // [K + n_shared][32]
  uint32_t* s_bm = reinterpret_cast<uint32_t*>(perm_smem) + (K + n_shared) * kTokBlkPerm;  // [K][m_loc] lanes
  uint16_t* s_pre = reinterpret_cast<uint16_t*>(s_bm + K * m_loc);    // [K][m_loc] cells at earlier slots
  int* s_base = reinterpret_cast<int*>(s_pre + round_up(K * m_loc, 2));  // [m_loc + n_shared] block's first rows
  for (int i = threadIdx.x; i < K * m_loc; i += blockDim.x) s_bm[i] = 0u;
  const int tb = blockIdx.x, j = blockIdx.y;
  const int t0 = tb * kTokBlkPerm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA's slice of its tokens' rows: x does not depend on the predecessor (it was final
  // before the re-route/align kernel started), so single-GPU the loads are in flight before
  // the PDL wait; expert parallel, peers' rows are ordered by the barrier inside align
  const int cpr = d_h_pad / 8;  // 16-B pieces per row
  const int q = j * 32 + lane;
  uint4 v[kPermTokPerWarp];
  auto load_rows = [&]() {
    const bool vec = (d_h & 7) == 0;
#pragma unroll
    for (int i = 0; i < kPermTokPerWarp; ++i) {
      const int l = warp * kPermTokPerWarp + i, t = t0 + l;
      const int k0 = q * 8;
      v[i] = make_uint4(0u, 0u, 0u, 0u);
      if (q < cpr && t < T && k0 < d_h) {
        const __nv_bfloat16* src = x + static_cast<size_t>(t) * d_h + k0;
        if (vec) {
          v[i] = __ldg(reinterpret_cast<const uint4*>(src));
        } else {
          alignas(16) __nv_bfloat16 tmp[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) tmp[e] = (k0 + e < d_h) ? src[e] : __float2bfloat16(0.f);
          v[i] = *reinterpret_cast<uint4*>(tmp);
        }
      }
    }
  };
  if (x_early) load_rows();
  if (y_dead != nullptr) {
    // before the PDL wait (the CTAs are resident while re-route/align runs): the previous
    // layer's expert outputs were consumed by its combine, so their dirty lines leave L2
    // without a DRAM write-back that would compete with this layer's weight stream
    // Rows past the previous layer's total were never written: the plan's total (rewritten by
    // re-route/align concurrently, so only a hint: old or new, both bound the live rows
    // closely) limits the sweep to [0, rows) of every K-split plane of y_perm.
    const int rows = min(r_max, max(0, *reinterpret_cast<const volatile int32_t*>(plan + P_TOTAL_ROWS)));
    const long long lpr = d_h_pad / 32, per_split = static_cast<long long>(rows) * lpr;
    const long long n = per_split * (y_lines / (static_cast<long long>(r_max) * lpr));
    const long long nthr = static_cast<long long>(gridDim.x) * gridDim.y * blockDim.x;
    for (long long i = (static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
         i < n; i += nthr) {
      const long long s = i / per_split, j = i - s * per_split;
      l2_discard128(y_dead + (s * r_max * lpr + j) * 32);
    }
  }
  pdl_wait();
  pdl_trigger();
  if (plan[P_STATUS] != 0) return;
  if (!x_early) load_rows();
  const int nslot = K + n_shared;
  const int32_t* erow0 = plan + plan_offsets(Et).erow0;
  const int t_lane = t0 + lane;
  __syncthreads();
  // the block's first row of every local expert (group start + rows of earlier token blocks),
  // loaded in the same round trip as the ids
  for (int i = threadIdx.x; i < m_loc + n_shared; i += blockDim.x)
    s_base[i] = __ldg(erow0 + i) + (i < m_loc ? static_cast<int>(__ldg(blk_prefix + static_cast<size_t>(tb) * Et + i)) : 0);
  for (int k = warp; k < K; k += kPermThreads / 32) {  // warp = slot, lane = token
    const int e = t_lane < T ? __ldg(ids_final + static_cast<size_t>(t_lane) * K + k) : -1;
    const int el = (e >= e_lo && e < e_lo + m_loc) ? e - e_lo : -1;  // -1: another rank's expert (EP)
    s_row[k][lane] = el;
    if (el >= 0) atomicOr(s_bm + k * m_loc + el, 1u << lane);
  }
  __syncthreads();
  for (int el = threadIdx.x; el < m_loc; el += blockDim.x) {
    int run = 0;
    for (int k = 0; k < K; ++k) {
      s_pre[k * m_loc + el] = static_cast<uint16_t>(run);
      run += __popc(s_bm[k * m_loc + el]);
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int k = warp; k < K; k += kPermThreads / 32) {
    const int el = s_row[k][lane];
    s_row[k][lane] = el < 0 ? -1 : s_base[el] + s_pre[k * m_loc + el] + __popc(s_bm[k * m_loc + el] & lt);
  }
  for (int s2 = warp; s2 < n_shared; s2 += kPermThreads / 32)  // shared experts: every token, in token order
    s_row[K + s2][lane] = t_lane < T ? s_base[m_loc + s2] + t_lane : -1;
  __syncthreads();
  if (j == 0) {
    for (int i = threadIdx.x; i < kTokBlkPerm * nslot; i += blockDim.x) {
      const int slot = i / kTokBlkPerm, l = i - slot * kTokBlkPerm;
      const int t = t0 + l;
      if (t >= T) continue;
      const int r = s_row[slot][l];
      slot_row[slot < K ? static_cast<size_t>(t) * K + slot : static_cast<size_t>(T) * K + t * n_shared + (slot - K)] = r;
      if (r >= 0) row_token[r] = t;
    }
  }
  // gather: lane owns 16-B piece q of the slice; tokens loaded first (all in flight), then stored
  if (q >= cpr) return;
  const int kt = q >> 3, c = q & 7;
  uint8_t* dst_kt = x_pack + static_cast<size_t>(kt) * r_max * 128;
#pragma unroll
  for (int i = 0; i < kPermTokPerWarp; ++i) {
    const int l = warp * kPermTokPerWarp + i;
    if (t0 + l >= T) continue;
    for (int slot = 0; slot < nslot; ++slot) {
      const int r = s_row[slot][l];
      if (r >= 0) *reinterpret_cast<uint4*>(dst_kt + static_cast<size_t>(r) * 128 + sw128_chunk(c, r) * 16) = v[i];
    }
  }
}

cudaError_t launch_permute(const __nv_bfloat16* x, const Dims& d, const int32_t* plan, int Et, int m_loc, int e_lo,
                           const int32_t* ids_final, const uint16_t* blk_prefix, int T, int K, int n_shared,
                           int32_t* slot_row, int32_t* row_token, int r_max, uint8_t* x_pack, cudaStream_t stream,
                           const float* y_dead, long long y_lines, bool x_early) {
  if (T <= 0) return cudaSuccess;
  if (K + n_shared > kPermMaxSlots) return cudaErrorInvalidValue;
  const size_t smem = permute_smem_bytes(K, n_shared, m_loc);
  static SmemAttrCache attr;
  if (cudaError_t e = ensure_smem_attr(permute_kernel, smem, attr, 32 * 1024); e != cudaSuccess) return e;
  const dim3 grid((T + kTokBlkPerm - 1) / kTokBlkPerm, (d.d_h_pad / 8 + 31) / 32);
  return launch_pdl((g_pdl & PDL_PERMUTE) != 0, permute_kernel, grid, dim3(kPermThreads), smem, stream, x, d.d_h, d.d_h_pad, plan, Et,
                    m_loc, e_lo, ids_final, blk_prefix, T, K, n_shared, slot_row, row_token, r_max, x_pack,
                    (g_l2 & L2_DISCARD_Y) ? y_dead : nullptr, y_lines, x_early ? 1 : 0);
}

// ------------------------------------------------------------------ combine
// y[t] = sum_k w[t,k] * Y[slot_row[t,k]]  (k ascending)  + sum_s Y[shared row]   (moe.py:302-309)
// Y = sum over down-GEMM K splits in split order. Products and sums rounded
// separately (no FMA contraction), mirroring numpy's `y[rows] += w * E(x)`.
// Optional decode-block epilogue (x_res != null): x_res[t] += y[t], then
// h_next[t] = bf16(x_res[t] * rsqrt(mean(x_res[t]^2) + eps)) -- the residual add and the
// next layer's RMSNorm fused into the same pass over the token row.
// One CTA per token (rowops.cuh traversal); the token's slot rows and weights are staged
// in shared memory once, then each thread gathers its 8 features of kCombBatch slots at
// a time (16 independent 16-B loads in flight).
// residual row fetched into shared memory by cp.async at the start of the pass (no
// registers held while the slot gathers are in flight): combine 10.7 -> 9.4 us per C4 layer
#ifndef SERE_COMB_BATCH
#define SERE_COMB_BATCH 4
#endif
constexpr int kCombBatch = SERE_COMB_BATCH;  // slots whose rows are in flight at once per thread

__device__ __forceinline__ float4 load_y4(const float* src, int ksplit, size_t split_stride) {
  float4 a = __ldcg(reinterpret_cast<const float4*>(src));
  for (int s = 1; s < ksplit; ++s) {
    const float4 o = __ldcg(reinterpret_cast<const float4*>(src + s * split_stride));
    a.x = __fadd_rn(a.x, o.x); a.y = __fadd_rn(a.y, o.y); a.z = __fadd_rn(a.z, o.z); a.w = __fadd_rn(a.w, o.w);
  }
  return a;
}

// Expert-parallel form (ep.world > 0, ep_p2p.cu): CTA t combines this rank's token
// t0 + t; each slot's expert output row is read from its owner rank's y_perm over NVLink
// peer memory (the owner's slot_row says which row), in the same slot order and with the
// same arithmetic as the single-GPU pass, and h_next is stored into every rank's gathered
// token-state buffer -- the reduce-scatter and the next layer's all-gather of h are this
// kernel's loads and stores.
__device__ __forceinline__ int ep_owner(const EpPeers& ep, int e) {
  int o = 0;
  while (o + 1 < ep.world && e >= ep.e_lo[o + 1]) ++o;
  return o;
}



__global__ void __launch_bounds__(kRowMaxThreads) combine_kernel(const float* __restrict__ y_perm, int ksplit, int r_max,
                                                      int d_h, int d_h_pad, const int32_t* __restrict__ plan,
                                                      const int32_t* __restrict__ slot_row,
                                                      const float* __restrict__ w, int T, int K, int n_shared,
                                                      float* __restrict__ y, __nv_bfloat16* __restrict__ y_bf16,
                                                      float* __restrict__ x_res, __nv_bfloat16* __restrict__ h_next,
                                                      float eps, const EpPeers ep, const int32_t* __restrict__ ids_rr) {
  __shared__ float s_red[16];
  __shared__ __align__(16) float s_xr[kRowMaxThreads * kRowVec];  // this token's residual row (d_h <= 4096)
  __shared__ const float* s_src[64];  // slot's expert-output row (nullptr: not evaluated / not owned)
  __shared__ size_t s_split[64];      // its K-split plane stride
  __shared__ float s_w[64];
  // slot rows / weights / the plan come from kernels that completed before the FFN started;
  // y_perm (FFN) and x_res (RMW) need the predecessor grid: wait after staging the slots
  if (plan[P_STATUS] != 0) { pdl_wait(); return; }
  const int t = blockIdx.x;
  const int nslot = K + n_shared;  // <= 32 + 31 (EP: n_shared = all shared experts of the layer)
  if (ep.world == 0) {
    const int TK = T * K;
    const size_t split_stride = static_cast<size_t>(r_max) * d_h_pad;
    for (int k = threadIdx.x; k < nslot; k += blockDim.x) {
      const int row = k < K ? slot_row[t * K + k] : slot_row[TK + t * n_shared + (k - K)];
      s_src[k] = row >= 0 ? y_perm + static_cast<size_t>(row) * d_h_pad : nullptr;
      s_split[k] = split_stride;
      s_w[k] = k < K ? w[t * K + k] : 1.f;
    }
  } else {
    pdl_wait();  // peers' slot rows are ordered by the barrier kernel before us: wait for it
    if (ep.epoch != nullptr) {  // fused barrier: every rank's expert outputs are final
      __shared__ int s_ok;
      if (threadIdx.x == 0) {
        EpSync sy = ep_sync_dev(ep);
        if (blockIdx.x != 0) sy.wait_ns = nullptr;  // CTA 0 stands for the pass
        s_ok = ep_wait(sy);
      }
      __syncthreads();
      if (!s_ok) return;
    }
    if (ep_aborted(ep)) return;  // a barrier timed out: no peer loads or stores on this step
    const int tg = ep.t0 + t, TK = ep.T_all * K;
    for (int k = threadIdx.x; k < nslot; k += blockDim.x) {
      int o, idx;
      if (k < K) {
        o = ep_owner(ep, ids_rr[tg * K + k]);
        idx = tg * K + k;
      } else {
        const int s = k - K;
        o = s % ep.world;
        idx = TK + tg * ep.nsh[o] + s / ep.world;
      }
      const int row = ep.slot_row[o][idx];  // peer load (NVLink) unless o == rank
      s_src[k] = row >= 0 ? ep.y_perm[o] + static_cast<size_t>(row) * d_h_pad : nullptr;
      s_split[k] = static_cast<size_t>(ep.r_max[o]) * d_h_pad;
      s_w[k] = k < K ? w[tg * K + k] : 1.f;
    }
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  // the residual row goes to shared memory with cp.async now (no registers held), so its
  // latency overlaps the slot gathers instead of following them
  const bool xr_async = x_res != nullptr && (d_h & 3) == 0 && d_h <= kRowMaxThreads * kRowVec;
  if (xr_async) {
    for (int f = threadIdx.x * 4; f < d_h; f += blockDim.x * 4)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s_xr + f)),
                   "l"(x_res + static_cast<size_t>(t) * d_h + f)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const bool vec4 = (d_h & 3) == 0;
  float ss = 0.f;
  for (int base = 0; base < d_h; base += blockDim.x * kRowVec) {
    // y_perm rows are d_h_pad (multiple of 128) wide, so the 4-float reads never leave the row
    float acc[kRowChunks][4] = {};
    for (int k0 = 0; k0 < nslot; k0 += kCombBatch) {
      float4 v[kCombBatch][kRowChunks];
#pragma unroll
      for (int b = 0; b < kCombBatch; ++b) {
        const int k = k0 + b;
        const float* src = k < nslot ? s_src[k] : nullptr;
#pragma unroll
        for (int c = 0; c < kRowChunks; ++c) {
          const int f = row_chunk(base, c);
          v[b][c] = (src != nullptr && f < d_h_pad) ? load_y4(src + f, ksplit, s_split[k])
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int b = 0; b < kCombBatch; ++b) {
        const int k = k0 + b;
        if (k >= nslot || s_src[k] == nullptr) continue;  // batch padding, or an expert owned by another rank (EP)
#pragma unroll
        for (int c = 0; c < kRowChunks; ++c) {
          float* a = acc[c];
          if (k < K) {  // routed slot: products and sums rounded separately, slot order (moe.py:302-307)
            const float wk = s_w[k];
            a[0] = __fadd_rn(a[0], __fmul_rn(wk, v[b][c].x));
            a[1] = __fadd_rn(a[1], __fmul_rn(wk, v[b][c].y));
            a[2] = __fadd_rn(a[2], __fmul_rn(wk, v[b][c].z));
            a[3] = __fadd_rn(a[3], __fmul_rn(wk, v[b][c].w));
          } else {  // shared experts: weight 1 (moe.py:308-309)
            a[0] = __fadd_rn(a[0], v[b][c].x);
            a[1] = __fadd_rn(a[1], v[b][c].y);
            a[2] = __fadd_rn(a[2], v[b][c].z);
            a[3] = __fadd_rn(a[3], v[b][c].w);
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kRowChunks; ++c) {
      const int f0 = row_chunk(base, c);
      if (f0 >= d_h) continue;
      const size_t o = static_cast<size_t>(t) * d_h + f0;
      const bool full = vec4 && f0 + 4 <= d_h;
      if (y) {
        if (full) *reinterpret_cast<float4*>(y + o) = make_float4(acc[c][0], acc[c][1], acc[c][2], acc[c][3]);
        else for (int q = 0; q < 4 && f0 + q < d_h; ++q) y[o + q] = acc[c][q];
      }
      if (y_bf16) {
        if (full) store_bf16x4(y_bf16 + o, acc[c]);
        else for (int q = 0; q < 4 && f0 + q < d_h; ++q) y_bf16[o + q] = __float2bfloat16_rn(acc[c][q]);
      }
      if (x_res) {
        if (xr_async) asm volatile("cp.async.wait_group 0;" ::: "memory");  // own copies only: same thread
        for (int q = 0; q < 4 && f0 + q < d_h; ++q) {
          const float vv = (xr_async ? s_xr[f0 + q] : x_res[o + q]) + acc[c][q];
          x_res[o + q] = vv;
          acc[c][q] = vv;
          ss = fmaf(vv, vv, ss);
        }
      }
    }
    if (x_res && (h_next || ep.world) && base + static_cast<int>(blockDim.x) * kRowVec >= d_h) {
      // single-block rows (d_h <= 8 * nthreads, the common case): normalise from registers.
      // Destinations: h_next row t, or (EP) row t0 + t of every rank's gathered states
      const float tot = block_sum(ss, s_red);
      const float r = rsqrtf(tot / static_cast<float>(d_h) + eps);
      const int ndst = ep.world ? ep.world : 1;
      if (base == 0) {
#pragma unroll
        for (int c = 0; c < kRowChunks; ++c) {
          const int f0 = row_chunk(base, c);
          if (f0 >= d_h) continue;
          float hv[4] = {acc[c][0] * r, acc[c][1] * r, acc[c][2] * r, acc[c][3] * r};
          for (int p = 0; p < ndst; ++p) {
            __nv_bfloat16* hd = (ep.world ? ep.h_all[p] + static_cast<size_t>(ep.t0 + t) * d_h
                                          : h_next + static_cast<size_t>(t) * d_h) + f0;
            if (vec4 && f0 + 4 <= d_h) store_bf16x4(hd, hv);
            else for (int q = 0; q < 4 && f0 + q < d_h; ++q) hd[q] = __float2bfloat16_rn(hv[q]);
          }
        }
        if (ep.world) __threadfence_system();  // peer stores visible before the next barrier
        return;
      }
      for (int b2 = 0; b2 < d_h; b2 += blockDim.x * kRowVec)
        for (int c = 0; c < kRowChunks; ++c) {
          const int f0 = row_chunk(b2, c);
          for (int q = 0; q < 4 && f0 + q < d_h; ++q) {
            const float hv = x_res[static_cast<size_t>(t) * d_h + f0 + q] * r;
            for (int p = 0; p < ndst; ++p)
              (ep.world ? ep.h_all[p] + static_cast<size_t>(ep.t0 + t) * d_h
                        : h_next + static_cast<size_t>(t) * d_h)[f0 + q] = __float2bfloat16_rn(hv);
          }
        }
      if (ep.world) __threadfence_system();
      return;
    }
  }
}

cudaError_t launch_combine(const float* y_perm, const Dims& d, int r_max, const int32_t* plan,
                           const int32_t* slot_row, const float* w, int T, int K, int n_shared, float* y,
                           __nv_bfloat16* y_bf16, float* x_res, __nv_bfloat16* h_next, float eps,
                           cudaStream_t stream, const EpPeers* ep, const int32_t* ids_rr) {
  if (T <= 0) return cudaSuccess;
  EpPeers none{};
  return launch_pdl((g_pdl & PDL_COMBINE) != 0, combine_kernel, dim3(T), dim3(row_threads(d.d_h)), 0, stream, y_perm, d.ksplit_dn, r_max,
                    d.d_h, d.d_h_pad, plan, slot_row, w, T, K, n_shared, y, y_bf16, x_res, h_next, eps,
                    ep ? *ep : none, ids_rr);
}

}  // namespace sere
