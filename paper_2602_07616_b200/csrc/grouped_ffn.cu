// grouped_ffn.cu -- the expert SwiGLU FFN of one MoE layer as ONE persistent kernel on
// the 5th-gen tensor cores (tcgen05), gate/up and down phases fused.
//
// Decode-time MoE is expert-weight streaming: each active expert's weights are read
// once per layer while only 8..256 tokens use them, so the kernel is built to keep
// HBM busy, not the tensor pipe:
//  * swap-AB: A = a 128-row weight tile (MMA M = 128 output features), B = the
//    group's token rows (MMA N = 16..256), D = fp32 accumulator in TMEM;
//  * weights live in the bank as contiguous 16 KB pre-swizzled tiles, so one bulk
//    async copy (TMA engine, cp.async.bulk) per k-step streams 16 KB at full DRAM
//    burst length with an evict-first L2 policy; activations come from the grouped
//    swizzled buffers (L2-resident, evict-last);
//  * persistent CTAs (one per SM) take work units from a global ticket counter:
//    first every gate/up unit (expert group, 64-feature m-tile, column block), then
//    every down unit (group, 128-feature m-tile, k-split, column block), groups in
//    the plan's schedule order (padded rows descending = longest-processing-time
//    first, since a unit's cost grows with its column count). A down unit waits,
//    before its first copy, until every gate/up unit of its group has published h
//    (per-group counters in the plan, release/acquire + async-proxy fences), so the
//    down phase of the heavy groups overlaps the gate/up tail of the light ones and
//    there is no grid-wide barrier and no second launch;
//  * the smem ring (6 x 32 KB slots) runs across unit boundaries so the stream
//    never drains; two TMEM accumulators (2 x 256 columns) let the epilogue of
//    unit i overlap the MMAs of unit i+1; unit ids reach the MMA and epilogue warps
//    through a 4-entry smem queue;
//  * warp roles: warp 0 = producer (one lane), warp 1 = MMA issuer (one lane,
//    also owns TMEM alloc), warps 2..5 = epilogue (TMEM lane quadrants 2,3,0,1).
// Epilogues:
//  * gate/up: A rows interleave gate and up features in 16-row blocks
//    (pack_w13_kernel), so one warp's TMEM quadrant holds gate (lanes 0-15) and up
//    (lanes 16-31) of the same 16 features; h = act(g) * u via one shfl_xor, rounded
//    to bf16, stored straight into the swizzled B layout of the down phase
//    (moe.py:243-245);
//  * down: fp32 expert outputs per (row, feature), coalesced.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "params.cuh"
#include "plan.cuh"
#include "ptx.cuh"

namespace sere {

constexpr int kSlots = 6;
constexpr int kSlotBytes = 32768;
constexpr int kFfnThreads = 192;
constexpr int kTmemCols = 512;
constexpr int kQueue = 4;

struct Unit {
  int dn, g, expert, mt, ks, row0, n_mma, rows_valid, kt_begin, kt_end, need;
};

struct __align__(16) FfnSmemTail {
  uint64_t full[kSlots];
  uint64_t empty[kSlots];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint64_t q_full[kQueue];
  uint64_t q_empty[kQueue];
  int32_t queue[kQueue];
  uint32_t tmem_base;
  int32_t n_groups, units_gu, units_dn;
};

// per-schedule-position copies of the plan (6 arrays of Et + 1)
__host__ __device__ inline size_t ffn_smem_bytes(int Et) {
  return 1024 /*align slack*/ + static_cast<size_t>(kSlots) * kSlotBytes + sizeof(FfnSmemTail) +
         static_cast<size_t>(6) * (Et + 1) * sizeof(int32_t);
}

struct SchedView {
  const int32_t *uoff_gu, *uoff_dn, *gid, *gexp, *grow0, *grows;
};

__device__ __forceinline__ Unit decode_unit(int u, int n_groups, int units_gu, const SchedView& v,
                                            const FfnParams& p) {
  Unit U;
  U.dn = u >= units_gu;
  if (U.dn) u -= units_gu;
  const int32_t* uoff = U.dn ? v.uoff_dn : v.uoff_gu;
  int lo = 0, hi = n_groups - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (uoff[mid] <= u) lo = mid; else hi = mid - 1;
  }
  const int local = u - uoff[lo];
  const int rows = v.grows[lo];
  const int n16 = round_up(rows, kRowAlign);
  const int ncb = (n16 + kColBlock - 1) / kColBlock;
  const int nc = local % ncb;
  const int tmp = local / ncb;
  const int ksplit = U.dn ? p.ksplit_dn : 1;
  const int ktiles = U.dn ? p.ktiles_dn : p.ktiles_gu;
  U.ks = tmp % ksplit;
  U.mt = tmp / ksplit;
  U.g = v.gid[lo];
  U.expert = v.gexp[lo];
  const int col0 = nc * kColBlock;
  U.n_mma = min(kColBlock, n16 - col0);
  U.rows_valid = min(kColBlock, rows - col0);
  U.row0 = v.grow0[lo] + col0;
  const int kchunk = (ktiles + ksplit - 1) / ksplit;
  U.kt_begin = U.ks * kchunk;
  U.kt_end = min(ktiles, U.kt_begin + kchunk);
  U.need = p.tiles_gu * ncb;  // gate/up units of this group (the down units' dependency)
  return U;
}

__device__ __forceinline__ float act_apply(float g, int act) {
  if (act == 0) return g * __frcp_rn(1.0f + __expf(-g));  // SiLU (moe.py:28-35)
  if (act == 1) return fmaxf(g, 0.0f);                     // ReLU (moe.py:38-39)
  const float c = 0.7978845608028654f;                     // GELU-tanh (moe.py:42-45)
  return 0.5f * g * (1.0f + tanhf(c * (g + 0.044715f * g * g * g)));
}

__global__ void __launch_bounds__(kFfnThreads, 1) moe_ffn_kernel(const FfnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  FfnSmemTail* tail = reinterpret_cast<FfnSmemTail*>(smem + kSlots * kSlotBytes);
  int32_t* s_arr = reinterpret_cast<int32_t*>(tail + 1);
  const int E1 = p.Et + 1;
  SchedView sv{s_arr, s_arr + E1, s_arr + 2 * E1, s_arr + 3 * E1, s_arr + 4 * E1, s_arr + 5 * E1};

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const PlanOffsets po = plan_offsets(p.Et);
  int32_t* plan = p.plan;
  const int status = plan[P_STATUS];
  const int ng = status == 0 ? plan[P_NGROUPS] : 0;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kSlots; ++i) { mbar_init(&tail->full[i], 1); mbar_init(&tail->empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tail->tmem_full[i], 1); mbar_init(&tail->tmem_empty[i], 4); }
    for (int i = 0; i < kQueue; ++i) { mbar_init(&tail->q_full[i], 1); mbar_init(&tail->q_empty[i], 1 + 4); }
    fence_mbar_init();
    tail->n_groups = ng;
    tail->units_gu = status == 0 ? plan[P_UNITS_GU] : 0;
    tail->units_dn = status == 0 ? plan[P_UNITS_DN] : 0;
  }
  if (warp == 1) tmem_alloc(&tail->tmem_base, kTmemCols);
  for (int i = threadIdx.x; i <= ng; i += blockDim.x) {
    const_cast<int32_t*>(sv.uoff_gu)[i] = plan[po.unit_off_gu + i];
    const_cast<int32_t*>(sv.uoff_dn)[i] = plan[po.unit_off_dn + i];
    if (i < ng) {
      const int g = plan[po.sched + i];
      const_cast<int32_t*>(sv.gid)[i] = g;
      const_cast<int32_t*>(sv.gexp)[i] = plan[po.group_expert + g];
      const_cast<int32_t*>(sv.grow0)[i] = plan[po.group_row0 + g];
      const_cast<int32_t*>(sv.grows)[i] = plan[po.group_rows + g];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tail->tmem_base;
  const int n_groups = tail->n_groups, units_gu = tail->units_gu;
  const int units_total = units_gu + tail->units_dn;
  int32_t* dep = plan + po.dep;

  if (warp == 0) {
    if (lane == 0) {
      // ===================== producer: tickets -> unit queue; bulk async copies into the slot ring
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int slot = 0, qs = 0;
      uint32_t phase = 0, qph = 0;
      for (;;) {
        const int u = units_total > 0 ? atomicAdd(plan + P_TICKET, 1) : 0;
        const bool done = u >= units_total;
        mbar_wait(&tail->q_empty[qs], qph ^ 1u);
        tail->queue[qs] = done ? -1 : u;
        mbar_arrive(&tail->q_full[qs]);
        if (++qs == kQueue) { qs = 0; qph ^= 1u; }
        if (done) break;
        const Unit U = decode_unit(u, n_groups, units_gu, sv, p);
        const uint8_t* a_unit;
        const uint8_t* b_base;
        if (U.dn) {
          // h of this group must be complete: every gate/up unit of the group published it
          if (ld_acquire_gpu(dep + U.g) < U.need) {
            while (ld_acquire_gpu(dep + U.g) < U.need) __nanosleep(64);
          }
          fence_proxy_async_global();
          a_unit = p.w2 + (static_cast<size_t>(U.expert) * p.tiles_dn + U.mt) * p.ktiles_dn *
                              static_cast<size_t>(kTileBytes);
          b_base = p.h_pack;
        } else {
          a_unit = p.w13 + (static_cast<size_t>(U.expert) * p.tiles_gu + U.mt) * p.ktiles_gu *
                               static_cast<size_t>(kTileBytes);
          b_base = p.x_pack;
        }
        const int n0 = min(U.n_mma, 128), n1 = U.n_mma - n0;
        for (int kt = U.kt_begin; kt < U.kt_end; ++kt) {
          const uint8_t* b_src = b_base + (static_cast<size_t>(kt) * p.r_max + U.row0) * 128;
          mbar_wait(&tail->empty[slot], phase ^ 1u);
          uint8_t* sdst = smem + slot * kSlotBytes;
          mbar_arrive_expect_tx(&tail->full[slot], kTileBytes + n0 * 128);
          bulk_g2s(sdst, a_unit + static_cast<size_t>(kt) * kTileBytes, kTileBytes, &tail->full[slot], pol_w);
          bulk_g2s(sdst + kTileBytes, b_src, n0 * 128, &tail->full[slot], pol_x);
          if (++slot == kSlots) { slot = 0; phase ^= 1u; }
          if (n1 > 0) {
            mbar_wait(&tail->empty[slot], phase ^ 1u);
            sdst = smem + slot * kSlotBytes;
            mbar_arrive_expect_tx(&tail->full[slot], n1 * 128);
            bulk_g2s(sdst, b_src + 128 * 128, n1 * 128, &tail->full[slot], pol_x);
            if (++slot == kSlots) { slot = 0; phase ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===================== MMA issuer (single thread)
      int slot = 0, qs = 0, iter = 0;
      uint32_t phase = 0, qph = 0;
      for (;; ++iter) {
        mbar_wait(&tail->q_full[qs], qph);
        const int u = tail->queue[qs];
        mbar_arrive(&tail->q_empty[qs]);
        if (++qs == kQueue) { qs = 0; qph ^= 1u; }
        if (u < 0) break;
        const Unit U = decode_unit(u, n_groups, units_gu, sv, p);
        const int buf = iter & 1;
        const uint32_t use = static_cast<uint32_t>(iter >> 1);
        mbar_wait(&tail->tmem_empty[buf], (use & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d0 = tmem_base + buf * 256;
        const int n0 = min(U.n_mma, 128), n1 = U.n_mma - n0;
        const uint32_t idesc0 = umma_idesc_bf16(128, n0);
        const uint32_t idesc1 = n1 > 0 ? umma_idesc_bf16(128, n1) : 0u;
        for (int kt = U.kt_begin; kt < U.kt_end; ++kt) {
          const int s0 = slot;
          mbar_wait(&tail->full[s0], phase);
          if (++slot == kSlots) { slot = 0; phase ^= 1u; }
          int s1 = -1;
          if (n1 > 0) {
            s1 = slot;
            mbar_wait(&tail->full[s1], phase);
            if (++slot == kSlots) { slot = 0; phase ^= 1u; }
          }
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s0 * kSlotBytes);
          const uint32_t b0_addr = a_addr + kTileBytes;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t acc = (kt > U.kt_begin || k > 0) ? 1u : 0u;
            umma_bf16(d0, umma_desc_sw128(a_addr + 32 * k), umma_desc_sw128(b0_addr + 32 * k), idesc0, acc);
          }
          if (n1 > 0) {
            const uint32_t b1_addr = smem_u32(smem + s1 * kSlotBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t acc = (kt > U.kt_begin || k > 0) ? 1u : 0u;
              umma_bf16(d0 + 128, umma_desc_sw128(a_addr + 32 * k), umma_desc_sw128(b1_addr + 32 * k), idesc1,
                        acc);
            }
          }
          umma_commit(&tail->empty[s0]);
          if (s1 >= 0) umma_commit(&tail->empty[s1]);
        }
        umma_commit(&tail->tmem_full[buf]);
      }
    }
  } else {
    // ===================== epilogue warps 2..5 -> TMEM lane quadrant q = warp % 4
    const int q = warp & 3;
    int qs = 0, iter = 0;
    uint32_t qph = 0;
    for (;; ++iter) {
      mbar_wait(&tail->q_full[qs], qph);
      const int u = tail->queue[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail->q_empty[qs]);
      if (++qs == kQueue) { qs = 0; qph ^= 1u; }
      if (u < 0) break;
      const Unit U = decode_unit(u, n_groups, units_gu, sv, p);
      const int buf = iter & 1;
      const uint32_t use = static_cast<uint32_t>(iter >> 1);
      mbar_wait(&tail->tmem_full[buf], use & 1u);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * 256;
      if (!U.dn) {
        // lanes 0-15: gate of feature f, lanes 16-31: up of the same f
        const int f = 16 * q + (lane & 15);  // feature within the 64-feature tile == column of h tile
        const int chunk = f >> 3;
        uint8_t* hbase = p.h_pack + static_cast<size_t>(U.mt) * p.r_max * 128;
        for (int c0 = 0; c0 < U.n_mma; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(taddr + c0, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float g = __uint_as_float(r[i]);
            const float up = __shfl_xor_sync(0xffffffffu, g, 16);
            const float h = act_apply(g, p.act) * up;
            const float h_next = __shfl_down_sync(0xffffffffu, h, 1);
            if (lane < 16 && (lane & 1) == 0) {
              const int row = U.row0 + c0 + i;
              __nv_bfloat162 pair = __floats2bfloat162_rn(h, h_next);
              uint8_t* dst = hbase + static_cast<size_t>(row) * 128 + sw128_chunk(chunk, row) * 16 + (f & 7) * 2;
              *reinterpret_cast<__nv_bfloat162*>(dst) = pair;
            }
          }
        }
      } else {
        const int feat = U.mt * 128 + q * 32 + lane;
        float* ybase = p.y_perm + static_cast<size_t>(U.ks) * p.r_max * p.d_h_pad;
        for (int c0 = 0; c0 < U.n_mma; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(taddr + c0, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int j = c0 + i;
            if (j < U.rows_valid)
              ybase[static_cast<size_t>(U.row0 + j) * p.d_h_pad + feat] = __uint_as_float(r[i]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail->tmem_empty[buf]);
      if (!U.dn) {
        // publish this unit's slice of h: the down units of the group (any SM) read it with
        // bulk copies (async proxy) after acquiring the counter
        fence_proxy_async_global();
        named_bar_sync(1, 128);
        if (warp == 2 && lane == 0) {
          __threadfence();
          atomicAdd(dep + U.g, 1);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
}

cudaError_t launch_moe_ffn(const FfnParams& p, int num_sms, cudaStream_t stream) {
  const size_t smem = ffn_smem_bytes(p.Et);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(moe_ffn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  moe_ffn_kernel<<<num_sms, kFfnThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

size_t moe_ffn_smem(int Et) { return ffn_smem_bytes(Et); }

}  // namespace sere
