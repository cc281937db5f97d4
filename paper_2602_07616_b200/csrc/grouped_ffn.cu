// grouped_ffn.cu -- grouped expert GEMMs on the 5th-gen tensor cores (tcgen05).
//
// Decode-time MoE is expert-weight streaming: each active expert's weights are read
// once per layer while only 8..256 tokens use them, so the kernel is built to keep
// HBM busy, not the tensor pipe:
//  * swap-AB: A = a 128-row weight tile (MMA M = 128 output features), B = the
//    group's token rows (MMA N = 16..256), D = fp32 accumulator in TMEM;
//  * weights live in the bank as contiguous 16 KB pre-swizzled tiles, so one bulk
//    async copy (TMA engine, cp.async.bulk) per k-step streams 16 KB at full DRAM
//    burst length with an evict-first L2 policy; activations come from the grouped
//    swizzled buffer written by permute (L2-resident, evict-last);
//  * persistent CTAs (one per SM), static round-robin over work units
//    (expert group, m-tile, k-split, column block) read from the device-side plan;
//    the smem ring (6 x 32 KB slots) runs across unit boundaries so the stream
//    never drains; two TMEM accumulators (2 x 256 columns) let the epilogue of
//    unit i overlap the MMAs of unit i+1;
//  * warp roles: warp 0 = producer (one lane), warp 1 = MMA issuer (one lane,
//    also owns TMEM alloc), warps 2..5 = epilogue (TMEM lane quadrants 2,3,0,1).
// Epilogues:
//  * SWIGLU (gate/up GEMM): A rows interleave gate and up features in 16-row
//    blocks (pack_w13_kernel), so one warp's TMEM quadrant holds gate (lanes 0-15)
//    and up (lanes 16-31) of the same 16 features; h = act(g) * u via one
//    shfl_xor, rounded to bf16, stored straight into the swizzled B layout of the
//    down GEMM (moe.py:243-245);
//  * STORE_F32 (down GEMM): fp32 expert outputs per (row, feature), coalesced.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "params.cuh"
#include "plan.cuh"
#include "ptx.cuh"

namespace sere {

constexpr int kSlots = 6;
constexpr int kSlotBytes = 32768;
constexpr int kGemmThreads = 192;
constexpr int kTmemCols = 512;
constexpr int kMaxGroupsSmem = 1056;  // Et <= 1055 supported by the smem plan cache

struct Unit {
  int expert, mt, ks, row0, n_mma, rows_valid, kt_begin, kt_end;
};

struct __align__(16) GemmSmemTail {
  uint64_t full[kSlots];
  uint64_t empty[kSlots];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint32_t tmem_base;
  int32_t n_groups, n_units;
};

__host__ __device__ inline size_t gemm_smem_bytes(int Et) {
  return 1024 /*align slack*/ + static_cast<size_t>(kSlots) * kSlotBytes + sizeof(GemmSmemTail) +
         static_cast<size_t>(4) * (Et + 1) * sizeof(int32_t);
}

__device__ __forceinline__ Unit decode_unit(int u, int n_groups, const int32_t* s_uoff, const int32_t* s_exp,
                                            const int32_t* s_row0, const int32_t* s_rows, int ksplit,
                                            int ktiles) {
  int lo = 0, hi = n_groups - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_uoff[mid] <= u) lo = mid; else hi = mid - 1;
  }
  const int g = lo;
  const int local = u - s_uoff[g];
  const int rows = s_rows[g];
  const int n16 = round_up(rows, kRowAlign);
  const int ncb = (n16 + kColBlock - 1) / kColBlock;
  const int nc = local % ncb;
  const int tmp = local / ncb;
  Unit U;
  U.ks = tmp % ksplit;
  U.mt = tmp / ksplit;
  U.expert = s_exp[g];
  const int col0 = nc * kColBlock;
  U.n_mma = min(kColBlock, n16 - col0);
  U.rows_valid = min(kColBlock, rows - col0);
  U.row0 = s_row0[g] + col0;
  const int kchunk = (ktiles + ksplit - 1) / ksplit;
  U.kt_begin = U.ks * kchunk;
  U.kt_end = min(ktiles, U.kt_begin + kchunk);
  return U;
}

__device__ __forceinline__ float act_apply(float g, int act) {
  if (act == 0) return g / (1.0f + __expf(-g));  // SiLU (moe.py:28-35)
  if (act == 1) return fmaxf(g, 0.0f);           // ReLU (moe.py:38-39)
  const float c = 0.7978845608028654f;           // GELU-tanh (moe.py:42-45)
  return 0.5f * g * (1.0f + tanhf(c * (g + 0.044715f * g * g * g)));
}

__global__ void __launch_bounds__(kGemmThreads, 1) grouped_gemm_kernel(const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  GemmSmemTail* tail = reinterpret_cast<GemmSmemTail*>(smem + kSlots * kSlotBytes);
  int32_t* s_uoff = reinterpret_cast<int32_t*>(tail + 1);
  int32_t* s_exp = s_uoff + (p.Et + 1);
  int32_t* s_row0 = s_exp + (p.Et + 1);
  int32_t* s_rows = s_row0 + (p.Et + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const PlanOffsets po = plan_offsets(p.Et);
  const int status = p.plan[P_STATUS];

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kSlots; ++i) { mbar_init(&tail->full[i], 1); mbar_init(&tail->empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tail->tmem_full[i], 1); mbar_init(&tail->tmem_empty[i], 4); }
    fence_mbar_init();
    const int ng = status == 0 ? p.plan[P_NGROUPS] : 0;
    tail->n_groups = ng;
    tail->n_units = status == 0 ? p.plan[p.which == 0 ? P_UNITS_GU : P_UNITS_DN] : 0;
  }
  if (warp == 1) tmem_alloc(&tail->tmem_base, kTmemCols);
  if (status == 0) {
    const int ng = p.plan[P_NGROUPS];
    const int32_t* uoff = p.plan + (p.which == 0 ? po.unit_off_gu : po.unit_off_dn);
    for (int i = threadIdx.x; i <= ng; i += blockDim.x) {
      s_uoff[i] = uoff[i];
      if (i < ng) {
        s_exp[i] = p.plan[po.group_expert + i];
        s_row0[i] = p.plan[po.group_row0 + i];
        s_rows[i] = p.plan[po.group_rows + i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tail->tmem_base;
  const int n_groups = tail->n_groups, n_units = tail->n_units;

  if (warp == 0) {
    if (lane == 0) {
      // ===================== producer: bulk async copies into the slot ring
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int slot = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit U = decode_unit(u, n_groups, s_uoff, s_exp, s_row0, s_rows, p.ksplit, p.ktiles);
        const uint8_t* a_unit =
            p.a_base + (static_cast<size_t>(U.expert) * p.tiles_m + U.mt) * p.ktiles * static_cast<size_t>(kTileBytes);
        const int n0 = min(U.n_mma, 128), n1 = U.n_mma - n0;
        for (int kt = U.kt_begin; kt < U.kt_end; ++kt) {
          const uint8_t* b_src = p.b_base + (static_cast<size_t>(kt) * p.r_max + U.row0) * 128;
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
      int slot = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++iter) {
        const Unit U = decode_unit(u, n_groups, s_uoff, s_exp, s_row0, s_rows, p.ksplit, p.ktiles);
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
    int iter = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++iter) {
      const Unit U = decode_unit(u, n_groups, s_uoff, s_exp, s_row0, s_rows, p.ksplit, p.ktiles);
      const int buf = iter & 1;
      const uint32_t use = static_cast<uint32_t>(iter >> 1);
      mbar_wait(&tail->tmem_full[buf], use & 1u);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * 256;
      if (p.epi == EPI_SWIGLU) {
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
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
}

cudaError_t launch_grouped_gemm(const GemmParams& p, int num_sms, cudaStream_t stream) {
  const size_t smem = gemm_smem_bytes(p.Et);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(grouped_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  grouped_gemm_kernel<<<num_sms, kGemmThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

size_t grouped_gemm_smem(int Et) { return gemm_smem_bytes(Et); }

}  // namespace sere
