// grouped_ffn.cu -- the expert SwiGLU FFN of one MoE layer as ONE persistent kernel on
// the 5th-gen tensor cores (tcgen05), gate/up and down phases fused.
//
// Decode-time MoE is expert-weight streaming: each active expert's weights are read
// once per layer while only 8..256 tokens use them. Two bandwidths bound the kernel:
// HBM (the weights) and the L2 -> SM path, which carries the weights AND every
// re-read of the activation operand. The design therefore (a) streams weights as
// large contiguous bulk copies with an evict-first policy and (b) loads each
// activation tile once per k-step for several weight tiles:
//  * swap-AB: A = 128-row weight tiles (MMA M = 128 output features), B = the group's
//    token rows (MMA N = 16..256), D = fp32 accumulators in TMEM;
//  * a work unit is (phase, expert group, `mw` consecutive m-tiles, column block[, k
//    split]) -- plan.cuh unit_mw(): a gate/up unit takes 128-feature blocks (a gate
//    and an up tile each), a down unit up to 2 m-tiles, bounded by the 512 TMEM
//    columns. One k-step = one B tile + the unit's A tiles, so activations are re-read
//    d_m/128 (gate/up) and d_h/256 (down) times;
//  * weights live in the bank as contiguous 16 KB pre-swizzled tiles (one bulk async
//    copy each, TMA engine); activations come from the grouped swizzled buffers
//    (L2-resident, evict-last);
//  * shared memory is a ring of 104 granules of 2 KB (13 x 16 KB; an activation tile of n_mma
//    rows takes n_mma/16 granules, a weight tile 8); a pipeline step covers kKT k-tiles (1):
//    their B tiles and the unit's A tiles, consecutive granules, one (full, empty) mbarrier
//    pair from a 12-entry ring and one commit, so the stream never drains across unit
//    boundaries. The ring is allocated and released in FIFO order: a free-granule count
//    admits the next k-step in O(1);
//  * TMEM is a ring of columns: a unit takes mw * n_mma columns, the MMA of the next
//    unit starts as soon as no in-flight unit (4 unit slots, released in order by the
//    epilogue) holds its columns, so epilogues overlap MMAs whenever two units fit;
//  * persistent CTAs (one per SM) take units from a global ticket counter: every
//    gate/up unit first, then every down unit, groups in the plan's schedule order
//    (padded rows descending). A down unit waits, before its first copy, until every
//    gate/up unit of its group has published h (per-group counters in the plan,
//    release/acquire + async-proxy fences): no grid barrier, no second launch;
//  * warp roles: warp 0 = producer, warps 1-2 = MMA issuers (warp 1 also owns the TMEM
//    allocation; producer and issuers run converged and issue from an elected lane, so
//    tcgen05/bulk-copy operands reach the uniform registers without per-instruction
//    waterfall loops), warps 3..10 = epilogue (TMEM lane quadrant = warp % 4, two
//    warps per quadrant splitting the 16-column chunks: the fp32 down-output stores
//    otherwise hold TMEM long enough to stall the MMA issuer). Page,
//    column and slot positions are pure functions of the unit sequence, so the three
//    roles recompute them instead of exchanging them.
// Epilogues:
//  * gate/up: a feature block's gate tile and up tile (adjacent in the bank, one 32 KB
//    copy) accumulate into two TMEM accumulators, so the thread owning TMEM lane f
//    holds gate and up of feature f: h = act(g) * u without any exchange, rounded to
//    bf16 and stored straight into the swizzled B layout of the down phase
//    (moe.py:243-245);
//  * down: fp32 expert outputs per (row, feature), coalesced.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "params.cuh"
#include "plan.cuh"
#include "ptx.cuh"

namespace sere {

constexpr int kPageBytes = 16384;
// The operand ring is allocated in 2 KB granules: a weight tile takes 8, an activation tile
// n_mma/16 (a 16-row down tile 1 instead of a whole 16 KB page), so small-N k-steps keep more
// weight bytes in flight per SM
constexpr int kGranBytes = 2048;
#ifndef SERE_RING_GRANS
#define SERE_RING_GRANS 104
#endif
constexpr int kGrans = SERE_RING_GRANS;  // operand ring size in granules (104 = 13 x 16 KB)
constexpr int kRingBytes = kGrans * kGranBytes;
constexpr int kTileGrans = kPageBytes / kGranBytes;
#ifndef SERE_KENTRIES
#define SERE_KENTRIES 12
#endif
constexpr int kEntries = SERE_KENTRIES;   // k-step barrier ring
constexpr int kQueue = 4;     // unit-id queue producer -> MMA / epilogue
constexpr int kTq = 4;        // TMEM unit slots (barrier pairs)
#ifndef SERE_EPI_WARPS
#define SERE_EPI_WARPS 8
#endif
constexpr int kEpiWarps = SERE_EPI_WARPS;   // epilogue warps: kEpiWarps/4 per TMEM lane quadrant
constexpr int kEpiGroups = kEpiWarps / 4;   // warp groups splitting a unit's 16-column chunks
#ifndef SERE_MMA_WARPS
#define SERE_MMA_WARPS 2
#endif
// MMA issuer warps (one lane each), splitting a unit's accumulators: tcgen05.mma issue is
// latency-bound per issuing thread (scripts/micro/mma_rate.cu: 87 -> 59 cycles/MMA at
// N = 96 with two issuers), so two issuers interleave their issue chains
constexpr int kMmaWarps = SERE_MMA_WARPS;
constexpr int kEpiWarp0 = 1 + kMmaWarps;
constexpr int kFfnThreads = 32 * (1 + kMmaWarps + kEpiWarps);
constexpr int kPdlPrefetch = 4;
static_assert(kPageBytes == kTileBytes, "a page holds one weight tile");

struct Unit {
  int dn, g, expert, mt0, mwu, ks, row0, n_mma, rows_valid, kt_begin, kt_end, need;
};

struct __align__(16) FfnSmemTail {
  uint64_t full[kEntries];
  uint64_t empty[kEntries];
  uint64_t tfull[kTq];
  uint64_t tempty[kTq];
  uint64_t q_full[kQueue];
  uint64_t q_empty[kQueue];
  int32_t queue[kQueue];
  int32_t e_grans[kEntries];  // producer: granules held by each in-flight k-step (incl. a wrap's skipped tail)
  int32_t t_col[kMmaWarps][kTq], t_need[kMmaWarps][kTq];  // MMA: TMEM columns of in-flight units
  uint32_t tmem_base;
  int32_t n_groups, units_gu, units_dn;
};

// per-schedule-position copies of the plan (7 arrays of Et + 1)
__host__ __device__ inline size_t ffn_smem_bytes(int Et) {
  return 1024 /*align slack*/ + static_cast<size_t>(kRingBytes) + sizeof(FfnSmemTail) +
         static_cast<size_t>(7) * (Et + 1) * sizeof(int32_t);
}

struct SchedView {
  const int32_t *uoff_gu, *uoff_dn, *gid, *gexp, *grow0, *grows, *mw_gu;
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
  const int ncb = col_blocks(n16);
  const int tiles = U.dn ? p.tiles_dn : p.tiles_gu;
  const int mw = unit_mw(n16, U.dn ? dn_cap(n16) : v.mw_gu[lo], tiles, U.dn ? 1 : 2);
  const int nc = local % ncb;
  const int tmp = local / ncb;
  const int ksplit = U.dn ? p.ksplit_dn : 1;
  const int ktiles = U.dn ? p.ktiles_dn : p.ktiles_gu;
  U.ks = tmp % ksplit;
  U.mt0 = (tmp / ksplit) * mw;
  U.mwu = min(mw, tiles - U.mt0);
  U.g = v.gid[lo];
  U.expert = v.gexp[lo];
  const int col0 = nc * kColBlock;
  U.n_mma = min(kColBlock, n16 - col0);
  U.rows_valid = min(kColBlock, rows - col0);
  U.row0 = v.grow0[lo] + col0;
  const int kchunk = (ktiles + ksplit - 1) / ksplit;
  U.kt_begin = U.ks * kchunk;
  U.kt_end = min(ktiles, U.kt_begin + kchunk);
  U.need = group_units_gu(n16, p.tiles_gu, v.mw_gu[lo]);  // gate/up units of this group (the down units' dependency)
  return U;
}

#ifndef SERE_KT
#define SERE_KT 1
#endif
constexpr int kKT = SERE_KT;  // 64-wide k-tiles per pipeline step (1: finest-grained page release; 2 measured slower)
// A tiles (= TMEM accumulators) of one k-tile: gate and up per gate/up feature block, one per down m-tile
__device__ __forceinline__ int kstep_atiles(const Unit& U) { return U.dn ? U.mwu : 2 * U.mwu; }
// granules of the B tile of one k-tile (n_mma rows of 128 B)
__device__ __forceinline__ int ktile_bgrans(const Unit& U) { return U.n_mma / 16; }
// granules of a step of nk k-tiles: the nk B tiles, then per m-tile block j its nk k-tiles' A tiles
__device__ __forceinline__ int kstep_grans(const Unit& U, int nk) {
  return nk * (ktile_bgrans(U) + kstep_atiles(U) * kTileGrans);
}

__device__ __forceinline__ bool ranges_overlap(int a, int na, int b, int nb) { return a < b + nb && b < a + na; }

__device__ __forceinline__ float act_apply(float g, int act) {
  if (act == 0) return __fdividef(g, 1.0f + __expf(-g));  // SiLU (moe.py:28-35); -> -0 for g << 0
  if (act == 1) return fmaxf(g, 0.0f);                     // ReLU (moe.py:38-39)
  const float c = 0.7978845608028654f;                     // GELU-tanh (moe.py:42-45)
  return 0.5f * g * (1.0f + tanhf(c * (g + 0.044715f * g * g * g)));
}

__global__ void __launch_bounds__(kFfnThreads, 1) moe_ffn_kernel(const FfnParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1 KB alignment (SW128 atoms) by offsetting the __shared__ array itself, so the
  // compiler keeps shared-state accesses in the shared address space (LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  FfnSmemTail* tail = reinterpret_cast<FfnSmemTail*>(smem + kRingBytes);
  int32_t* s_arr = reinterpret_cast<int32_t*>(tail + 1);
  const int E1 = p.Et + 1;
  SchedView sv{s_arr, s_arr + E1, s_arr + 2 * E1, s_arr + 3 * E1, s_arr + 4 * E1, s_arr + 5 * E1, s_arr + 6 * E1};

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const PlanOffsets po = plan_offsets(p.Et);
  int32_t* plan = p.plan;
  const int status = plan[P_STATUS];
  const int ng = status == 0 ? plan[P_NGROUPS] : 0;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kEntries; ++i) {
      mbar_init(&tail->full[i], 1);
      mbar_init(&tail->empty[i], kMmaWarps);
    }
    for (int i = 0; i < kTq; ++i) { mbar_init(&tail->tfull[i], kMmaWarps); mbar_init(&tail->tempty[i], kEpiWarps); }
    for (int i = 0; i < kQueue; ++i) {
      mbar_init(&tail->q_full[i], 1);
      mbar_init(&tail->q_empty[i], kMmaWarps + kEpiWarps);
    }
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
      const_cast<int32_t*>(sv.mw_gu)[i] = plan[po.mw_gu + i];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tail->tmem_base;
  const int n_groups = tail->n_groups, units_gu = tail->units_gu;
  const int units_total = units_gu + tail->units_dn;
  int32_t* dep = plan + po.dep;
  unsigned long long* tr = p.trace ? p.trace + static_cast<size_t>(blockIdx.x) * kFfnTraceStride : nullptr;
  if (tr && threadIdx.x == 0) { tr[0] = globaltimer_ns(); tr[813] = clock64(); }
  // no early pdl_trigger: a combine grid resident during the FFN measurably slows it down

  if (warp == 0) {
    {
      // ===================== producer: tickets -> unit queue; bulk async copies into the page ring.
      // The whole warp walks the loop converged (every value warp-uniform) and one elected lane
      // issues each barrier arrival and copy, so the copies' operands reach the TMA unit without
      // a per-copy ELECT/R2UR.BROADCAST waterfall
      if (lane != 0) tr = nullptr;
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int qs = 0, nu = 0, head = 0, kstep = 0, oldest = 0;
      int ring_free = kGrans;  // granules not held by in-flight k-steps
      int e = 0, e_old = 0;     // barrier entries of the next and the oldest in-flight k-step
      uint32_t ph_old = 0;      // parity of the oldest one's empty barrier
      uint32_t qph = 0;
      unsigned long long w_empty = 0, w_dep = 0, w_q = 0, w_empty_dn = 0;
      // PDL: weights do not depend on the preceding kernel (permute), so the first k-steps'
      // weight tiles are issued before griddepcontrol.wait; their activation tiles follow it
      // The same deferral serves a down unit whose group's h is not complete yet: its weight
      // tiles stream while the gate/up units of the group finish, and its h tiles follow
      // the dependency wait. "gates" = PDL not yet waited / dependency not yet met.
      bool pdl_done = false;
      int dep_g = -1, dep_need = 0;  // open dependency gate of the current down unit
      int n_pend = 0;
      uint32_t pend_dst[kPdlPrefetch], pend_bytes[kPdlPrefetch], pend_bar[kPdlPrefetch];
      const uint8_t* pend_src[kPdlPrefetch];
      auto pdl_flush = [&]() {
        if (!pdl_done) pdl_wait();
        if (dep_g >= 0) {
          const long long t0 = tr ? clock64() : 0;
          while (ld_acquire_gpu(dep + dep_g) < dep_need) __nanosleep(64);
          if (tr) w_dep += static_cast<unsigned long long>(clock64() - t0);
          fence_proxy_async_global();  // h was written by generic stores on other SMs
          dep_g = -1;
        }
        for (int i = 0; i < n_pend; ++i) bulk_g2s_elect(pend_dst[i], pend_src[i], pend_bytes[i], pend_bar[i], pol_x);
        n_pend = 0;
        pdl_done = true;
      };
      unsigned long long* acc_empty = tr ? &w_empty : nullptr;
      for (;; ++nu) {
        // the first unit of CTA b is ticket b (no atomic round trip before the first copy);
        // the counter hands out tickets from gridDim.x on
        int tk = 0;
        if (lane == 0 && units_total > 0 && nu > 0) tk = atomicAdd(plan + P_TICKET, 1);
        tk = __shfl_sync(0xffffffffu, tk, 0);
        const int u = units_total <= 0 ? 0 : nu == 0 ? static_cast<int>(blockIdx.x) : static_cast<int>(gridDim.x) + tk;
        unsigned long long* ut = (tr && nu < kFfnTraceUnits) ? tr + 8 + 4 * nu : nullptr;
        if (ut) { ut[0] = u; ut[1] = globaltimer_ns(); }
        const bool done = u >= units_total;
        mbar_wait_timed(&tail->q_empty[qs], qph ^ 1u, tr ? &w_q : nullptr);
        if (lane == 0) {
          tail->queue[qs] = done ? -1 : u;
          mbar_arrive(&tail->q_full[qs]);
        }
        __syncwarp();
        if (++qs == kQueue) { qs = 0; qph ^= 1u; }
        if (done) {
          if (tr) { tr[1] = w_empty + w_empty_dn; tr[3] = nu; tr[4] = w_dep; tr[809] = w_q; tr[1018] = w_empty_dn; }
          break;
        }
        const Unit U = decode_unit(u, n_groups, units_gu, sv, p);
        const uint8_t* a_unit;
        const uint8_t* b_base;
        size_t a_mt_stride;  // bytes between consecutive m-tiles (feature blocks) of the expert
        uint32_t a_copy;     // bytes of one m-tile at one k-step (gate+up adjacent for gate/up)
        if (U.dn) {
          // h of this group must be complete (every gate/up unit of the group published it)
          // before its h tiles are copied; if not yet, the gate defers them (pdl_flush)
          if (ld_acquire_gpu(dep + U.g) < U.need) {
            dep_g = U.g;
            dep_need = U.need;
            pdl_flush();  // (streaming the weights before this wait measured 1.5% slower)
          } else {
            fence_proxy_async_global();
          }
          a_copy = kTileBytes;
          a_mt_stride = 0;  // unused: the unit's m-tiles are adjacent per k-tile (w2_tile_offset)
          a_unit = p.w2 + w2_tile_offset(U.expert, U.mt0, 0, p.tiles_dn, p.ktiles_dn);
          b_base = p.h_pack;
        } else {
          a_copy = 2 * kTileBytes;
          a_mt_stride = static_cast<size_t>(p.ktiles_gu) * a_copy;
          a_unit = p.w13 + (static_cast<size_t>(U.expert) * p.tiles_gu + U.mt0) * a_mt_stride;
          b_base = p.x_pack;
        }
        if (ut) {  // ticket | weight KB << 24 | n_mma << 44 | down << 53
          ut[0] = static_cast<unsigned long long>(u) |
                  (static_cast<unsigned long long>(U.mwu) * a_copy * (U.kt_end - U.kt_begin) / 1024 << 24) |
                  (static_cast<unsigned long long>(U.n_mma) << 44) | (static_cast<unsigned long long>(U.dn) << 53);
          ut[2] = globaltimer_ns();
        }
        const int bgr = ktile_bgrans(U);
        const uint32_t b_bytes = static_cast<uint32_t>(U.n_mma) * 128u;
        for (int kt = U.kt_begin; kt < U.kt_end; kt += kKT, ++kstep) {
          const int nk = min(kKT, U.kt_end - kt);
          const int np = kstep_grans(U, nk);
          const size_t a_off = static_cast<size_t>(nk) * bgr * kGranBytes;  // A tiles follow the nk B tiles
          const uint32_t tx = nk * (b_bytes + ((p.dbg_mode & 1) ? 0u : static_cast<uint32_t>(U.mwu) * a_copy));
          // the ring is allocated and released in FIFO order, so the in-flight k-steps hold one
          // contiguous arc and a count of free granules decides admission (a k-step that would
          // cross the end of the ring starts at 0 and also holds the skipped tail)
          const bool wrap = head + np > kGrans;
          // (a k-step larger than the skipped tail needs the whole ring free: cap at the ring size,
          // a conservative count that still releases exactly what it took)
          const int hold = min(kGrans, (wrap ? kGrans - head : 0) + np);
          while (kstep - oldest >= kEntries || ring_free < hold) {
            // an in-flight k-step can only complete once its deferred activation copy is issued
            if (!pdl_done || dep_g >= 0) pdl_flush();
            mbar_wait_timed(&tail->empty[e_old], ph_old, acc_empty ? (U.dn ? &w_empty_dn : acc_empty) : nullptr);
            ring_free += tail->e_grans[e_old];
            ++oldest;
            if (++e_old == kEntries) { e_old = 0; ph_old ^= 1u; }
          }
          if (wrap) head = 0;
          ring_free -= hold;
          tail->e_grans[e] = hold;
          uint8_t* pg = smem + static_cast<size_t>(head) * kGranBytes;
          mbar_arrive_expect_tx_elect(&tail->full[e], tx);
          const uint32_t bar_e = smem_u32(&tail->full[e]);
          if (!(p.dbg_mode & 1)) {
            if (U.dn) {  // k-tile kk: the unit's 1-2 adjacent m-tiles, one copy (pages kk-major)
              for (int kk = 0; kk < nk; ++kk) {
                bulk_g2s_elect(smem_u32(pg + a_off + static_cast<size_t>(kk * U.mwu) * kPageBytes),
                               a_unit + static_cast<size_t>(kt + kk) * kW2Group * kTileBytes, U.mwu * kTileBytes, bar_e,
                               pol_w);
              }
            } else {  // feature block j at k-tiles kt..kt+nk-1: gate/up tiles, one contiguous copy
              const uint8_t* a_kt = a_unit + static_cast<size_t>(kt) * a_copy;
              for (int j = 0; j < U.mwu; ++j)
                bulk_g2s_elect(smem_u32(pg + a_off + j * nk * a_copy), a_kt + j * a_mt_stride, nk * a_copy, bar_e,
                               pol_w);
            }
          }
          const bool gated = !pdl_done || dep_g >= 0;
          if (gated && n_pend + nk > kPdlPrefetch) pdl_flush();
          for (int kk = 0; kk < nk; ++kk) {
            uint8_t* bdst = pg + static_cast<size_t>(kk * bgr) * kGranBytes;
            const uint8_t* bsrc = b_base + (static_cast<size_t>(kt + kk) * p.r_max + U.row0) * 128;
            if (pdl_done && dep_g < 0) {
              bulk_g2s_elect(smem_u32(bdst), bsrc, b_bytes, bar_e, pol_x);
            } else {
              pend_dst[n_pend] = smem_u32(bdst);
              pend_src[n_pend] = bsrc;
              pend_bytes[n_pend] = b_bytes;
              pend_bar[n_pend] = bar_e;
              ++n_pend;
            }
          }
          head += np;
          if (++e == kEntries) e = 0;
        }
        if (!pdl_done || dep_g >= 0) pdl_flush();
        if (ut) ut[3] = globaltimer_ns();
      }
      if (!pdl_done) pdl_flush();
    }
  } else if (warp < kEpiWarp0) {
    {
      // ===================== MMA issuers: issuer mi takes the unit's accumulators a with
      // a % kMmaWarps == mi; both walk every k-step (full/empty barriers count both). The whole
      // warp walks the loop converged and one elected lane issues (umma_bf16_elect)
      const int mi = warp - 1;
      int qs = 0, iter = 0, head = 0, kstep = 0, tcol = 0, oldest = 0;
      int e = 0;          // barrier entry of the k-step
      uint32_t eph = 0;   // its full-barrier parity
      uint32_t qph = 0;
      unsigned long long w_full = 0, w_tmem = 0, nks = 0, w_full_dn = 0, w_tmem_dn = 0, nks_dn = 0;
      unsigned long long* acc_full = (tr && mi == 0) ? &w_full : nullptr;
      if (mi != 0 || lane != 0) tr = nullptr;  // issuer 0 keeps the trace
      if (lane != 0) acc_full = nullptr;
      for (;; ++iter) {
        mbar_wait(&tail->q_full[qs], qph);
        const int u = tail->queue[qs];
        __syncwarp();
        if (lane == 0) mbar_arrive(&tail->q_empty[qs]);
        if (++qs == kQueue) { qs = 0; qph ^= 1u; }
        if (u < 0) {
          if (tr) {
            tr[2] = w_full + w_full_dn; tr[5] = w_tmem + w_tmem_dn; tr[810] = nks;
            tr[1019] = w_full_dn; tr[1020] = w_tmem_dn; tr[1021] = nks_dn;
          }
          break;
        }
        const Unit U = decode_unit(u, n_groups, units_gu, sv, p);
        // TMEM columns of this unit: FIFO ring over the 512 columns
        const int na = kstep_atiles(U);
        const int need = na * U.n_mma;
        if (tcol + need > kTmemCols) tcol = 0;
        const int col = tcol;
        tcol += need;
        for (;;) {  // release in FIFO order until no in-flight unit holds these columns
          bool busy = iter - oldest >= kTq;
          for (int i2 = oldest; !busy && i2 < iter; ++i2)
            busy = ranges_overlap(col, need, tail->t_col[mi][i2 % kTq], tail->t_need[mi][i2 % kTq]);
          if (!busy) break;
          mbar_wait_timed(&tail->tempty[oldest % kTq], static_cast<uint32_t>(oldest / kTq) & 1u,
                          tr ? (U.dn ? &w_tmem_dn : &w_tmem) : nullptr);
          ++oldest;
        }
        __syncwarp();
        if (lane == 0) {
          tail->t_col[mi][iter % kTq] = col;
          tail->t_need[mi][iter % kTq] = need;
        }
        __syncwarp();
        tc_fence_after();
        const int bgr = ktile_bgrans(U), apj = U.dn ? 1 : 2;  // A tiles per m-tile block and k-tile
        const uint32_t idesc = umma_idesc_bf16(128, U.n_mma);
        const uint32_t d0 = tmem_base + col;
        for (int kt = U.kt_begin; kt < U.kt_end; kt += kKT, ++kstep) {
          const int nk = min(kKT, U.kt_end - kt);
          const int np = kstep_grans(U, nk);
          const uint32_t a_off = static_cast<uint32_t>(nk * bgr * kGranBytes);
          if (head + np > kGrans) head = 0;
          mbar_wait_timed(&tail->full[e], eph,
                          acc_full ? (U.dn ? &w_full_dn : acc_full) : nullptr);
          nks_dn += U.dn;
          tc_fence_after();
          const uint32_t pg_addr = smem_u32(smem + static_cast<size_t>(head) * kGranBytes);
          if (!(p.dbg_mode & 2)) {
            for (int kk = 0; kk < nk; ++kk) {
              const uint32_t b_addr = pg_addr + kk * bgr * kGranBytes;
              for (int j = 0; j < U.mwu; ++j) {
                for (int s2 = 0; s2 < apj; ++s2) {  // accumulator j*apj + s2 (gate/up: gate then up)
                  if ((j * apj + s2) % kMmaWarps != mi) continue;
                  const int apage = U.dn ? kk * U.mwu + j : (j * nk + kk) * apj + s2;
                  const uint32_t a_addr = pg_addr + a_off + apage * kPageBytes;
                  const uint32_t dj = d0 + (j * apj + s2) * U.n_mma;
#pragma unroll
                  for (int k = 0; k < 4; ++k) {
                    const uint32_t acc = (kt + kk > U.kt_begin || k > 0) ? 1u : 0u;
                    umma_bf16_elect(dj, umma_desc_sw128(a_addr + 32 * k), umma_desc_sw128(b_addr + 32 * k), idesc,
                                    acc);
                  }
                }
              }
            }
          }
          ++nks;
          umma_commit_elect(&tail->empty[e]);
          if (++e == kEntries) { e = 0; eph ^= 1u; }
          head += np;
        }
        umma_commit_elect(&tail->tfull[iter % kTq]);
        if (tr && iter < kFfnTraceUnits) tr[1280 + iter] = globaltimer_ns();  // last MMA issued
      }
    }
  } else {
    // ===================== epilogue warps -> TMEM lane quadrant q = warp % 4
    const int q = warp & 3;                    // TMEM lane quadrant of this warp
    const int eg = (warp - kEpiWarp0) / 4;     // column group: chunks c0 = 16 * (eg + kEpiGroups * i)
    int qs = 0, iter = 0, tcol = 0;
    uint32_t qph = 0;
    unsigned long long w_tf = 0;
    for (;; ++iter) {
      mbar_wait(&tail->q_full[qs], qph);
      const int u = tail->queue[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail->q_empty[qs]);
      if (++qs == kQueue) { qs = 0; qph ^= 1u; }
      if (u < 0) {
        if (tr && warp == kEpiWarp0 && lane == 0) tr[6] = w_tf;
        break;
      }
      const Unit U = decode_unit(u, n_groups, units_gu, sv, p);
      const int need = kstep_atiles(U) * U.n_mma;
      if (tcol + need > kTmemCols) tcol = 0;
      const int col = tcol;
      tcol += need;
      mbar_wait_timed(&tail->tfull[iter % kTq], static_cast<uint32_t>(iter / kTq) & 1u,
                      (tr && warp == kEpiWarp0 && lane == 0) ? &w_tf : nullptr);
      if (tr && warp == kEpiWarp0 && lane == 0 && iter < kFfnTraceUnits) tr[1024 + iter] = globaltimer_ns();
      __syncwarp();
      tc_fence_after();
      const uint32_t tq = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + col;
      // The epilogue is issue-bound (one store per element per thread): addresses are
      // strength-reduced per 16-row chunk. Unit rows start on a 16-row boundary
      // (kRowAlign) and chunks are 16 rows, so the swizzle phase of row c0 + i is i & 7.
      if (!U.dn) {
        // feature f of block fb: its gate and up accumulators sit in this thread's TMEM lane,
        // so h = act(g) * u needs no data exchange; one bf16 per (row, f) into the swizzled
        // B layout of the down phase
        for (int j = 0; j < U.mwu; ++j) {
          const int f = (U.mt0 + j) * 128 + q * 32 + lane;
          const int fl = f & 63, ch = fl >> 3;
          uint8_t* hcol = p.h_pack + static_cast<size_t>(f >> 6) * p.r_max * 128 +
                          static_cast<size_t>(U.row0) * 128 + (fl & 7) * 2;
          const uint32_t tg = tq + (2 * j) * U.n_mma, tu = tg + U.n_mma;
          for (int c0 = 16 * eg; c0 < U.n_mma; c0 += 16 * kEpiGroups) {
            uint32_t rg[16], ru[16];
            tmem_ld16(tg + c0, rg);
            tmem_ld16(tu + c0, ru);
            tmem_wait_ld();
            float hv[16];
            if (p.act == 0) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float g = __uint_as_float(rg[i]);
                hv[i] = __fdividef(g, 1.0f + __expf(-g)) * __uint_as_float(ru[i]);
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) hv[i] = act_apply(__uint_as_float(rg[i]), p.act) * __uint_as_float(ru[i]);
            }
            uint8_t* hp = hcol + static_cast<size_t>(c0) * 128;
#pragma unroll
            for (int i = 0; i < 16; ++i)
              *reinterpret_cast<__nv_bfloat16*>(hp + i * 128 + ((ch ^ (i & 7)) << 4)) = __float2bfloat16_rn(hv[i]);
          }
        }
      } else {
        // down: both m-tiles' chunk loads in flight behind one wait; fp32 rows of y_perm
        const size_t ld = p.d_h_pad;
        float* ycol = p.y_perm + static_cast<size_t>(U.ks) * p.r_max * ld + static_cast<size_t>(U.row0) * ld +
                      U.mt0 * 128 + q * 32 + lane;
        const bool store = !(p.dbg_mode & 4);
        for (int c0 = 16 * eg; c0 < U.n_mma; c0 += 16 * kEpiGroups) {
          uint32_t r[kMwDnMax][16];
#pragma unroll
          for (int j = 0; j < kMwDnMax; ++j)
            if (j < U.mwu) tmem_ld16(tq + j * U.n_mma + c0, r[j]);
          tmem_wait_ld();
          const int nv = U.rows_valid - c0;
          if (store) {
#pragma unroll
            for (int j = 0; j < kMwDnMax; ++j) {
              if (j < U.mwu) {
                float* yp = ycol + static_cast<size_t>(c0) * ld + j * 128;
                if (nv >= 16) {
#pragma unroll
                  for (int i = 0; i < 16; ++i) { *yp = __uint_as_float(r[j][i]); yp += ld; }
                } else {
#pragma unroll
                  for (int i = 0; i < 16; ++i) { if (i < nv) *yp = __uint_as_float(r[j][i]); yp += ld; }
                }
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail->tempty[iter % kTq]);
      if (tr && warp == kEpiWarp0 && lane == 0 && iter < kFfnTraceUnits) tr[816 + iter] = globaltimer_ns();
      if (!U.dn) {
        // publish this unit's slice of h: the down units of the group (any SM) read it with
        // bulk copies (async proxy) after acquiring the counter
        fence_proxy_async_global();
        named_bar_sync(1, 32 * kEpiWarps);
        if (warp == kEpiWarp0 && lane == 0) {
          __threadfence();
          atomicAdd(dep + U.g, 1);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tr && threadIdx.x == 0) { tr[7] = globaltimer_ns(); tr[814] = clock64(); }
  if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
  if (threadIdx.x == 0) {  // last CTA out re-arms the plan's counters (and, expert parallel, arrives)
    if (p.sync.world > 0) __threadfence_system();  // this CTA's expert outputs, read by the peers
    else __threadfence();
    if (atomicAdd(plan + P_DONE, 1) == static_cast<int>(gridDim.x) - 1) {
      for (int g = 0; g < ng; ++g) dep[g] = 0;
      plan[P_TICKET] = 0;
      plan[P_DONE] = 0;
      __threadfence();
      if (p.sync.world > 0) ep_arrive(p.sync);
    }
  }
}

cudaError_t launch_moe_ffn(const FfnParams& p, int num_sms, cudaStream_t stream) {
  const size_t smem = ffn_smem_bytes(p.Et);
  static SmemAttrCache attr;
  if (cudaError_t e = ensure_smem_attr(moe_ffn_kernel, smem, attr, 0); e != cudaSuccess) return e;
  return launch_pdl((g_pdl & PDL_FFN) != 0, moe_ffn_kernel, dim3(num_sms), dim3(kFfnThreads), smem, stream, p);
}

size_t moe_ffn_smem(int Et) { return ffn_smem_bytes(Et); }

}  // namespace sere
