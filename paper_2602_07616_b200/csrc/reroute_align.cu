// reroute_align.cu -- the SERE re-routing kernel fused with count/align.
//
// One CTA of 1024 threads does, entirely in shared memory:
//  (1) re-routing, restating rerouting.apply_sere (rerouting.py:130-171) as the
//      Alg. 2 data-parallel kernel (rerouting.py:174-249):
//      primary H-mask from slots < S by atomicOr into a smem bitmask, one warp per
//      distinct secondary expert u for the fp64 argmax over {v : H[v]} of sim[u,v]
//      (ties -> lowest index, exactly the ascending strict-`>` scan of
//      best_primary_match rerouting.py:78-97), the `rho > 0 && s* < rho` test
//      (rerouting.py:160) and the per-cell rewrite of slots >= S;
//  (2) count/align for the grouped FFN: per-expert counts over the (rewritten)
//      table, groups = active experts ascending then shared experts, each padded
//      to 16 rows; a deterministic rank inside each group (rows ordered by token
//      block, slot, token) from per-warp smem token masks + popc, giving
//      slot_row[t,k] and the inverse row_token[row]; work-unit prefixes for both
//      grouped GEMMs. Threads own whole token rows (no div/mod by K).
// Everything is integer / fp64-compare work on <= 16K cells: latency-bound, so a
// single CTA with no global round trips between phases is the fastest shape.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "../../include/sere_b200.h"
#include "params.cuh"
#include "plan.cuh"
#include "ptx.cuh"

namespace sere {

#ifndef SERE_ALIGN_THREADS
#define SERE_ALIGN_THREADS 1024  // 256: the block size a fused router-tail variant would have (f1 A/B)
#endif
constexpr int kAlignThreads = SERE_ALIGN_THREADS;
constexpr int kTokBlk = kTokBlkPerm;  // token block of the group row order (the permute ranks inside it)
constexpr int kMaxGroupsSched = 320;  // >= max bank experts + shared experts (capi.cu kMaxExperts + kMaxShared)
#define SERE_PHASE(i) do { if (p.dbg && threadIdx.x == 0) p.dbg[(i)] = clock64(); } while (0)

// M = global expert count (ids, sim, classes); Et = local groups (bank experts + shared)
__host__ __device__ inline size_t align_smem_bytes(int T, int K, int M, int Et) {
  const int TK = T * K, TB = (T + kTokBlk - 1) / kTokBlk;
  size_t b = 0;
  b += static_cast<size_t>(TK) * 4;                   // s_ids
  b += static_cast<size_t>(M) * 4;                    // s_map
  b += static_cast<size_t>(Et) * 4 * 4;               // s_cnt, s_row0, s_gpad, s_sched
  b += static_cast<size_t>(round_up(TB * Et, 2)) * 2; // s_cntb (u16 pairs updated by 32-bit atomics)
  b += static_cast<size_t>(round_up(M, 4)) * 3;       // s_hflag, s_sec, s_cls
  return round_up(static_cast<int>(b), 16);
}
// The similarity matrix is staged into shared memory after the fixed arrays when it fits: one
// bulk copy issued BEFORE the PDL wait (the sim is static per layer, so the copy overlaps the
// router); the argmax then reads shared memory instead of L2.
constexpr size_t kAlignSmemCap = 200 * 1024;
__host__ __device__ inline size_t align_smem_total(int T, int K, int M, int Et, bool stage_sim) {
  return align_smem_bytes(T, K, M, Et) + (stage_sim ? static_cast<size_t>(M) * M * 8 : 0);
}

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = lane_id();
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v += o;
  }
  return v;
}

__global__ void __launch_bounds__(kAlignThreads, 1) reroute_align_kernel(AlignParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = p.T, K = p.K, M = p.M, S = p.S;
  const int TK = T * K, TB = (T + kTokBlk - 1) / kTokBlk;
  const int e_lo = p.e_lo, m_loc = p.m_local, Et = m_loc + p.n_shared;  // expert-parallel ownership
  int32_t* s_ids = reinterpret_cast<int32_t*>(smem);
  int32_t* s_map = s_ids + TK;
  int32_t* s_cnt = s_map + M;    // per bank-expert totals
  int32_t* s_row0 = s_cnt + Et;  // first permuted row of each bank expert's group
  int32_t* s_gpad = s_row0 + Et;  // padded rows of group g
  int32_t* s_sched = s_gpad + Et; // schedule order of the groups
  uint16_t* s_cntb = reinterpret_cast<uint16_t*>(s_sched + Et);  // [TB][Et] counts -> prefixes
  uint8_t* s_hflag = reinterpret_cast<uint8_t*>(s_cntb + round_up(TB * Et, 2));
  uint8_t* s_sec = s_hflag + round_up(M, 4);   // expert named by some slot >= S
  uint8_t* s_cls = s_sec + round_up(M, 4);
  const double* s_sim = reinterpret_cast<const double*>(smem + align_smem_bytes(T, K, M, Et));  // if p.stage_sim
  __shared__ int s_err_id, s_err_sim, s_err_route, s_err_domain;
  __shared__ __align__(8) uint64_t s_sim_bar;

  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  const bool reroute = (p.mode & MODE_REROUTE) != 0;
  const bool align = (p.mode & MODE_ALIGN) != 0;
  const int s_eff = S < K ? S : K;  // S == K: identity re-routing, every routed expert is primary
  auto local_of = [&](int e) { return (e >= e_lo && e < e_lo + m_loc) ? e - e_lo : -1; };

  const bool stage = reroute && p.stage_sim;
  if (tid == 0) {
    s_err_id = 0; s_err_sim = 0; s_err_route = 0; s_err_domain = 0;
    if (stage) {  // static data: issued before the PDL wait, lands while the router runs
      mbar_init(&s_sim_bar, 1);
      fence_mbar_init();
      const uint32_t bytes = static_cast<uint32_t>(M) * M * 8;
      mbar_arrive_expect_tx(&s_sim_bar, bytes);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(s_sim)),
          "l"(p.sim), "r"(bytes), "r"(smem_u32(&s_sim_bar))
          : "memory");
    }
  }
  for (int e = tid; e < M; e += nthr) { s_map[e] = -1; s_cls[e] = 0; s_hflag[e] = 0; s_sec[e] = 0; }
  if (align)
    for (int i = tid; i < round_up(TB * Et, 2) / 2; i += nthr) reinterpret_cast<uint32_t*>(s_cntb)[i] = 0u;
  __syncthreads();
  pdl_wait();  // ids come from the router; outputs are read by the previous layer's kernels
  pdl_trigger();
  if (p.sync.world > 0) {  // expert parallel: every rank's router rows must have landed (fused barrier)
    if (tid == 0 && !ep_wait(p.sync)) s_err_domain = -1;
    __syncthreads();
    if (s_err_domain < 0) {
      if (stage) mbar_wait(&s_sim_bar, 0);  // no CTA exit with the bulk copy in flight
      if (tid == 0) {
        if (p.status_dev) *p.status_dev = SERE_ERR_CUDA;
        if (p.plan) p.plan[P_STATUS] = SERE_ERR_CUDA;
      }
      return;
    }
  }
  SERE_PHASE(0);

  // ---- load + validate ids (rerouting.py:111-114 / moe.py:299-300); lane = token, no div/mod
  const bool vec = (K & 3) == 0 && (reinterpret_cast<uintptr_t>(p.ids_in) & 15) == 0;
  // s_ids is column-major [K][T] so that lane = token accesses are bank-conflict free. One
  // item per (token, 4-slot quad): T * ceil(K/4) items keep every thread busy
  {
    const int nq = (K + 3) >> 2;
    bool bad = false;
    for (int it = tid; it < T * nq; it += nthr) {
      const int t = it / nq, k0 = (it - t * nq) * 4;
      const int32_t* src = p.ids_in + static_cast<size_t>(t) * K + k0;
      int v4[4];
      if (vec) {
        const int4 q = __ldg(reinterpret_cast<const int4*>(src));
        v4[0] = q.x; v4[1] = q.y; v4[2] = q.z; v4[3] = q.w;
      } else {
        for (int j = 0; j < 4; ++j) v4[j] = k0 + j < K ? __ldg(src + j) : 0;
      }
      for (int j = 0; j < 4 && k0 + j < K; ++j) {
        const int k = k0 + j, v = v4[j];
        s_ids[k * T + t] = v;
        const bool ok = v >= 0 && v < M;
        bad |= !ok;
        if (v == SERE_ID_NONFINITE) s_err_domain = 1;  // the router saw a non-finite token state
        if (reroute && ok) {
          if (k < s_eff) s_hflag[v] = 1;  // primary set H (rerouting.py:147; Alg. 2 l.467-471)
          else s_sec[v] = 1;              // a secondary candidate (needed unless primary, below)
        }
      }
    }
    if (bad) s_err_id = 1;
  }
  if (stage) mbar_wait(&s_sim_bar, 0);
  const double* simr = stage ? s_sim : p.sim;
  if (reroute && (p.flags & SERE_FLAG_CHECK_SIM)) {  // rerouting.py:115-116 (NaN passes, as there)
    for (int i = tid; i < M * M; i += nthr) {
      const double v = simr[i];
      if (v < 0.0 || v > 1.0) s_err_sim = 1;
    }
  }
  __syncthreads();
  SERE_PHASE(1);
  if (s_err_id || s_err_sim) {
    if (tid == 0) {
      const int code = s_err_domain ? SERE_ERR_DOMAIN
                                    : s_err_id ? (reroute ? SERE_ERR_DIMENSION : SERE_ERR_ROUTING) : SERE_ERR_INPUT;
      if (p.status_dev) *p.status_dev = code;
      if (p.plan) p.plan[P_STATUS] = code;
    }
    return;
  }

  if (reroute) {
    // ---- per-secondary argmax over the primary set (rerouting.py:78-97,152-164). The needed
    // secondaries are the experts of slots >= S that are not primary (rerouting.py:152-156):
    // one 8-lane group per expert u (128 groups: M <= 128 in one round; a group skips u unless
    // it is needed). Every lane issues all its loads of row u first (independent, so they
    // overlap), then compares ascending with strict '>' and the group reduces to the first
    // maximum (larger value, then lower index) -- the ascending strict-'>' scan's answer.
    // The group leader also writes u's class (primary / critical / redirected).
    constexpr int kGl = 8, kVals = 16;
    const int grp = tid / kGl, glane = tid % kGl, ngrp = nthr / kGl;
    for (int base = 0; base < M; base += ngrp) {
      const int e = base + grp;
      const bool in = e < M;
      const bool prim = in && s_hflag[e];
      const bool need = in && !prim && s_sec[e];
      if (glane == 0 && prim) s_cls[e] = SERE_CLASS_PRIMARY;
      if (!__any_sync(0xffffffffu, need)) continue;  // warp-uniform: the warp's 4 groups skip together
      const double* row = simr + static_cast<size_t>(need ? e : 0) * M;
      double bs = -CUDART_INF;
      int bi = -1;
      if (need) {
        for (int v0 = 0; v0 < M; v0 += kGl * kVals) {
          double vals[kVals];
#pragma unroll
          for (int j = 0; j < kVals; ++j) {
            const int v = v0 + glane + kGl * j;
            vals[j] = v < M ? row[v] : 0.0;
          }
#pragma unroll
          for (int j = 0; j < kVals; ++j) {
            const int v = v0 + glane + kGl * j;
            if (v < M && s_hflag[v] && vals[j] > bs) { bs = vals[j]; bi = v; }
          }
        }
      }
#pragma unroll
      for (int off = kGl / 2; off > 0; off >>= 1) {  // within each 8-lane group (xor < 8)
        const double os = __shfl_xor_sync(0xffffffffu, bs, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (oi >= 0 && (bi < 0 || os > bs || (os == bs && oi < bi))) { bs = os; bi = oi; }
      }
      if (need && glane == 0) {
        if (p.rho > 0.0 && bs < p.rho) {
          s_cls[e] = SERE_CLASS_CRITICAL;  // preserved (rerouting.py:160-161)
        } else {
          s_cls[e] = SERE_CLASS_REROUTED;  // redirected (rerouting.py:162-164)
          s_map[e] = bi;
        }
      }
    }
    __syncthreads();
    SERE_PHASE(4);
  }

  // ---- the final table: rewrite the secondary cells (weights are never touched),
  // write it out, and count the cells of each (token block, bank expert) for the align below
  // (shared-memory atomics on u16 pairs). One work item per (token, 4-slot quad): T * ceil(K/4)
  // items keep all threads busy.
  {
    bool bad = false;
    const bool vec_out = vec && (reinterpret_cast<uintptr_t>(p.ids_out) & 15) == 0;
    const bool vec_ws = vec && (reinterpret_cast<uintptr_t>(p.ids_final) & 15) == 0;
    uint32_t* cntb32 = reinterpret_cast<uint32_t*>(s_cntb);
    const int nq = (K + 3) >> 2;
    for (int it = tid; it < T * nq; it += nthr) {
      const int t = it / nq, k0 = (it - t * nq) * 4;
      const int tbE = (t / kTokBlk) * Et;
      int v4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = k0 + j;
        v4[j] = 0;
        if (k < K) {
          int e = s_ids[k * T + t];
          if (reroute && k >= S && (s_cls[e] & SERE_CLASS_REROUTED)) {
            e = s_map[e];
            bad |= (e < 0 || e >= M);  // reference NaN quirk: a secondary mapped to -1
          }
          v4[j] = e;
          if (align) {
            const int el = local_of(e);
            if (el >= 0) {
              const int idx = tbE + el;
              atomicAdd(cntb32 + (idx >> 1), 1u << (16 * (idx & 1)));
            }
          }
        }
      }
      if (reroute && p.ids_out) {
        int32_t* dst = p.ids_out + static_cast<size_t>(t) * K + k0;
        if (vec_out) *reinterpret_cast<int4*>(dst) = make_int4(v4[0], v4[1], v4[2], v4[3]);
        else for (int j = 0; j < 4 && k0 + j < K; ++j) dst[j] = v4[j];
      }
      if (align) {
        int32_t* dst = p.ids_final + static_cast<size_t>(t) * K + k0;
        if (vec_ws) *reinterpret_cast<int4*>(dst) = make_int4(v4[0], v4[1], v4[2], v4[3]);
        else for (int j = 0; j < 4 && k0 + j < K; ++j) dst[j] = v4[j];
      }
    }
    if (bad) s_err_route = 1;
  }
  if (reroute) {
    if (p.expert_class)
      for (int e = tid; e < M; e += nthr) p.expert_class[e] = s_cls[e];
    if (p.reroute_map)
      for (int e = tid; e < M; e += nthr) p.reroute_map[e] = s_map[e];
    if (warp == 0) {  // final_active = primary | critical, ascending (rerouting.py:168-169)
      int base = 0;
      for (int c0 = 0; c0 < M; c0 += 32) {
        const int e = c0 + lane;
        const bool act = e < M && (s_cls[e] & (SERE_CLASS_PRIMARY | SERE_CLASS_CRITICAL));
        const unsigned m = __ballot_sync(0xffffffffu, act);
        if (act && p.active_list) p.active_list[base + __popc(m & ((1u << lane) - 1u))] = e;
        base += __popc(m);
      }
      if (lane == 0) {
        if (p.n_active) *p.n_active = base;
        if (p.plan) p.plan[P_NACTIVE] = base;
      }
    }
  }
  __syncthreads();
  SERE_PHASE(5);

  if (!align) {
    if (tid == 0 && p.status_dev) *p.status_dev = SERE_OK;
    return;
  }
  // the rewritten table may hold -1 (reference NaN quirk at rho == 0): layer_forward then
  // raises RoutingError (moe.py:299-300)
  if (s_err_route) {
    if (tid == 0) {
      if (p.status_dev) *p.status_dev = SERE_ERR_ROUTING;
      p.plan[P_STATUS] = SERE_ERR_ROUTING;
    }
    return;
  }

  // ================================================================ count/align
  // Rows of a group are ordered by (token block of 32, slot k, token): deterministic and
  // computable without sorting. Here: block counts -> exclusive prefixes over blocks and
  // totals per bank expert, the group layout, the FFN schedule. The rank of each cell inside
  // its token block, the permutation (slot_row / row_token) and the gather of the token rows
  // are the permute kernel's (many CTAs; layout.cu), which reads the prefixes from
  // `blk_prefix` and the groups' first rows from the plan.
  for (int e = tid; e < Et; e += nthr) {
    if (e < m_loc) {
      int run = 0;
      for (int tb = 0; tb < TB; ++tb) {
        const int v = s_cntb[tb * Et + e];
        s_cntb[tb * Et + e] = static_cast<uint16_t>(run);
        run += v;
      }
      s_cnt[e] = run;
    } else {
      s_cnt[e] = T;  // shared experts: every token (moe.py:308-309)
    }
  }
  __syncthreads();
  SERE_PHASE(7);

  const PlanOffsets po = plan_offsets(Et);
  int32_t* plan = p.plan;
  // group layout: groups = bank experts with cells (ascending) then shared experts; each
  // padded to 16 rows. One warp per chunk of 32 experts scans in parallel, then every
  // chunk adds the totals of the chunks before it.
  __shared__ int s_tot[2][40];
  __shared__ int s_ngroups;
  const int nch = (Et + 31) / 32;
  {
    const int e = warp * 32 + lane;
    int cnt = 0, pad = 0, gi = 0, r_in = 0;
    bool act = false;
    if (warp < nch) {
      cnt = e < Et ? s_cnt[e] : 0;
      act = cnt > 0;
      const unsigned m = __ballot_sync(0xffffffffu, act);
      gi = __popc(m & ((1u << lane) - 1u));
      pad = round_up(cnt, kRowAlign);
      r_in = warp_incl_scan(pad);
      if (lane == 31) {
        s_tot[0][warp] = __popc(m);
        s_tot[1][warp] = r_in;
      }
    }
    __syncthreads();
    if (warp < nch) {
      int gb = 0, rb = 0;
      for (int w = 0; w < warp; ++w) { gb += s_tot[0][w]; rb += s_tot[1][w]; }
      if (e < Et) {
        const int row0 = act ? rb + r_in - pad : -1;
        if (act) {
          plan[po.group_expert + gb + gi] = e;
          plan[po.group_row0 + gb + gi] = row0;
          plan[po.group_rows + gb + gi] = cnt;
          s_gpad[gb + gi] = pad;
        }
        s_row0[e] = row0;
        plan[po.counts + e] = cnt;
        plan[po.erow0 + e] = row0;
      }
      if (warp == nch - 1 && lane == 0) {
        const int g_tot = gb + s_tot[0][warp], r_tot = rb + s_tot[1][warp];
        s_ngroups = g_tot;
        plan[P_NGROUPS] = g_tot;
        plan[P_TOTAL_ROWS] = r_tot;
        plan[P_TICKET] = 0;
        plan[P_DONE] = 0;
        if (!reroute) plan[P_NACTIVE] = g_tot - p.n_shared;
      }
    }
  }
  __syncthreads();
  SERE_PHASE(10);
  // schedule order of the fused FFN: padded rows descending, ties by group index (a
  // unit's cost grows with its column count, so this is longest-processing-time first)
  const int G = s_ngroups;
  __shared__ int s_ugu[kMaxGroupsSched], s_udn[kMaxGroupsSched];  // work units per schedule position
  for (int g = tid; g < G; g += nthr) {
    const int key = s_gpad[g];
    int rank = 0;
#pragma unroll 8
    for (int j = 0; j < G; ++j) {
      const int kj = s_gpad[j];
      rank += (kj > key) | ((kj == key) & (j < g));
    }
    s_sched[rank] = g;
    s_ugu[rank] = group_units_gu(key, p.tiles_gu);
    s_udn[rank] = group_units_dn(key, p.tiles_dn, p.ksplit_dn);
    plan[po.sched + rank] = g;
    plan[po.dep + g] = 0;
  }
  __syncthreads();
  SERE_PHASE(11);
  if (warp < nwarps - 1) {
    // block prefixes out for the permute kernel (coalesced 32-bit words); padding rows of every
    // group carry no token (their FFN columns are never read): row_token = -1
    const int nthr2 = nthr - 32;
    for (int i = tid; i < round_up(TB * Et, 2) / 2; i += nthr2)
      reinterpret_cast<uint32_t*>(p.blk_prefix)[i] = reinterpret_cast<const uint32_t*>(s_cntb)[i];
    for (int i = tid; i < Et * kRowAlign; i += nthr2) {
      const int e = i / kRowAlign, r = s_row0[e] + s_cnt[e] + (i - e * kRowAlign);
      if (s_row0[e] >= 0 && r < s_row0[e] + round_up(s_cnt[e], kRowAlign)) p.row_token[r] = -1;
    }
  } else {  // unit prefixes over the schedule order (one warp)
    // A small active set leaves SMs idle for the whole gate/up phase (Qwen3 T=128 after SERE:
    // 31 groups x 3 two-block units = 93 units for 148 SMs, every group's h complete only at
    // the end of it). Then the first groups in schedule order (the largest) take one-block
    // gate/up units while the total still fits one wave: they finish in half the time, and
    // their down units (first in the down order) fill the SMs that free up. Greedy in schedule
    // order: group i converts iff tot + D(i-1) < ffn_ctas and tot + D(i) <= ffn_ctas, D = the
    // inclusive prefix of the conversions' extra units (>= 0, so the first refusal ends it).
    int tot = 0;
    for (int c0 = 0; c0 < G; c0 += 32) tot += c0 + lane < G ? s_ugu[c0 + lane] : 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
    int gu_base = 0, dn_base = 0, d_base = 0;
    for (int c0 = 0; c0 < G; c0 += 32) {
      const int i = c0 + lane;
      int ugu = 0, udn = 0, dlt = 0;
      if (i < G) {
        ugu = s_ugu[i];
        udn = s_udn[i];
        dlt = group_units_gu(s_gpad[s_sched[i]], p.tiles_gu, 1) - ugu;
      }
      const int d_in = d_base + warp_incl_scan(dlt);
      const bool one = i < G && tot + d_in - dlt < p.ffn_ctas && tot + d_in <= p.ffn_ctas;
      d_base = __shfl_sync(0xffffffffu, d_in, 31);
      if (one) ugu += dlt;
      if (i < G) plan[po.mw_gu + i] = one ? 1 : kMwGuMax;
      const int gu_in = warp_incl_scan(ugu), dn_in = warp_incl_scan(udn);
      if (i < G) {
        plan[po.unit_off_gu + i] = gu_base + gu_in - ugu;
        plan[po.unit_off_dn + i] = dn_base + dn_in - udn;
      }
      gu_base += __shfl_sync(0xffffffffu, gu_in, 31);
      dn_base += __shfl_sync(0xffffffffu, dn_in, 31);
    }
    if (lane == 0) {
      plan[P_UNITS_GU] = gu_base;
      plan[P_UNITS_DN] = dn_base;
      plan[po.unit_off_gu + G] = gu_base;
      plan[po.unit_off_dn + G] = dn_base;
      plan[P_STATUS] = SERE_OK;
      if (p.status_dev) *p.status_dev = SERE_OK;
    }
  }
  SERE_PHASE(8);
}

cudaError_t launch_reroute_align(const AlignParams& p, cudaStream_t stream) {
  AlignParams q = p;
  const int Et = p.m_local + p.n_shared;
  q.stage_sim = (p.mode & MODE_REROUTE) && p.sim != nullptr && (reinterpret_cast<uintptr_t>(p.sim) & 15) == 0 &&
                (static_cast<size_t>(p.M) * p.M * 8) % 16 == 0 && align_smem_total(p.T, p.K, p.M, Et, true) <= kAlignSmemCap;
  const size_t smem = align_smem_total(p.T, p.K, p.M, Et, q.stage_sim != 0);
  static SmemAttrCache attr;  // dynamic + ~4 KB static may cross the 48 KB default
  if (cudaError_t e = ensure_smem_attr(reroute_align_kernel, smem, attr, 32 * 1024); e != cudaSuccess) return e;
  return launch_pdl((g_pdl & PDL_ALIGN) != 0, reroute_align_kernel, dim3(1), dim3(kAlignThreads), smem, stream, q);
}

size_t reroute_align_smem(int T, int K, int M, int Et) { return align_smem_bytes(T, K, M, Et); }

}  // namespace sere
