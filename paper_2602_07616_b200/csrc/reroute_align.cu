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
//      to 16 rows; a STABLE (token, slot)-ordered rank inside each group from a
//      two-pass warp __match_any_sync count, giving slot_row[t,k] and the inverse
//      row_token[row]; work-unit prefixes for both grouped GEMMs.
// Everything is integer / fp64-compare work on <= 16K cells: latency-bound, so a
// single CTA with no global round trips between phases is the fastest shape.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "../../include/sere_b200.h"
#include "params.cuh"
#include "plan.cuh"
#include "ptx.cuh"

namespace sere {

constexpr int kAlignThreads = 1024;
constexpr int kAlignWarps = kAlignThreads / 32;

// M = global expert count (ids, sim, classes); Et = local groups (bank experts + shared)
__host__ __device__ inline size_t align_smem_bytes(int T, int K, int M, int Et) {
  const int TK = T * K, MW = (M + 31) / 32;
  size_t b = 0;
  b += static_cast<size_t>(TK) * 4;          // s_ids
  b += static_cast<size_t>(MW) * 4 * 2;      // s_h, s_need
  b += static_cast<size_t>(M) * 4 * 2;       // s_map, s_list
  b += static_cast<size_t>(Et) * 4 * 3;      // s_cnt, s_row0, s_gidx
  b += static_cast<size_t>(round_up(M, 4));  // s_cls
  b += static_cast<size_t>(kAlignWarps) * Et * 2;  // s_wc
  return round_up(static_cast<int>(b), 16);
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
  const int TK = T * K, MW = (M + 31) / 32;
  const int e_lo = p.e_lo, m_loc = p.m_local, Et = m_loc + p.n_shared;  // expert-parallel ownership
  int32_t* s_ids = reinterpret_cast<int32_t*>(smem);
  uint32_t* s_h = reinterpret_cast<uint32_t*>(s_ids + TK);
  uint32_t* s_need = s_h + MW;
  int32_t* s_map = reinterpret_cast<int32_t*>(s_need + MW);
  int32_t* s_list = s_map + M;  // compact list of needed secondaries
  int32_t* s_cnt = s_list + M;
  int32_t* s_row0 = s_cnt + Et;
  int32_t* s_gidx = s_row0 + Et;
  uint8_t* s_cls = reinterpret_cast<uint8_t*>(s_gidx + Et);
  uint16_t* s_wc = reinterpret_cast<uint16_t*>(s_cls + round_up(M, 4));
  __shared__ int s_err_id, s_err_sim, s_err_route;

  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  const bool reroute = (p.mode & MODE_REROUTE) != 0;
  const bool align = (p.mode & MODE_ALIGN) != 0;

  if (tid == 0) { s_err_id = 0; s_err_sim = 0; s_err_route = 0; }
  for (int i = tid; i < MW; i += nthr) { s_h[i] = 0u; s_need[i] = 0u; }
  for (int e = tid; e < M; e += nthr) { s_map[e] = -1; s_cls[e] = 0; }
  for (int e = tid; e < Et; e += nthr) s_cnt[e] = 0;
  __syncthreads();

  // ---- load + validate ids (rerouting.py:111-114 / moe.py:299-300)
  for (int c = tid; c < TK; c += nthr) {
    const int v = p.ids_in[c];
    s_ids[c] = v;
    if (v < 0 || v >= M) s_err_id = 1;
  }
  if (reroute && (p.flags & SERE_FLAG_CHECK_SIM)) {  // rerouting.py:115-116 (NaN passes, as there)
    for (int i = tid; i < M * M; i += nthr) {
      const double s = p.sim[i];
      if (s < 0.0 || s > 1.0) s_err_sim = 1;
    }
  }
  __syncthreads();
  if (s_err_id || s_err_sim) {
    if (tid == 0) {
      const int code = s_err_id ? (reroute ? SERE_ERR_DIMENSION : SERE_ERR_ROUTING) : SERE_ERR_INPUT;
      if (p.status_dev) *p.status_dev = code;
      if (p.plan) p.plan[P_STATUS] = code;
    }
    return;
  }

  if (reroute) {
    // ---- primary mask H (rerouting.py:147; Alg. 2).  S == K: identity, all primary.
    const int s_eff = S < K ? S : K;
    for (int c = tid; c < TK; c += nthr) {
      if ((c % K) < s_eff) {
        const int e = s_ids[c];
        atomicOr(&s_h[e >> 5], 1u << (e & 31));
      }
    }
    __syncthreads();
    // ---- distinct secondary experts of slots >= S that are not primary (rerouting.py:152-156)
    if (S < K) {
      for (int c = tid; c < TK; c += nthr) {
        if ((c % K) >= S) {
          const int e = s_ids[c];
          if (!((s_h[e >> 5] >> (e & 31)) & 1u)) atomicOr(&s_need[e >> 5], 1u << (e & 31));
        }
      }
    }
    __syncthreads();
    // ---- compact list of the needed secondaries (ascending)
    __shared__ int s_nneed;
    if (warp == 0) {
      int base = 0;
      for (int c0 = 0; c0 < M; c0 += 32) {
        const int e = c0 + lane;
        const bool nd = e < M && ((s_need[e >> 5] >> (e & 31)) & 1u);
        const unsigned m = __ballot_sync(0xffffffffu, nd);
        if (nd) s_list[base + __popc(m & ((1u << lane) - 1u))] = e;
        base += __popc(m);
      }
      if (lane == 0) s_nneed = base;
    }
    __syncthreads();
    // ---- per-secondary argmax over the primary set (rerouting.py:78-97,157-164): one 16-lane
    // group per secondary u; every lane first issues all its loads of row u (independent, so
    // they overlap), then compares ascending with strict '>' and the group reduces to the
    // first maximum (larger value, then lower index).
    const int n_need = s_nneed;
    const int grp = tid >> 4, glane = tid & 15, ngrp = nthr >> 4;
    for (int base = 0; base < n_need; base += ngrp) {
      const int li = base + grp;
      const bool have = li < n_need;
      const int e = have ? s_list[li] : 0;
      const double* row = p.sim + static_cast<size_t>(e) * M;
      double bs = -CUDART_INF;
      int bi = -1;
      if (have) {
        for (int v0 = 0; v0 < M; v0 += 16 * 8) {
          double vals[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int v = v0 + glane + 16 * j;
            vals[j] = v < M ? __ldg(row + v) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int v = v0 + glane + 16 * j;
            if (v < M && ((s_h[v >> 5] >> (v & 31)) & 1u) && vals[j] > bs) { bs = vals[j]; bi = v; }
          }
        }
      }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, off, 16);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off, 16);
        if (oi >= 0 && (bi < 0 || os > bs || (os == bs && oi < bi))) { bs = os; bi = oi; }
      }
      if (have && glane == 0) {
        if (p.rho > 0.0 && bs < p.rho) {
          s_cls[e] = SERE_CLASS_CRITICAL;  // preserved (rerouting.py:160-161)
        } else {
          s_cls[e] = SERE_CLASS_REROUTED;  // redirected (rerouting.py:162-164)
          s_map[e] = bi;
        }
      }
    }
    for (int e = tid; e < M; e += nthr)
      if ((s_h[e >> 5] >> (e & 31)) & 1u) s_cls[e] = SERE_CLASS_PRIMARY;
    __syncthreads();
    // ---- rewrite the secondary cells (weights are never touched)
    if (S < K) {
      for (int c = tid; c < TK; c += nthr) {
        if ((c % K) >= S) {
          const int e = s_ids[c];
          if (s_cls[e] & SERE_CLASS_REROUTED) s_ids[c] = s_map[e];
        }
      }
    }
    __syncthreads();
    // ---- outputs
    if (p.ids_out)
      for (int c = tid; c < TK; c += nthr) p.ids_out[c] = s_ids[c];
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

  if (!align) {
    if (tid == 0 && p.status_dev) *p.status_dev = SERE_OK;
    return;
  }

  // ================================================================ count/align
  // the rewritten table may hold -1 (reference NaN quirk at rho == 0): layer_forward
  // then raises RoutingError (moe.py:299-300)
  if (reroute) {
    for (int c = tid; c < TK; c += nthr) {
      const int v = s_ids[c];
      if (v < 0 || v >= M) s_err_route = 1;
    }
    __syncthreads();
    if (s_err_route) {
      if (tid == 0) {
        if (p.status_dev) *p.status_dev = SERE_ERR_ROUTING;
        p.plan[P_STATUS] = SERE_ERR_ROUTING;
      }
      return;
    }
  }
  // cells routed to experts this bank does not own (expert parallelism) take no row
  auto local_of = [&](int e) { return (e >= e_lo && e < e_lo + m_loc) ? e - e_lo : -1; };
  for (int c = tid; c < TK; c += nthr) {
    const int el = local_of(s_ids[c]);
    if (el >= 0) atomicAdd(&s_cnt[el], 1);
  }
  for (int s = tid; s < p.n_shared; s += nthr) s_cnt[m_loc + s] = T;
  __syncthreads();

  const PlanOffsets po = plan_offsets(Et);
  int32_t* plan = p.plan;
  if (warp == 0) {
    int g_base = 0, row_base = 0, ugu_base = 0, udn_base = 0;
    for (int c0 = 0; c0 < Et; c0 += 32) {
      const int e = c0 + lane;
      const int cnt = e < Et ? s_cnt[e] : 0;
      const bool act = cnt > 0;
      const unsigned m = __ballot_sync(0xffffffffu, act);
      const int gi = g_base + __popc(m & ((1u << lane) - 1u));
      const int pad = round_up(cnt, kRowAlign);
      const int ncb = (pad + kColBlock - 1) / kColBlock;
      const int ugu = p.tiles_gu * ncb, udn = p.units_dn_per * ncb;
      const int r_incl = warp_incl_scan(pad);
      const int gu_incl = warp_incl_scan(ugu);
      const int dn_incl = warp_incl_scan(udn);
      if (e < Et) {
        if (act) {
          plan[po.group_expert + gi] = e;
          plan[po.group_row0 + gi] = row_base + r_incl - pad;
          plan[po.group_rows + gi] = cnt;
          plan[po.unit_off_gu + gi] = ugu_base + gu_incl - ugu;
          plan[po.unit_off_dn + gi] = udn_base + dn_incl - udn;
          s_row0[e] = row_base + r_incl - pad;
          s_gidx[e] = gi;
        } else {
          s_row0[e] = -1;
          s_gidx[e] = -1;
        }
        plan[po.counts + e] = cnt;
      }
      g_base += __popc(m);
      row_base += __shfl_sync(0xffffffffu, r_incl, 31);
      ugu_base += __shfl_sync(0xffffffffu, gu_incl, 31);
      udn_base += __shfl_sync(0xffffffffu, dn_incl, 31);
    }
    if (lane == 0) {
      plan[P_NGROUPS] = g_base;
      plan[P_TOTAL_ROWS] = row_base;
      plan[P_UNITS_GU] = ugu_base;
      plan[P_UNITS_DN] = udn_base;
      plan[po.unit_off_gu + g_base] = ugu_base;
      plan[po.unit_off_dn + g_base] = udn_base;
      if (!reroute) plan[P_NACTIVE] = g_base - (p.n_shared > 0 ? p.n_shared : 0);
    }
  }
  // zero the per-warp per-expert counters
  for (int i = tid; i < nwarps * Et; i += nthr) s_wc[i] = 0;
  __syncthreads();

  // ---- stable ranks: warp w owns cells [w*L, (w+1)*L) in (token, slot) order
  const int L = (TK + nwarps - 1) / nwarps;
  const int c_lo = warp * L, c_hi = min(TK, c_lo + L);
  uint16_t* wc = s_wc + warp * Et;
  for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
    const int c = c0 + lane;
    const int el = c < c_hi ? local_of(s_ids[c]) : -1;
    const int e = el >= 0 ? el : -1 - lane;  // unique sentinel for idle / foreign cells
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    if (el >= 0 && lane == __ffs(peers) - 1) wc[e] += static_cast<uint16_t>(__popc(peers));
    __syncwarp();
  }
  __syncthreads();
  for (int e = tid; e < Et; e += nthr) {  // exclusive prefix over warps
    int run = 0;
    for (int w = 0; w < nwarps; ++w) {
      const int v = s_wc[w * Et + e];
      s_wc[w * Et + e] = static_cast<uint16_t>(run);
      run += v;
    }
  }
  __syncthreads();
  for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
    const int c = c0 + lane;
    const int el = c < c_hi ? local_of(s_ids[c]) : -1;
    const int e = el >= 0 ? el : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    int base = 0;
    if (el >= 0) base = wc[e];
    __syncwarp();
    if (el >= 0) {
      const int row = s_row0[e] + base + __popc(peers & ((1u << lane) - 1u));
      p.slot_row[c] = row;
      p.row_token[row] = c / K;
      if (lane == __ffs(peers) - 1) wc[e] = static_cast<uint16_t>(base + __popc(peers));
    } else if (c < c_hi) {
      p.slot_row[c] = -1;  // owned by another rank: the combine skips it
    }
    __syncwarp();
  }
  // shared experts: every token, in token order (moe.py:308-309)
  for (int i = tid; i < T * p.n_shared; i += nthr) {
    const int t = i / p.n_shared, s = i % p.n_shared;
    const int row = s_row0[m_loc + s] + t;
    p.slot_row[TK + i] = row;
    p.row_token[row] = t;
  }
  // padding rows of each group
  for (int e = warp; e < Et; e += nwarps) {
    const int cnt = s_cnt[e];
    if (cnt == 0) continue;
    const int pad = round_up(cnt, kRowAlign);
    if (lane < pad - cnt) p.row_token[s_row0[e] + cnt + lane] = -1;
  }
  if (tid == 0) {
    plan[P_STATUS] = SERE_OK;
    if (p.status_dev) *p.status_dev = SERE_OK;
  }
}

cudaError_t launch_reroute_align(const AlignParams& p, cudaStream_t stream) {
  const size_t smem = align_smem_bytes(p.T, p.K, p.M, p.m_local + p.n_shared);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(reroute_align_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  reroute_align_kernel<<<1, kAlignThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

size_t reroute_align_smem(int T, int K, int M, int Et) { return align_smem_bytes(T, K, M, Et); }

}  // namespace sere
