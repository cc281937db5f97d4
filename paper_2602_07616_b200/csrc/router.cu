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

#include "../../include/sere_b200.h"
#include "params.cuh"
#include "ptx.cuh"
#include "rowops.cuh"

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
  __shared__ int s_bad[kTok];
  if (threadIdx.x < kTok) s_bad[threadIdx.x] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < kTok * M; i += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < KS; ++q) s += s_part[q * kTok * M + i];
    if (bias) s += bias[i % M];
    if (!isfinite(s)) s_bad[i / M] = 1;  // non-finite token state -> SERE_ID_NONFINITE (DomainError)
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
      if (lane == 0) ids[static_cast<size_t>(t) * K + r] = s_bad[warp] ? SERE_ID_NONFINITE : bi;
      __syncwarp();
      if (bi >= 0 && lane == (bi & 31)) lg[bi] = -CUDART_INF_F;  // remove the pick (ties resolved on index above)
      __syncwarp();
    }
    if (lane == 0) {
      float den = 0.f;
      for (int r = 0; r < K; ++r) { sel_val[r] = expf(sel_val[r] - top); den += sel_val[r]; }
      for (int r = 0; r < K; ++r) weights[static_cast<size_t>(t) * K + r] = sel_val[r] / den;
    }
  }
}

// Fast path (M % 8 == 0, M <= 256, K <= 32, d_h % 8 == 0): one thread-block CLUSTER per
// 16-token tile, its S CTAs split d_h into S chunks of kc. Each CTA stages its x rows and
// W_r^T rows with cp.async (one round trip), runs mma.sync m16n8k16 (bf16 in,
// fp32 accumulate) into a [16][M] partial in its own shared memory; after a cluster
// barrier the CTAs exchange row slices of their partials over distributed shared memory
// (bulk copies), so that each CTA owns 16/S tokens: it sums their S partials in split
// order (deterministic: identical logits every launch), adds the bias and selects the
// top K by rank + softmax. No global partials, no tickets, no serial warp argmax.
constexpr int kRcTok = 16, kRcPad = 8, kRcThreads = 256, kRcMaxSplit = 8;

struct RouteGeom {
  int S, kc;
  size_t smem;
};

__host__ __device__ inline RouteGeom route_geom(int d_h, int M) {
  RouteGeom g;
#ifndef SERE_ROUTE_KCHUNK
#define SERE_ROUTE_KCHUNK 256  // d_h per split CTA (8 splits at d_h = 2048)
#endif
  int S = (d_h + SERE_ROUTE_KCHUNK - 1) / SERE_ROUTE_KCHUNK;
  if (S > kRcMaxSplit) S = kRcMaxSplit;
  if (S < 1) S = 1;
  g.kc = round_up((d_h + S - 1) / S, 16);
  g.S = (d_h + g.kc - 1) / g.kc;
  g.smem = static_cast<size_t>(kRcTok + M) * (g.kc + kRcPad) * 2 + static_cast<size_t>(kRcTok) * M * 4;
  return g;
}

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// bulk copy of this CTA's shared memory into another CTA's shared memory (same cluster);
// completion is counted on the destination CTA's mbarrier
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst_cluster, const void* src, uint32_t bytes,
                                               uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(smem_u32(src)), "r"(bytes), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

long long* g_route_dbg = nullptr;  // sere_debug_set_route_clocks: per-CTA phase clock64 [cta][8]
#define RC_PROBE(i) do { if (dbg && threadIdx.x == 0) dbg[(blockIdx.x * gridDim.y + blockIdx.y) * 8 + (i)] = clock64(); } while (0)

// Split-K partials -> logits -> top-K + softmax, shared by both router kernels: the tile's
// tokens are spread over the cluster (CTA q owns tokens [q*tpc, (q+1)*tpc)); every CTA
// bulk-copies each owner its rows of this split's partial over distributed shared memory
// (S-1 copies per CTA, into the owner's idle staging buffer `rsm`), then every CTA reduces
// and ranks its own tokens -- the whole cluster works on the top-K.
__device__ __forceinline__ void route_finish(uint8_t* rsm, float* part, uint64_t& s_gather, int S, uint32_t split,
                                             int t0, int nt_valid, int M, int K, const float* __restrict__ bias,
                                             int32_t* __restrict__ ids, float* __restrict__ weights,
                                             float* __restrict__ logits_out, long long* dbg, const EpPeers& ep,
                                             int ntok = kRcTok) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tpc = (ntok + S - 1) / S;
  const int my_t0 = static_cast<int>(split) * tpc;
  const int my_rows = max(0, min(tpc, nt_valid - my_t0));
  float* gath = reinterpret_cast<float*>(rsm);  // [S][tpc][M] (own slot unused)
  __shared__ int s_nonfinite[kRcTok];
  for (int r = tid; r < kRcTok; r += blockDim.x) s_nonfinite[r] = 0;
  fence_proxy_async_smem();  // generic smem accesses above before the async-proxy copies below
  if (tid == 0 && my_rows > 0 && S > 1) mbar_arrive_expect_tx(&s_gather, static_cast<uint32_t>(my_rows * M * 4 * (S - 1)));
  cluster_sync_all();  // partials written, barriers armed, staging buffers no longer read
  RC_PROBE(4);
  if (tid < S && tid != static_cast<int>(split)) {
    const int d = tid;
    const int rows_d = max(0, min(tpc, nt_valid - d * tpc));
    if (rows_d > 0)
      bulk_s2cluster(mapa_shared(gath + (static_cast<int>(split) * tpc) * M, d), part + d * tpc * M,
                     static_cast<uint32_t>(rows_d * M * 4), mapa_shared(&s_gather, d));
  }
  if (my_rows > 0) {
    if (S > 1) mbar_wait(&s_gather, 0);
    RC_PROBE(6);
    float* lgt = part + my_t0 * M;  // my tokens' logits, summed in place
    for (int i = tid; i < my_rows * M; i += blockDim.x) {
      const int r = i / M;
      const float b = bias ? bias[i % M] : 0.f;  // shared memory (tcgen05 path) or global
      float pv[kRcMaxSplit];
#pragma unroll
      for (int q = 0; q < kRcMaxSplit; ++q)
        pv[q] = q >= S ? 0.f : (q == static_cast<int>(split) ? lgt[i] : gath[(q * tpc + r) * M + (i % M)]);
      float acc_l = 0.f;
#pragma unroll
      for (int q = 0; q < kRcMaxSplit; ++q)
        if (q < S) acc_l += pv[q];  // split order
      if (bias) acc_l += b;
      if (logits_out) logits_out[static_cast<size_t>(t0 + my_t0) * M + i] = acc_l;
      // a non-finite logit (non-finite token state: the reference raises DomainError,
      // moe.py:274-275) flags its token; NaN is ranked as -inf so the top-K below stays a
      // well-defined permutation
      if (!isfinite(acc_l)) {
        s_nonfinite[i / M] = 1;
        if (isnan(acc_l)) acc_l = -INFINITY;
      }
      lgt[i] = acc_l;
    }
    __syncthreads();
    RC_PROBE(7);
    // top-K by rank: candidate v of token r is selected at position rank(v) = #{u : l_u > l_v
    // or (l_u == l_v and u < v)} < K -- descending, ties to the lower index (moe.py:260)
    float* sel_v = gath;                                        // [my_rows][K] (gath slot of this CTA)
    int* sel_i = reinterpret_cast<int*>(gath + my_rows * K);  // [my_rows][K]
    for (int i = tid; i < my_rows * M; i += blockDim.x) {
      const int r = i / M, v = i % M;
      const float lv = lgt[i];
      const float4* row = reinterpret_cast<const float4*>(lgt + r * M);
      int rank = 0;
#pragma unroll 8
      for (int u4 = 0; u4 < M / 4; ++u4) {
        const float4 q4 = row[u4];
        const int u = u4 * 4;
        rank += (q4.x > lv) | ((q4.x == lv) & (u < v));
        rank += (q4.y > lv) | ((q4.y == lv) & (u + 1 < v));
        rank += (q4.z > lv) | ((q4.z == lv) & (u + 2 < v));
        rank += (q4.w > lv) | ((q4.w == lv) & (u + 3 < v));
      }
      if (rank < K) { sel_v[r * K + rank] = lv; sel_i[r * K + rank] = v; }
    }
    __syncthreads();
    for (int r = warp; r < my_rows; r += blockDim.x / 32) {  // softmax over the K picks (moe.py:261-264)
      const float top = sel_v[r * K];
      float den = 0.f;
      for (int k = 0; k < K; ++k) den += __expf(sel_v[r * K + k] - top);
      if (lane < K) {
        const size_t o = static_cast<size_t>(t0 + my_t0 + r) * K + lane;
        const bool bad = s_nonfinite[r] != 0;
        const int id = bad ? SERE_ID_NONFINITE : sel_i[r * K + lane];  // -> DomainError downstream
        const float wv = __expf(sel_v[r * K + lane] - top) / den;
        if (ep.world == 0) {
          ids[o] = id;
          weights[o] = wv;
        } else if (!ep_aborted(ep)) {  // expert parallel: this rank's rows of every rank's gathered table (NVLink stores)
          const size_t og = static_cast<size_t>(ep.t0) * K + o;
          for (int p = 0; p < ep.world; ++p) {
            ep.ids_all[p][og] = id;
            ep.w_all[p][og] = wv;
          }
          __threadfence_system();  // peer stores visible before the barrier kernel's release
        }
      }
    }
  }
  cluster_sync_relaxed();  // no CTA leaves before the copies out of its shared memory landed
  RC_PROBE(5);
}

// expert parallel with the fused barrier: every CTA counts itself out after its peer stores;
// the last one arrives (its rows and every other CTA's are published under a new epoch)
__device__ __forceinline__ void route_ep_arrive(const EpPeers& ep) {
  if (ep.world == 0 || ep.epoch == nullptr || threadIdx.x != 0) return;
  __threadfence_system();
  const int total = static_cast<int>(gridDim.x * gridDim.y);
  if (atomicAdd(ep.arrivals, 1) == total - 1) {
    *ep.arrivals = 0;
    EpSync s{};
    s.world = ep.world;
    s.rank = ep.rank;
    for (int r = 0; r < kMaxEpRanks; ++r) s.flags[r] = ep.flags[r];
    s.epoch = ep.epoch;
    ep_arrive(s);
  }
}

__global__ void __launch_bounds__(kRcThreads) route_cluster_kernel(const __nv_bfloat16* __restrict__ x,
                                                                   const __nv_bfloat16* __restrict__ wr,
                                                                   const float* __restrict__ bias, int T, int d_h,
                                                                   int M, int K, int kc,
                                                                   int32_t* __restrict__ ids,
                                                                   float* __restrict__ weights,
                                                                   float* __restrict__ logits_out, long long* dbg,
                                                                   const EpPeers ep) {
  extern __shared__ __align__(16) uint8_t rsm[];
  const int LD = kc + kRcPad;  // padded row (bank-conflict-free fragment loads)
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(rsm);  // [16][LD]
  __nv_bfloat16* wt = xs + kRcTok * LD;                       // [M][LD]  (W_r transposed: expert-major)
  float* part = reinterpret_cast<float*>(wt + M * LD);         // [16][M] this split's partial logits
  __shared__ __align__(8) uint64_t s_bar, s_gather;
  const int S = gridDim.y;
  const uint32_t split = cluster_ctarank();
  const int t0 = blockIdx.x * kRcTok, k0 = static_cast<int>(split) * kc;
  const int kn = max(0, min(kc, d_h - k0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt_valid = min(kRcTok, T - t0);
  const int cpr = kc / 8;
  if (tid == 0) { mbar_init(&s_bar, 1); mbar_init(&s_gather, 1); fence_mbar_init(); }
  RC_PROBE(0);
  for (int i = tid; i < kRcTok * cpr; i += blockDim.x) {  // zero the tails (short K chunk, missing tokens)
    const int t = i / cpr, k = (i % cpr) * 8;
    if (t >= nt_valid || k >= kn) *reinterpret_cast<uint4*>(xs + t * LD + k) = make_uint4(0u, 0u, 0u, 0u);
  }
  if (kn < kc)
    for (int i = tid; i < M * cpr; i += blockDim.x) {
      const int e = i / cpr, k = (i % cpr) * 8;
      if (k >= kn) *reinterpret_cast<uint4*>(wt + e * LD + k) = make_uint4(0u, 0u, 0u, 0u);
    }
  __syncthreads();
  RC_PROBE(1);
  // stage x rows and W_r^T rows of this K chunk with 16-B cp.async (LDGSTS): every thread
  // keeps all its copies in flight, one memory round trip (small bulk copies would
  // serialise in the TMA unit: ~150 of 512 B each)
  {
    const int cpn = kn / 8;  // 16-B chunks per row in this K chunk
    // router weights are static: stage them before waiting on the previous kernel (PDL)
    for (int i = tid; i < M * cpn; i += blockDim.x) {
      const int r = i / cpn, c = (i % cpn) * 8;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(wt + r * LD + c)),
                   "l"(wr + static_cast<size_t>(r) * d_h + k0 + c)
                   : "memory");
    }
    pdl_wait();  // x = the previous layer's RMSNorm output; ids/weights are read by its kernels
    pdl_trigger();
    for (int i = tid; i < nt_valid * cpn; i += blockDim.x) {
      const int r = i / cpn, c = (i % cpn) * 8;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(xs + r * LD + c)),
                   "l"(x + static_cast<size_t>(t0 + r) * d_h + k0 + c)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  RC_PROBE(2);
  }
  // MMA: the 16 tokens x M experts; warp w takes n-tiles w, w+8, ... (M <= 256: 4 per warp)
  constexpr int kW = kRcThreads / 32, kJ = 32 / kW;
  const int g = lane >> 2, tg = lane & 3;
  const int n_tiles = M / 8;
  float acc[kJ][4];
#pragma unroll
  for (int j = 0; j < kJ; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  const __nv_bfloat16* xa = xs + g * LD + tg * 2;
  for (int kk = 0; kk < kc; kk += 16) {
    const uint32_t a0 = *reinterpret_cast<const uint32_t*>(xa + kk);
    const uint32_t a1 = *reinterpret_cast<const uint32_t*>(xa + 8 * LD + kk);
    const uint32_t a2 = *reinterpret_cast<const uint32_t*>(xa + kk + 8);
    const uint32_t a3 = *reinterpret_cast<const uint32_t*>(xa + 8 * LD + kk + 8);
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int nt = warp + kW * j;
      if (nt < n_tiles) {
        const __nv_bfloat16* wb = wt + (nt * 8 + g) * LD + tg * 2 + kk;
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(wb);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(wb + 8);
        mma_bf16_16816(acc[j], a0, a1, a2, a3, b0, b1);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kJ; ++j) {
    const int nt = warp + kW * j;
    if (nt < n_tiles) {
      const int e = nt * 8 + tg * 2;
      part[g * M + e] = acc[j][0];
      part[g * M + e + 1] = acc[j][1];
      part[(g + 8) * M + e] = acc[j][2];
      part[(g + 8) * M + e + 1] = acc[j][3];
    }
  }
  RC_PROBE(3);
  route_finish(rsm, part, s_gather, S, split, t0, nt_valid, M, K, bias, ids, weights, logits_out, dbg, ep);
  route_ep_arrive(ep);
}

// tcgen05 variant (default for M <= 256, K chunk a multiple of 64): the experts are the MMA's
// M dimension (swap-AB, as in the FFN): A = this split's W_r^T chunk as [128 experts x 64 k]
// SW128 tiles, B = the tile's 16 token rows, D = [128 experts x 16 tokens] fp32 in TMEM --
// n_mt * kc/16 MMAs issued by one thread instead of 16 warps of mma.sync (which the profile
// showed throughput-bound at ~4k cycles). Same split-K cluster and top-K tail.
// The tcgen05 router always launches with programmatic dependent launch: its CTAs stage the
// static router weights while the previous kernel (combine) finishes and write their outputs
// after griddepcontrol.wait (-1% step time on a 24-layer trace)
// tokens per cluster tile (MMA N). 32 measured slower (13.6 vs 11.1 us): half the CTAs, and
// each CTA's top-K tail ranks twice the tokens
constexpr int kRtTok = 16;
static_assert(kRtTok == 16 || kRtTok == 32, "one or two 16-column TMEM loads per quadrant");
constexpr int kRtTileA = 16384, kRtTileB = kRtTok * 128;

struct RouteTcGeom {
  int S, kc, nkt, n_mt;
  size_t smem;
};
__host__ __device__ inline RouteTcGeom route_tc_geom(int d_h, int M) {
  const RouteGeom g = route_geom(d_h, M);
  RouteTcGeom t;
  t.S = g.S;
  t.kc = g.kc;
  t.nkt = g.kc / 64;
  t.n_mt = (M + 127) / 128;
  t.smem = 1024 + static_cast<size_t>(t.n_mt) * t.nkt * kRtTileA + static_cast<size_t>(t.nkt) * kRtTileB +
           static_cast<size_t>(kRtTok) * M * 4;
  return t;
}
bool route_tc_path(int M, int K, int d_h) {
  const RouteTcGeom t = route_tc_geom(d_h, M);
  return route_fast_path(M, K, d_h) && M <= 256 && t.kc % 64 == 0 && t.smem <= 200 * 1024;
}

__global__ void __launch_bounds__(kRcThreads) route_tc_kernel(const __nv_bfloat16* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ wr,
                                                              const float* __restrict__ bias, int T, int d_h, int M,
                                                              int K, int kc, int32_t* __restrict__ ids,
                                                              float* __restrict__ weights,
                                                              float* __restrict__ logits_out, long long* dbg,
                                                              const EpPeers ep) {
  extern __shared__ __align__(16) uint8_t rt_raw[];
  uint8_t* rsm = rt_raw + ((1024u - (smem_u32(rt_raw) & 1023u)) & 1023u);
  const int nkt = kc / 64, n_mt = (M + 127) / 128;
  uint8_t* A = rsm;                                          // [n_mt][nkt] SW128 tiles of 128 x 64
  uint8_t* B = A + static_cast<size_t>(n_mt) * nkt * kRtTileA;  // [nkt] SW128 tiles of 16 x 64
  float* part = reinterpret_cast<float*>(B + static_cast<size_t>(nkt) * kRtTileB);  // [kRtTok][M]
  __shared__ __align__(8) uint64_t s_gather, s_mma;
  __shared__ uint32_t s_tmem;
  const int S = gridDim.y;
  const uint32_t split = cluster_ctarank();
  const int t0 = blockIdx.x * kRtTok, k0 = static_cast<int>(split) * kc;
  const int kn = max(0, min(kc, d_h - k0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt_valid = min(kRtTok, T - t0);
  if (tid == 0) { mbar_init(&s_gather, 1); mbar_init(&s_mma, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&s_tmem, 64);  // >= n_mt * kRtTok columns
  RC_PROBE(0);
  // stage W_r^T rows of this K chunk (static: before the PDL wait) and the token rows, 16-B
  // cp.async into the swizzled tile positions; out-of-range chunks are zero-filled
  // (no divisions in the issue loops: k-tile outer, 16-B chunk c = i & 7, row = i >> 3)
  for (int kt = 0; kt < nkt; ++kt)
    for (int i = tid; i < n_mt * 128 * 8; i += blockDim.x) {
      const int c = i & 7, e = i >> 3, r = e & 127;
      const int k = kt * 64 + c * 8;
      const uint32_t avail = (e < M && k < kn) ? 16u : 0u;
      const __nv_bfloat16* src = wr + (avail ? static_cast<size_t>(e) * d_h + k0 + k : 0);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                       smem_u32(A + ((e >> 7) * nkt + kt) * kRtTileA + r * 128 + ((c ^ (r & 7)) << 4))),
                   "l"(src), "r"(avail)
                   : "memory");
    }
  // the bias is static too: staged before the wait, so the logit reduction reads shared memory
  __shared__ float s_bias[256];
  if (bias)
    for (int i = tid; i < M; i += blockDim.x) s_bias[i] = __ldg(bias + i);
  RC_PROBE(1);
  pdl_wait();  // x = the previous layer's RMSNorm output; ids/weights are read by its kernels
  pdl_trigger();
  for (int i = tid; i < kRtTok * nkt * 8; i += blockDim.x) {
    const int c = i & 7, r = (i >> 3) & (kRtTok - 1), kt = i / (kRtTok * 8);  // (constant divisor)
    const int k = kt * 64 + c * 8;
    const uint32_t avail = (r < nt_valid && k < kn) ? 16u : 0u;
    const __nv_bfloat16* src = x + (avail ? static_cast<size_t>(t0 + r) * d_h + k0 + k : 0);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                     smem_u32(B + kt * kRtTileB + r * 128 + ((c ^ (r & 7)) << 4))),
                 "l"(src), "r"(avail)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  fence_proxy_async_shared_cta();  // generic (cp.async) smem writes -> async-proxy MMA reads
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  RC_PROBE(2);
  const uint32_t tmem = s_tmem;
  if (warp == 0) {  // converged warp, elected issuing lane (no per-MMA ELECT/R2UR waterfall)
    const uint32_t idesc = umma_idesc_bf16(128, kRtTok);
    for (int mt = 0; mt < n_mt; ++mt)
      for (int kt = 0; kt < nkt; ++kt) {
        const uint32_t a = smem_u32(A + (mt * nkt + kt) * kRtTileA), b = smem_u32(B + kt * kRtTileB);
#pragma unroll
        for (int k16 = 0; k16 < 4; ++k16)
          umma_bf16_elect(tmem + mt * kRtTok, umma_desc_sw128(a + 32 * k16), umma_desc_sw128(b + 32 * k16), idesc,
                          (kt | k16) ? 1u : 0u);
      }
    umma_commit_elect(&s_mma);
  }
  mbar_wait(&s_mma, 0);
  tc_fence_after();
  if (warp < 4 * (kRtTok / 16)) {  // TMEM lane quadrant = warp & 3: experts mt*128 + 32*(warp&3) +
                                    // lane; warps 4-7 take token columns 16-31 when kRtTok = 32
    const int q = warp & 3, c0 = (warp >> 2) * 16;
    for (int mt = 0; mt < n_mt; ++mt) {
      uint32_t v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + mt * kRtTok + c0, v);
      tmem_wait_ld();
      const int e = mt * 128 + q * 32 + lane;
      if (e < M) {
#pragma unroll
        for (int j = 0; j < 16; ++j) part[(c0 + j) * M + e] = __uint_as_float(v[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
  RC_PROBE(3);
  route_finish(rsm, part, s_gather, S, split, t0, nt_valid, M, K, bias ? s_bias : nullptr, ids, weights, logits_out,
               dbg, ep, kRtTok);
  route_ep_arrive(ep);
}

size_t route_workspace_bytes(int T, int d_h, int M) { return 256; }

bool route_fast_path(int M, int K, int d_h) {
  return M % 8 == 0 && M <= 256 && K <= 32 && d_h % 8 == 0 && route_geom(d_h, M).smem <= 200 * 1024;
}

cudaError_t launch_route_mma(const __nv_bfloat16* x, const __nv_bfloat16* w_router, const float* bias, int T,
                             int d_h, int M, int K, int32_t* ids, float* weights, float* logits_out, void* ws,
                             cudaStream_t stream, const EpPeers* ep) {
  (void)ws;
  if (T <= 0) return cudaSuccess;
  if (route_tc_path(M, K, d_h)) {
    const RouteTcGeom g = route_tc_geom(d_h, M);
    static SmemAttrCache attr_tc;
    if (cudaError_t e = ensure_smem_attr(route_tc_kernel, g.smem, attr_tc); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((T + kRtTok - 1) / kRtTok, g.S, 1);
    cfg.blockDim = dim3(kRcThreads, 1, 1);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = g.S;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    EpPeers none{};
    return cudaLaunchKernelEx(&cfg, route_tc_kernel, x, w_router, bias, T, d_h, M, K, g.kc, ids, weights,
                              logits_out, g_route_dbg, ep ? *ep : none);
  }
  const RouteGeom g = route_geom(d_h, M);
  static SmemAttrCache smem_attr;
  if (cudaError_t e = ensure_smem_attr(route_cluster_kernel, g.smem, smem_attr); e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((T + kRcTok - 1) / kRcTok, g.S, 1);
  cfg.blockDim = dim3(kRcThreads, 1, 1);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = g.S;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 2 : 1;
  EpPeers none{};
  return cudaLaunchKernelEx(&cfg, route_cluster_kernel, x, w_router, bias, T, d_h, M, K, g.kc, ids, weights,
                            logits_out, g_route_dbg, ep ? *ep : none);
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
  static SmemAttrCache smem_attr;
  if (cudaError_t e = ensure_smem_attr(route_topk_kernel, smem, smem_attr); e != cudaSuccess) return e;
  const int blocks = (T + kTok - 1) / kTok;
  route_topk_kernel<<<blocks, threads, smem, stream>>>(x, w_router, bias, T, d_h, M, K, KS, ids, weights,
                                                        logits_out);
  return cudaGetLastError();
}

// ------------------------------------------------------------ residual + RMSNorm
// x += y (if y), h = bf16(x * rsqrt(mean(x^2) + eps)); one CTA per token with the
// traversal and reduction tree of the combine kernel's fused epilogue (rowops.cuh), so
// the unfused expert-parallel step reproduces the fused single-GPU step bit for bit.
__global__ void __launch_bounds__(kRowMaxThreads) residual_rmsnorm_kernel(float* __restrict__ x, const float* __restrict__ y,
                                                               __nv_bfloat16* __restrict__ h, int d_h, float eps) {
  __shared__ float s_red[16];
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  float ss = 0.f;
  for (int base = 0; base < d_h; base += blockDim.x * kRowVec)
    for (int c = 0; c < kRowChunks; ++c) {
      const int f0 = row_chunk(base, c);
      for (int q = 0; q < 4 && f0 + q < d_h; ++q) {
        const size_t o = static_cast<size_t>(t) * d_h + f0 + q;
        float v = x[o];
        if (y) {
          v = v + y[o];
          x[o] = v;
        }
        ss = fmaf(v, v, ss);
      }
    }
  const float tot = block_sum(ss, s_red);
  const float r = rsqrtf(tot / static_cast<float>(d_h) + eps);
  for (int base = 0; base < d_h; base += blockDim.x * kRowVec)
    for (int c = 0; c < kRowChunks; ++c) {
      const int f0 = row_chunk(base, c);
      for (int q = 0; q < 4 && f0 + q < d_h; ++q) {
        const size_t o = static_cast<size_t>(t) * d_h + f0 + q;
        h[o] = __float2bfloat16_rn(x[o] * r);
      }
    }
}

cudaError_t launch_residual_rmsnorm(float* x, const float* y, __nv_bfloat16* h_out, int T, int d_h, float eps,
                                    cudaStream_t stream) {
  return launch_pdl((g_pdl & PDL_RMSNORM) != 0, residual_rmsnorm_kernel, dim3(T), dim3(row_threads(d_h)), 0, stream, x, y, h_out, d_h, eps);
}

}  // namespace sere
