// plan.cuh -- device/host shared description of one MoE layer launch.
//
// The count/align pass (reroute_align.cu) turns the [T,K] id table into a
// "plan" that every later kernel reads from device memory, so that no
// data-dependent size ever crosses to the host (the pipeline is CUDA-graph
// capturable and needs no sync):
//
//   plan[P_STATUS]        SERE_* status (kernels after a failed check do nothing)
//   plan[P_NGROUPS]       number of expert groups (active routed experts ascending, then shared)
//   plan[P_TOTAL_ROWS]    rows of the permuted batch (each group padded to 16)
//   plan[P_UNITS_GU/DN]   work units of the gate/up and down phases of the fused FFN
//   plan[P_TICKET]        work-unit ticket counter of the fused FFN (zeroed by align)
//   plan[P_DONE]          CTAs of the fused FFN that finished; the last one re-zeroes the
//                         ticket and dependency counters, so the FFN can be relaunched on
//                         the same plan (sere_debug_replay_ffn: kernel-only timing)
//   counts[Et]            cells routed to each bank expert (shared experts: T)
//   group_expert/row0/rows[Et]   bank expert, first permuted row, valid rows of group g
//   sched[Et]             groups in schedule order: padded rows descending (heaviest
//                         units first -> longest-processing-time-first balancing)
//   unit_off_gu/dn[Et+1]  prefix of work units over the schedule order
//   dep[Et]               gate/up units finished per group (the down units of a group
//                         wait for all of them); zeroed by align
//   mw_gu[Et]             feature blocks per gate/up unit by schedule position (kMwGuMax)
//   erow0[Et]             first permuted row of bank expert e's group (-1: no cells)
#pragma once
#include <cstddef>
#include <cstdint>

namespace sere {

enum PlanIdx : int {
  P_STATUS = 0,
  P_NGROUPS = 1,
  P_TOTAL_ROWS = 2,
  P_UNITS_GU = 3,
  P_UNITS_DN = 4,
  P_NACTIVE = 5,
  P_TICKET = 6,
  P_DONE = 7,
  P_HDR = 16
};

struct PlanOffsets {
  int counts, group_expert, group_row0, group_rows, sched, unit_off_gu, unit_off_dn, dep, mw_gu, erow0, total;
};

__host__ __device__ inline PlanOffsets plan_offsets(int Et) {
  PlanOffsets o;
  o.counts = P_HDR;
  o.group_expert = o.counts + Et;
  o.group_row0 = o.group_expert + Et;
  o.group_rows = o.group_row0 + Et;
  o.sched = o.group_rows + Et;
  o.unit_off_gu = o.sched + Et;
  o.unit_off_dn = o.unit_off_gu + Et + 1;
  o.dep = o.unit_off_dn + Et + 1;
  o.mw_gu = o.dep + Et;
  o.erow0 = o.mw_gu + Et;
  o.total = o.erow0 + Et;
  return o;
}

constexpr int kRowAlign = 16;     // group padding = MMA N granularity (M=128, cta_group::1)
constexpr int kTokBlkPerm = 32;   // token block of the group row order (align prefixes, permute ranks)
constexpr int kColBlock = 256;    // max MMA columns (tokens) per work unit
constexpr int kTile = 64;         // K elements per 128-B swizzled row
constexpr int kTileBytes = 16384; // 128 rows x 64 bf16

__host__ __device__ inline int round_up(int x, int a) { return (x + a - 1) / a * a; }

// ---- work-unit geometry of the fused FFN (shared by the planner and the kernel)
// A unit covers `mw` consecutive m-tiles of one expert group and one column block of
// its rows: every k-step loads the block's activation tile (B) ONCE and multiplies it
// with every weight tile (A) of the unit -- gate AND up for a gate/up feature block --
// so activations are re-read tiles/mw times. TMEM bounds mw: the unit's accumulators
// (2 per gate/up block, 1 per down m-tile) of n_mma fp32 columns fit 512 columns.
constexpr int kTmemCols = 512;
#ifndef SERE_MW_GU_MAX
#define SERE_MW_GU_MAX 2
#endif
#ifndef SERE_MW_DN_MAX
#define SERE_MW_DN_MAX 2
#endif
constexpr int kMwGuMax = SERE_MW_GU_MAX;  // gate/up: feature blocks of 128 (2 accumulators each; 2 measured
                                          // 5% faster than 1: 16 MMAs per k-step amortise the issue cost)
constexpr int kMwDnMax = SERE_MW_DN_MAX;  // down: 2 x 128 features per unit

// accs = TMEM accumulators per m-tile (2 for gate/up: gate and up; 1 for down)
__host__ __device__ inline int unit_mw(int n16, int cap, int tiles, int accs = 1) {
  const int nb = n16 < kColBlock ? (n16 > 0 ? n16 : kRowAlign) : kColBlock;
  int mw = kTmemCols / (nb * accs);
  mw = mw < cap ? mw : cap;
  mw = mw < tiles ? mw : tiles;
  return mw < 1 ? 1 : mw;
}
__host__ __device__ inline int col_blocks(int n16) { return (n16 + kColBlock - 1) / kColBlock; }
__host__ __device__ inline int group_units_gu(int n16, int tiles_gu, int cap = kMwGuMax) {
  const int mw = unit_mw(n16, cap, tiles_gu, 2);
  return col_blocks(n16) * ((tiles_gu + mw - 1) / mw);
}
// down units take kMwDnMax m-tiles (4-wide units for narrow groups: top-k FFN -2.9% but the SERE
// step +1%; one-m-tile units for the smallest groups: neutral for SERE, -7% for top-k)
__host__ __device__ inline int dn_cap(int) { return kMwDnMax; }
__host__ __device__ inline int group_units_dn(int n16, int tiles_dn, int ksplit_dn) {
  const int mw = unit_mw(n16, dn_cap(n16), tiles_dn);
  return col_blocks(n16) * ((tiles_dn + mw - 1) / mw) * ksplit_dn;
}

struct Dims {
  int d_h, d_m, d_h_pad, d_m_pad;
  int tiles_gu;   // gate/up feature blocks per expert: d_m_pad/128 (a gate tile + an up tile each)
  int ktiles_gu;  // d_h_pad/64
  int tiles_dn;   // down m-tiles per expert: d_h_pad/128
  int ktiles_dn;  // d_m_pad/64
  int ksplit_dn;  // K splits of the down GEMM (divides ktiles_dn)
};

inline Dims make_dims(int d_h, int d_m) {
  Dims d;
  d.d_h = d_h;
  d.d_m = d_m;
  d.d_h_pad = round_up(d_h, 128);
  d.d_m_pad = round_up(d_m, 128);
  d.tiles_gu = d.d_m_pad / 128;
  d.ktiles_gu = d.d_h_pad / 64;
  d.tiles_dn = d.d_h_pad / 128;
  d.ktiles_dn = d.d_m_pad / 64;
  // split the down GEMM's K so that one unit streams at most 32 K-tiles (512 KB of weights)
  int ks = 1;
  while (d.ktiles_dn / ks > 32 || d.ktiles_dn % ks != 0) {
    ++ks;
    if (ks > d.ktiles_dn) { ks = d.ktiles_dn; break; }
  }
  d.ksplit_dn = ks;
  return d;
}

// bank layout: W13 tiles [Et][tiles_gu][ktiles_gu][gate, up] then W2 tiles
// [Et][ceil(tiles_dn/G)][ktiles_dn][G] (G = kW2Group): the m-tiles of a down unit are
// adjacent at every k-tile, so one copy feeds all its accumulators
inline size_t bank_w13_bytes(int Et, const Dims& d) {
  return static_cast<size_t>(Et) * d.tiles_gu * d.ktiles_gu * 2 * kTileBytes;
}
// down tiles are stored in groups of kW2Group m-tiles that sit side by side at every
// k-tile (a down unit of up to kW2Group m-tiles reads one contiguous run per k-step)
constexpr int kW2Group = kMwDnMax;
inline size_t bank_w2_bytes(int Et, const Dims& d) {
  return static_cast<size_t>(Et) * ((d.tiles_dn + kW2Group - 1) / kW2Group) * kW2Group * d.ktiles_dn * kTileBytes;
}
// byte offset of down tile (expert e, m-tile mt, k-tile kt) inside the W2 region
__host__ __device__ inline size_t w2_tile_offset(int e, int mt, int kt, int tiles_dn, int ktiles_dn) {
  const int groups = (tiles_dn + kW2Group - 1) / kW2Group;
  return ((static_cast<size_t>(e) * groups + mt / kW2Group) * ktiles_dn + kt) * kW2Group * kTileBytes +
         static_cast<size_t>(mt % kW2Group) * kTileBytes;
}

}  // namespace sere
