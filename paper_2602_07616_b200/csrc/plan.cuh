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
//   counts[Et]            cells routed to each bank expert (shared experts: T)
//   group_expert/row0/rows[Et]   bank expert, first permuted row, valid rows of group g
//   sched[Et]             groups in schedule order: padded rows descending (heaviest
//                         units first -> longest-processing-time-first balancing)
//   unit_off_gu/dn[Et+1]  prefix of work units over the schedule order
//   dep[Et]               gate/up units finished per group (the down units of a group
//                         wait for all of them); zeroed by align
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
  P_HDR = 16
};

struct PlanOffsets {
  int counts, group_expert, group_row0, group_rows, sched, unit_off_gu, unit_off_dn, dep, total;
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
  o.total = o.dep + Et;
  return o;
}

constexpr int kRowAlign = 16;     // group padding = MMA N granularity (M=128, cta_group::1)
constexpr int kColBlock = 256;    // max MMA columns (tokens) per work unit
constexpr int kTile = 64;         // K elements per 128-B swizzled row
constexpr int kTileBytes = 16384; // 128 rows x 64 bf16

__host__ __device__ inline int round_up(int x, int a) { return (x + a - 1) / a * a; }

struct Dims {
  int d_h, d_m, d_h_pad, d_m_pad;
  int tiles_gu;   // gate/up m-tiles per expert: d_m_pad/64 (each 64 features = 128 MMA rows gate|up)
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
  d.d_m_pad = round_up(d_m, 64);
  d.tiles_gu = d.d_m_pad / 64;
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

// bank layout: W13 tiles [Et][tiles_gu][ktiles_gu] then W2 tiles [Et][tiles_dn][ktiles_dn]
inline size_t bank_w13_bytes(int Et, const Dims& d) {
  return static_cast<size_t>(Et) * d.tiles_gu * d.ktiles_gu * kTileBytes;
}
inline size_t bank_w2_bytes(int Et, const Dims& d) {
  return static_cast<size_t>(Et) * d.tiles_dn * d.ktiles_dn * kTileBytes;
}

}  // namespace sere
