// capi.cu -- extern "C" entry points of include/sere_b200.h: host-side checks
// (shape/config, in the reference's order), workspace carving, launch sequencing.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "../../include/sere_b200.h"
#include "params.cuh"
#include "plan.cuh"


namespace sere {

namespace {

constexpr int kMaxCells = 16384;  // T*K limit of the single-CTA align kernel (u16 counters, 64 KB ids)
constexpr int kMaxExperts = 256;  // smem of the single-CTA align kernel (per-warp expert masks)
constexpr int kMaxShared = 31;

int g_num_sms[64] = {0};

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (g_num_sms[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms[dev] = n > 0 ? n : 148;
  }
  return g_num_sms[dev];
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

long long* g_align_dbg = nullptr;  // sere_debug_set_align_clocks
unsigned long long* g_ffn_trace = nullptr;  // sere_debug_set_ffn_trace
int g_ffn_dbg_mode = 0;                     // sere_debug_set_ffn_mode
constexpr int kStageEvents = 6;
thread_local cudaEvent_t t_stage_events[kStageEvents];
thread_local bool t_stage_events_on = false;

inline void stage_mark(int i, cudaStream_t stream) {
  if (!t_stage_events_on) return;
  // under stream capture a plain record only marks a dependency; an external record
  // becomes a real event-record node of the graph, so the timestamps exist after replay
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(t_stage_events[i], stream, cudaEventRecordExternal);
  else
    cudaEventRecord(t_stage_events[i], stream);
}

struct WsLayout {
  size_t plan, slot_row, row_token, x_pack, h_pack, y_perm, ids_final, blk_prefix, total;
  int r_max;
  Dims d;
  int Et;
};

WsLayout ws_layout(int T, int K, int M, int n_shared, int d_h, int d_m) {
  WsLayout L;
  L.d = make_dims(d_h, d_m);
  L.Et = M + n_shared;
  L.r_max = round_up(T * (K + n_shared) + kRowAlign * L.Et, 8);
  const PlanOffsets po = plan_offsets(L.Et);
  const int TB = (T + kTokBlkPerm - 1) / kTokBlkPerm;
  size_t off = 0;
  L.plan = off;
  off = align_up(off + static_cast<size_t>(po.total) * 4, 1024);
  L.slot_row = off;
  off = align_up(off + static_cast<size_t>(T) * (K + n_shared) * 4, 1024);
  L.row_token = off;
  off = align_up(off + static_cast<size_t>(L.r_max) * 4, 1024);
  L.x_pack = off;
  off = align_up(off + static_cast<size_t>(L.d.ktiles_gu) * L.r_max * 128, 1024);
  L.h_pack = off;
  off = align_up(off + static_cast<size_t>(L.d.ktiles_dn) * L.r_max * 128, 1024);
  L.y_perm = off;
  off = align_up(off + static_cast<size_t>(L.d.ksplit_dn) * L.r_max * L.d.d_h_pad * 4, 1024);
  L.ids_final = off;
  off = align_up(off + static_cast<size_t>(T) * K * 4, 1024);
  L.blk_prefix = off;
  off = align_up(off + static_cast<size_t>(round_up(TB * L.Et, 2)) * 2, 1024);
  L.total = off + 1024;  // slack for aligning the caller's base to 1024 B
  return L;
}

int check_cuda(cudaError_t e) { return e == cudaSuccess ? SERE_OK : SERE_ERR_CUDA; }

int check_layer_shapes(int M, int n_shared, int d_h, int d_m, int activation, int T, int K) {
  if (M < 1 || M > kMaxExperts || n_shared < 0 || n_shared > kMaxShared) return SERE_ERR_UNSUPPORTED;
  if (d_h < 1 || d_m < 1) return SERE_ERR_CONFIG;
  if (activation < SERE_ACT_SILU || activation > SERE_ACT_GELU_TANH) return SERE_ERR_CONFIG;
  if (T < 0 || K < 1) return SERE_ERR_DIMENSION;
  if (K > M) return SERE_ERR_CONFIG;  // top_k <= M (moe.py:116-118)
  if (static_cast<long long>(T) * K > kMaxCells) return SERE_ERR_UNSUPPORTED;
  return SERE_OK;
}

int check_reroute_cfg(int K, int M, int S, double rho) {
  if (S < 1) return SERE_ERR_CONFIG;                         // rerouting.py:45-46
  if (!(rho >= 0.0 && rho <= 1.0)) return SERE_ERR_CONFIG;   // rerouting.py:48-49 (NaN rejected too)
  if (S > K) return SERE_ERR_CONFIG;                         // rerouting.py:104-107
  if (M < 1 || M > kMaxExperts) return SERE_ERR_UNSUPPORTED;
  return SERE_OK;
}

uint8_t* ws_base(const void* workspace) {
  return reinterpret_cast<uint8_t*>(align_up(reinterpret_cast<uintptr_t>(workspace), 1024));
}

FfnParams ffn_params(const void* bank, const WsLayout& L, uint8_t* ws, int activation) {
  const Dims& d = L.d;
  const uint8_t* w13 = reinterpret_cast<const uint8_t*>(bank);
  FfnParams fp{};
  fp.w13 = w13;
  fp.w2 = w13 + bank_w13_bytes(L.Et, d);
  fp.tiles_gu = d.tiles_gu;
  fp.ktiles_gu = d.ktiles_gu;
  fp.tiles_dn = d.tiles_dn;
  fp.ktiles_dn = d.ktiles_dn;
  fp.ksplit_dn = d.ksplit_dn;
  fp.x_pack = ws + L.x_pack;
  fp.h_pack = ws + L.h_pack;
  fp.y_perm = reinterpret_cast<float*>(ws + L.y_perm);
  fp.r_max = L.r_max;
  fp.d_h_pad = d.d_h_pad;
  fp.plan = reinterpret_cast<int32_t*>(ws + L.plan);
  fp.Et = L.Et;
  fp.act = activation;
  fp.trace = g_ffn_trace;
  fp.dbg_mode = g_ffn_dbg_mode;
  return fp;
}

// M = global expert count; the bank holds global experts [e_lo, e_lo + m_local) + n_shared shared ones
int run_layer(const void* bank, int M, int e_lo, int m_local, int n_shared, int d_h, int d_m, int activation,
              const double* sim, int S,
              double rho, int flags, int mode, const uint16_t* x, const int32_t* ids_in, const float* weights,
              int T, int K, int32_t* ids_out, uint8_t* expert_class, int32_t* reroute_map, int32_t* active_list,
              int32_t* n_active, float* y, uint16_t* y_bf16, void* workspace, size_t workspace_bytes,
              int32_t* status_dev, cudaStream_t stream, float* x_res = nullptr, uint16_t* h_next = nullptr,
              float eps = 0.f, bool do_combine = true, const EpSync* sync = nullptr) {
  const WsLayout L = ws_layout(T, K, m_local, n_shared, d_h, d_m);
  if (workspace == nullptr || workspace_bytes < L.total) return SERE_ERR_WORKSPACE;
  if (bank == nullptr || x == nullptr || ids_in == nullptr || weights == nullptr)
    return SERE_ERR_DIMENSION;
  if (do_combine && y == nullptr && (x_res == nullptr || h_next == nullptr)) return SERE_ERR_DIMENSION;
  uint8_t* ws = reinterpret_cast<uint8_t*>(align_up(reinterpret_cast<uintptr_t>(workspace), 1024));
  int32_t* plan = reinterpret_cast<int32_t*>(ws + L.plan);
  int32_t* slot_row = reinterpret_cast<int32_t*>(ws + L.slot_row);
  int32_t* row_token = reinterpret_cast<int32_t*>(ws + L.row_token);
  uint8_t* x_pack = ws + L.x_pack;
  uint8_t* h_pack = ws + L.h_pack;
  float* y_perm = reinterpret_cast<float*>(ws + L.y_perm);
  const Dims& d = L.d;
  const int sms = num_sms();

  AlignParams ap{};
  ap.ids_in = ids_in;
  ap.sim = sim;
  ap.T = T; ap.K = K; ap.M = M; ap.S = S; ap.n_shared = n_shared;
  ap.rho = rho;
  ap.flags = flags;
  ap.mode = mode;
  ap.ids_out = ids_out;
  ap.expert_class = expert_class;
  ap.reroute_map = reroute_map;
  ap.active_list = active_list;
  ap.n_active = n_active;
  ap.status_dev = status_dev;
  ap.plan = plan;
  ap.row_token = row_token;
  ap.ids_final = reinterpret_cast<int32_t*>(ws + L.ids_final);
  ap.blk_prefix = reinterpret_cast<uint16_t*>(ws + L.blk_prefix);
  if (sync != nullptr) ap.sync = *sync;
  ap.tiles_gu = d.tiles_gu;
  ap.tiles_dn = d.tiles_dn;
  ap.ksplit_dn = d.ksplit_dn;
  ap.e_lo = e_lo;
  ap.m_local = m_local;
  ap.r_max = L.r_max;
  ap.ffn_ctas = sms;
  ap.dbg = g_align_dbg;
  stage_mark(0, stream);
  cudaError_t e = launch_reroute_align(ap, stream);
  if (e != cudaSuccess) return SERE_ERR_CUDA;

  stage_mark(1, stream);
  e = launch_permute(reinterpret_cast<const __nv_bfloat16*>(x), d, plan, L.Et, m_local, e_lo, ap.ids_final,
                     ap.blk_prefix, T, K, n_shared, slot_row, row_token, L.r_max, x_pack, stream,
                     sync == nullptr ? y_perm : nullptr,  // expert parallel: peers may still read it
                     static_cast<long long>(d.ksplit_dn) * L.r_max * d.d_h_pad / 32,
                     sync == nullptr);  // single GPU: x rows loaded before the PDL wait
  if (e != cudaSuccess) return SERE_ERR_CUDA;

  FfnParams fp = ffn_params(bank, L, ws, activation);
  if (sync != nullptr) fp.sync = *sync;
  stage_mark(2, stream);
  e = launch_moe_ffn(fp, sms, stream);
  if (e != cudaSuccess) return SERE_ERR_CUDA;
  stage_mark(3, stream);  // gate/up and down run in one launch: stage 3 is empty
  if (!do_combine) return SERE_OK;  // expert parallel over peer memory: sere_combine_ep

  stage_mark(4, stream);
  e = launch_combine(y_perm, d, L.r_max, plan, slot_row, weights, T, K, n_shared, y,
                     reinterpret_cast<__nv_bfloat16*>(y_bf16), x_res, reinterpret_cast<__nv_bfloat16*>(h_next), eps,
                     stream);
  stage_mark(5, stream);
  return check_cuda(e);
}

}  // namespace
}  // namespace sere

namespace sere {
#ifndef SERE_PDL_DEFAULT
#define SERE_PDL_DEFAULT 31  // all: +2.8% on the C4 step (FFN alone +2%), same-box A/B r02
#endif
int g_pdl = SERE_PDL_DEFAULT;  // PDL_* bits (sere_set_pdl)
#ifndef SERE_L2_DEFAULT
#define SERE_L2_DEFAULT 1  // L2_DISCARD_Y: +2.2% C4 SERE, +3% top-k (profiles/r02_l2_scratch_discard.txt)
#endif
int g_l2 = SERE_L2_DEFAULT;  // L2_* bits (sere_set_l2)
}  // namespace sere

using namespace sere;

extern "C" {

int sere_abi_version(void) { return SERE_ABI_VERSION; }

const char* sere_status_string(int status) {
  switch (status) {
    case SERE_OK: return "ok";
    case SERE_ERR_CONFIG: return "ConfigError";
    case SERE_ERR_DIMENSION: return "DimensionError";
    case SERE_ERR_INPUT: return "InputError";
    case SERE_ERR_ROUTING: return "RoutingError";
    case SERE_ERR_DOMAIN: return "DomainError";
    case SERE_ERR_CUDA: return "CUDA error";
    case SERE_ERR_UNSUPPORTED: return "unsupported device or size";
    case SERE_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

int sere_device_check(int device) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SERE_ERR_CUDA;
  if (prop.major != 10 || prop.minor != 0) return SERE_ERR_UNSUPPORTED;
  return SERE_OK;
}

int sere_reroute(const int32_t* ids_in, const double* sim, int T, int K, int M, int S, double rho, int flags,
                 int32_t* ids_out, uint8_t* expert_class, int32_t* reroute_map, int32_t* active_list,
                 int32_t* n_active, int32_t* status_dev, void* stream) {
  if (T < 0 || K < 1) return SERE_ERR_DIMENSION;
  const int rc = check_reroute_cfg(K, M, S, rho);
  if (rc != SERE_OK) return rc;
  if (static_cast<long long>(T) * K > kMaxCells) return SERE_ERR_UNSUPPORTED;
  if ((ids_in == nullptr && T > 0) || sim == nullptr) return SERE_ERR_DIMENSION;
  AlignParams ap{};
  ap.ids_in = ids_in;
  ap.sim = sim;
  ap.T = T; ap.K = K; ap.M = M; ap.S = S; ap.n_shared = 0;
  ap.rho = rho;
  ap.flags = flags;
  ap.mode = MODE_REROUTE;
  ap.e_lo = 0;
  ap.m_local = M;
  ap.dbg = g_align_dbg;
  ap.ids_out = ids_out;
  ap.expert_class = expert_class;
  ap.reroute_map = reroute_map;
  ap.active_list = active_list;
  ap.n_active = n_active;
  ap.status_dev = status_dev;
  return check_cuda(launch_reroute_align(ap, static_cast<cudaStream_t>(stream)));
}

size_t sere_expert_bank_bytes(int n_experts_total, int d_h, int d_m) {
  if (n_experts_total < 1 || d_h < 1 || d_m < 1) return 0;
  const Dims d = make_dims(d_h, d_m);
  return bank_w13_bytes(n_experts_total, d) + bank_w2_bytes(n_experts_total, d);
}

int sere_pack_experts(const uint16_t* w_gate, const uint16_t* w_up, const uint16_t* w_down, int count, int d_h,
                      int d_m, void* bank, int n_experts_total, int first, void* stream) {
  if (count < 0 || first < 0 || first + count > n_experts_total || d_h < 1 || d_m < 1) return SERE_ERR_DIMENSION;
  if (bank == nullptr || (count > 0 && (!w_gate || !w_up || !w_down))) return SERE_ERR_DIMENSION;
  const Dims d = make_dims(d_h, d_m);
  return check_cuda(launch_pack(reinterpret_cast<const __nv_bfloat16*>(w_gate),
                                reinterpret_cast<const __nv_bfloat16*>(w_up),
                                reinterpret_cast<const __nv_bfloat16*>(w_down), count, d, n_experts_total, first,
                                reinterpret_cast<uint8_t*>(bank), 0, static_cast<cudaStream_t>(stream)));
}

int sere_unpack_experts(const void* bank, int n_experts_total, int first, int count, int d_h, int d_m,
                        uint16_t* w_gate, uint16_t* w_up, uint16_t* w_down, void* stream) {
  if (count < 0 || first < 0 || first + count > n_experts_total || d_h < 1 || d_m < 1) return SERE_ERR_DIMENSION;
  if (bank == nullptr || (count > 0 && (!w_gate || !w_up || !w_down))) return SERE_ERR_DIMENSION;
  const Dims d = make_dims(d_h, d_m);
  return check_cuda(launch_pack(reinterpret_cast<const __nv_bfloat16*>(w_gate),
                                reinterpret_cast<const __nv_bfloat16*>(w_up),
                                reinterpret_cast<const __nv_bfloat16*>(w_down), count, d, n_experts_total, first,
                                reinterpret_cast<uint8_t*>(const_cast<void*>(bank)), 1,
                                static_cast<cudaStream_t>(stream)));
}

size_t sere_layer_workspace_bytes(int T, int K, int M, int n_shared, int d_h, int d_m) {
  if (T < 0 || K < 1 || M < 1 || n_shared < 0 || d_h < 1 || d_m < 1) return 0;
  return ws_layout(T, K, M, n_shared, d_h, d_m).total;
}

int sere_layer_workspace_layout(int T, int K, int M, int n_shared, int d_h, int d_m, sere_ws_layout* out) {
  if (out == nullptr || T < 0 || K < 1 || M < 1 || n_shared < 0 || d_h < 1 || d_m < 1) return SERE_ERR_DIMENSION;
  const WsLayout L = ws_layout(T, K, M, n_shared, d_h, d_m);
  const PlanOffsets po = plan_offsets(L.Et);
  out->off_plan_i32 = L.plan;
  out->off_slot_row = L.slot_row;
  out->off_row_token = L.row_token;
  out->off_x_pack = L.x_pack;
  out->off_h_pack = L.h_pack;
  out->off_y_perm = L.y_perm;
  out->off_ids_final = L.ids_final;
  out->off_blk_prefix = L.blk_prefix;
  out->total_bytes = L.total;
  out->r_max = L.r_max;
  out->d_h_pad = L.d.d_h_pad;
  out->d_m_pad = L.d.d_m_pad;
  out->ksplit_down = L.d.ksplit_dn;
  out->plan_groups_off = P_NGROUPS;
  out->plan_group_expert_off = po.group_expert;
  out->plan_group_row0_off = po.group_row0;
  out->plan_group_rows_off = po.group_rows;
  out->plan_counts_off = po.counts;
  out->plan_unit_off_gu = po.unit_off_gu;
  out->plan_unit_off_dn = po.unit_off_dn;
  return SERE_OK;
}

int sere_layer_forward(const void* bank, int M, int n_shared, int d_h, int d_m, int activation, const uint16_t* x,
                       const int32_t* ids, const float* weights, int T, int K, float* y, uint16_t* y_bf16,
                       void* workspace, size_t workspace_bytes, int32_t* status_dev, void* stream) {
  const int rc = check_layer_shapes(M, n_shared, d_h, d_m, activation, T, K);
  if (rc != SERE_OK) return rc;
  if (T == 0) return SERE_OK;
  return run_layer(bank, M, 0, M, n_shared, d_h, d_m, activation, nullptr, K, 0.0, 0, MODE_ALIGN, x, ids, weights,
                   T, K,
                   nullptr, nullptr, nullptr, nullptr, nullptr, y, y_bf16, workspace, workspace_bytes, status_dev,
                   static_cast<cudaStream_t>(stream));
}

int sere_moe_forward(const void* bank, int M, int n_shared, int d_h, int d_m, int activation, const double* sim,
                     int S, double rho, int flags, const uint16_t* x, const int32_t* ids_in, const float* weights,
                     int T, int K, int32_t* ids_out, uint8_t* expert_class, int32_t* reroute_map,
                     int32_t* active_list, int32_t* n_active, float* y, uint16_t* y_bf16, void* workspace,
                     size_t workspace_bytes, int32_t* status_dev, void* stream) {
  int rc = check_layer_shapes(M, n_shared, d_h, d_m, activation, T, K);
  if (rc != SERE_OK) return rc;
  rc = check_reroute_cfg(K, M, S, rho);
  if (rc != SERE_OK) return rc;
  if (sim == nullptr) return SERE_ERR_DIMENSION;
  if (T == 0) return SERE_OK;
  return run_layer(bank, M, 0, M, n_shared, d_h, d_m, activation, sim, S, rho, flags, MODE_REROUTE | MODE_ALIGN, x,
                   ids_in, weights, T, K, ids_out, expert_class, reroute_map, active_list, n_active, y, y_bf16,
                   workspace, workspace_bytes, status_dev, static_cast<cudaStream_t>(stream));
}

int sere_moe_block_forward(const void* bank, int M, int n_shared, int d_h, int d_m, int activation,
                           const double* sim, int S, double rho, int flags, const uint16_t* h,
                           const int32_t* ids_in, const float* weights, int T, int K, int32_t* ids_out,
                           uint8_t* expert_class, int32_t* reroute_map, int32_t* active_list, int32_t* n_active,
                           float* x_residual, uint16_t* h_next, float eps, float* y, void* workspace,
                           size_t workspace_bytes, int32_t* status_dev, void* stream) {
  int rc = check_layer_shapes(M, n_shared, d_h, d_m, activation, T, K);
  if (rc != SERE_OK) return rc;
  rc = check_reroute_cfg(K, M, S, rho);
  if (rc != SERE_OK) return rc;
  if (sim == nullptr || x_residual == nullptr || h_next == nullptr) return SERE_ERR_DIMENSION;
  if (T == 0) return SERE_OK;
  return run_layer(bank, M, 0, M, n_shared, d_h, d_m, activation, sim, S, rho, flags, MODE_REROUTE | MODE_ALIGN, h,
                   ids_in, weights, T, K, ids_out, expert_class, reroute_map, active_list, n_active, y, nullptr,
                   workspace, workspace_bytes, status_dev, static_cast<cudaStream_t>(stream), x_residual, h_next,
                   eps);
}

int sere_moe_forward_ep(const void* bank, int M, int expert_lo, int expert_hi, int n_shared_local, int d_h,
                        int d_m, int activation, const double* sim, int S, double rho, int flags, const uint16_t* x,
                        const int32_t* ids_in, const float* weights, int T, int K, int32_t* ids_out,
                        uint8_t* expert_class, int32_t* reroute_map, int32_t* active_list, int32_t* n_active,
                        float* y_partial, void* workspace, size_t workspace_bytes, int32_t* status_dev,
                        void* stream) {
  if (expert_lo < 0 || expert_hi > M || expert_hi < expert_lo) return SERE_ERR_DIMENSION;
  const int m_local = expert_hi - expert_lo;
  if (m_local + n_shared_local < 1) return SERE_ERR_DIMENSION;
  int rc = check_layer_shapes(M, n_shared_local, d_h, d_m, activation, T, K);
  if (rc != SERE_OK) return rc;
  rc = check_reroute_cfg(K, M, S, rho);
  if (rc != SERE_OK) return rc;
  if (sim == nullptr) return SERE_ERR_DIMENSION;
  if (T == 0) return SERE_OK;
  return run_layer(bank, M, expert_lo, m_local, n_shared_local, d_h, d_m, activation, sim, S, rho, flags,
                   MODE_REROUTE | MODE_ALIGN, x, ids_in, weights, T, K, ids_out, expert_class, reroute_map,
                   active_list, n_active, y_partial, nullptr, workspace, workspace_bytes, status_dev,
                   static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- expert parallel, peer memory
static_assert(sizeof(sere_ep_peers) == sizeof(EpPeers), "sere_ep_peers must mirror EpPeers");
static_assert(offsetof(sere_ep_peers, flags) == offsetof(EpPeers, flags), "sere_ep_peers must mirror EpPeers");
static_assert(SERE_MAX_EP_RANKS == kMaxEpRanks, "rank limit");

static int ep_peers(const sere_ep_peers* in, EpPeers* out) {
  if (in == nullptr || in->world < 1 || in->world > kMaxEpRanks || in->rank < 0 || in->rank >= in->world)
    return SERE_ERR_CONFIG;
  std::memcpy(out, in, sizeof(EpPeers));
  for (int r = 0; r < in->world; ++r)
    if (!out->h_all[r] || !out->ids_all[r] || !out->w_all[r] || !out->flags[r]) return SERE_ERR_DIMENSION;
  if (out->epoch != nullptr && (out->status == nullptr || out->arrivals == nullptr || out->timeout_ns <= 0))
    return SERE_ERR_DIMENSION;
  return SERE_OK;
}

int sere_route_topk_ep(const sere_ep_peers* peers, const uint16_t* x_local, const uint16_t* w_router_t,
                       const float* bias, int T_local, int d_h, int M, int K, void* workspace,
                       size_t workspace_bytes, void* stream) {
  EpPeers ep;
  int rc = ep_peers(peers, &ep);
  if (rc != SERE_OK) return rc;
  if (T_local < 0 || d_h < 1 || M < 1 || K < 1) return SERE_ERR_DIMENSION;
  if (K > M) return SERE_ERR_CONFIG;
  if (ep.t0 < 0 || ep.t0 + T_local > ep.T_all) return SERE_ERR_DIMENSION;
  if (!route_fast_path(M, K, d_h) || M > kMaxExperts) return SERE_ERR_UNSUPPORTED;
  if (T_local == 0) return SERE_OK;
  if (!x_local || !w_router_t) return SERE_ERR_DIMENSION;
  if (workspace == nullptr || workspace_bytes < route_workspace_bytes(T_local, d_h, M)) return SERE_ERR_WORKSPACE;
  return check_cuda(launch_route_mma(reinterpret_cast<const __nv_bfloat16*>(x_local),
                                     reinterpret_cast<const __nv_bfloat16*>(w_router_t), bias, T_local, d_h, M, K,
                                     nullptr, nullptr, nullptr, workspace, static_cast<cudaStream_t>(stream), &ep));
}

int sere_ep_barrier(const sere_ep_peers* peers, int32_t* epoch_dev, int32_t* status_dev, int64_t timeout_ns,
                    void* stream) {
  EpPeers ep;
  const int rc = ep_peers(peers, &ep);
  if (rc != SERE_OK) return rc;
  if (epoch_dev == nullptr || timeout_ns <= 0) return SERE_ERR_DIMENSION;
  return check_cuda(launch_ep_barrier(ep, epoch_dev, status_dev, timeout_ns, static_cast<cudaStream_t>(stream)));
}

int sere_moe_ffn_ep(const void* bank, int M, int expert_lo, int expert_hi, int n_shared_local, int d_h, int d_m,
                    int activation, const double* sim, int S, double rho, int flags, const uint16_t* x_all,
                    const int32_t* ids_all, const float* w_all, int T_all, int K, int32_t* ids_out,
                    uint8_t* expert_class, int32_t* reroute_map, int32_t* active_list, int32_t* n_active,
                    void* workspace, size_t workspace_bytes, int32_t* status_dev, const sere_ep_peers* peers,
                    void* stream) {
  EpSync sync{};
  if (peers != nullptr) {
    EpPeers ep;
    const int rc = ep_peers(peers, &ep);
    if (rc != SERE_OK) return rc;
    if (ep.epoch == nullptr || ep.status == nullptr || ep.timeout_ns <= 0) return SERE_ERR_DIMENSION;
    sync = ep_sync_of(ep);
  }
  if (expert_lo < 0 || expert_hi > M || expert_hi < expert_lo) return SERE_ERR_DIMENSION;
  const int m_local = expert_hi - expert_lo;
  if (m_local + n_shared_local < 1) return SERE_ERR_DIMENSION;
  int rc = check_layer_shapes(M, n_shared_local, d_h, d_m, activation, T_all, K);
  if (rc != SERE_OK) return rc;
  rc = check_reroute_cfg(K, M, S, rho);
  if (rc != SERE_OK) return rc;
  if (sim == nullptr || ids_out == nullptr) return SERE_ERR_DIMENSION;
  if (T_all == 0) return SERE_OK;
  return run_layer(bank, M, expert_lo, m_local, n_shared_local, d_h, d_m, activation, sim, S, rho, flags,
                   MODE_REROUTE | MODE_ALIGN, x_all, ids_all, w_all, T_all, K, ids_out, expert_class, reroute_map,
                   active_list, n_active, nullptr, nullptr, workspace, workspace_bytes, status_dev,
                   static_cast<cudaStream_t>(stream), nullptr, nullptr, 0.f, /*do_combine=*/false,
                   sync.world > 0 ? &sync : nullptr);
}

int sere_combine_ep(const sere_ep_peers* peers, const int32_t* ids_rr, const void* workspace, int M_local,
                    int n_shared_local, int n_shared_total, int d_h, int d_m, int K, float* x_res, float* y_local,
                    float eps, void* stream) {
  EpPeers ep;
  int rc = ep_peers(peers, &ep);
  if (rc != SERE_OK) return rc;
  if (M_local < 0 || n_shared_local < 0 || n_shared_total < n_shared_local || d_h < 1 || d_m < 1 || K < 1)
    return SERE_ERR_DIMENSION;
  if (K + n_shared_total > 64) return SERE_ERR_UNSUPPORTED;
  for (int r = 0; r < ep.world; ++r)
    if (!ep.y_perm[r] || !ep.slot_row[r]) return SERE_ERR_DIMENSION;
  const int T_local = ep.T_all / ep.world;
  if (T_local * ep.world != ep.T_all || ep.t0 != ep.rank * T_local) return SERE_ERR_DIMENSION;
  if (T_local == 0) return SERE_OK;
  if (!ids_rr || !workspace || !x_res) return SERE_ERR_DIMENSION;
  const WsLayout L = ws_layout(ep.T_all, K, M_local, n_shared_local, d_h, d_m);
  uint8_t* ws = ws_base(workspace);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  stage_mark(4, st);
  const cudaError_t e = launch_combine(reinterpret_cast<const float*>(ws + L.y_perm), L.d, L.r_max,
                                       reinterpret_cast<const int32_t*>(ws + L.plan),
                                       reinterpret_cast<const int32_t*>(ws + L.slot_row), ep.w_all[ep.rank], T_local,
                                       K, n_shared_total, y_local, nullptr, x_res, nullptr, eps, st, &ep, ids_rr);
  stage_mark(5, st);
  return check_cuda(e);
}

int sere_alloc_peer(size_t bytes, void** out) {
  if (out == nullptr || bytes == 0) return SERE_ERR_DIMENSION;
  return check_cuda(cudaMalloc(out, bytes));
}
int sere_free_peer(void* ptr) { return check_cuda(cudaFree(ptr)); }
int sere_ipc_handle(void* base_ptr, uint8_t out_handle[64]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (base_ptr == nullptr || out_handle == nullptr) return SERE_ERR_DIMENSION;
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, base_ptr);
  if (e != cudaSuccess) return SERE_ERR_CUDA;
  std::memcpy(out_handle, &h, 64);
  return SERE_OK;
}
int sere_ipc_open(const uint8_t handle[64], void** out_ptr) {
  if (handle == nullptr || out_ptr == nullptr) return SERE_ERR_DIMENSION;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  return check_cuda(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess));
}
int sere_ipc_close(void* ptr) { return check_cuda(cudaIpcCloseMemHandle(ptr)); }

size_t sere_route_workspace_bytes(int T, int d_h, int M) {
  if (T < 0 || d_h < 1 || M < 1) return 0;
  return route_workspace_bytes(T, d_h, M);
}

int sere_route_topk(const uint16_t* x, const uint16_t* w_router_t, const float* bias, int T, int d_h, int M, int K,
                    int32_t* ids, float* weights, float* logits_out, void* workspace, size_t workspace_bytes,
                    void* stream) {
  if (T < 0 || d_h < 1 || M < 1 || K < 1) return SERE_ERR_DIMENSION;
  if (K > M || K > 32 || M > kMaxExperts) return K > M ? SERE_ERR_CONFIG : SERE_ERR_UNSUPPORTED;
  if (T == 0) return SERE_OK;
  if (!x || !w_router_t || !ids || !weights) return SERE_ERR_DIMENSION;
  const __nv_bfloat16* w_router = reinterpret_cast<const __nv_bfloat16*>(w_router_t);
  if (route_fast_path(M, K, d_h)) {
    if (workspace == nullptr || workspace_bytes < route_workspace_bytes(T, d_h, M)) return SERE_ERR_WORKSPACE;
    return check_cuda(launch_route_mma(reinterpret_cast<const __nv_bfloat16*>(x), w_router, bias, T, d_h, M, K, ids,
                                       weights, logits_out, workspace, static_cast<cudaStream_t>(stream)));
  }
  return check_cuda(launch_route_topk(reinterpret_cast<const __nv_bfloat16*>(x),
                                      reinterpret_cast<const __nv_bfloat16*>(w_router), bias, T, d_h, M, K, ids,
                                      weights, logits_out, static_cast<cudaStream_t>(stream)));
}

int sere_residual_rmsnorm(float* x, const float* y, uint16_t* h_out, int T, int d_h, float eps, void* stream) {
  if (T < 0 || d_h < 1) return SERE_ERR_DIMENSION;
  if (T == 0) return SERE_OK;
  if (!x || !h_out) return SERE_ERR_DIMENSION;
  return check_cuda(launch_residual_rmsnorm(x, y, reinterpret_cast<__nv_bfloat16*>(h_out), T, d_h, eps,
                                            static_cast<cudaStream_t>(stream)));
}

int sere_debug_set_align_clocks(int64_t* dev_buf) {
  g_align_dbg = reinterpret_cast<long long*>(dev_buf);
  return SERE_OK;
}

int sere_debug_set_ffn_trace(uint64_t* dev_buf) {
  g_ffn_trace = reinterpret_cast<unsigned long long*>(dev_buf);
  return SERE_OK;
}

int sere_debug_replay_ffn(const void* bank, int M, int n_shared, int d_h, int d_m, int activation, int T, int K,
                          void* workspace, size_t workspace_bytes, int reps, void* stream) {
  int rc = check_layer_shapes(M, n_shared, d_h, d_m, activation, T, K);
  if (rc != SERE_OK) return rc;
  if (!bank || !workspace || reps < 0) return SERE_ERR_DIMENSION;
  const WsLayout L = ws_layout(T, K, M, n_shared, d_h, d_m);
  if (workspace_bytes < L.total) return SERE_ERR_WORKSPACE;
  FfnParams fp = ffn_params(bank, L, ws_base(workspace), activation);
  for (int i = 0; i < reps; ++i) {
    const cudaError_t e = launch_moe_ffn(fp, num_sms(), static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return SERE_ERR_CUDA;
  }
  return SERE_OK;
}

int sere_set_pdl(int enable) {
  g_pdl = enable & PDL_ALL;
  return SERE_OK;
}

int sere_set_l2(int flags) {
  g_l2 = flags & L2_ALL;
  return SERE_OK;
}

int sere_debug_set_route_clocks(int64_t* dev_buf) {
  g_route_dbg = reinterpret_cast<long long*>(dev_buf);
  return SERE_OK;
}

int sere_debug_set_ffn_mode(int mode) {
  g_ffn_dbg_mode = mode;
  return SERE_OK;
}

int sere_set_stage_events(void* const* events, int n) {
  if (n != 0 && n != kStageEvents) return SERE_ERR_DIMENSION;
  if (n == 0 || events == nullptr) {
    t_stage_events_on = false;
    return SERE_OK;
  }
  for (int i = 0; i < kStageEvents; ++i) t_stage_events[i] = static_cast<cudaEvent_t>(events[i]);
  t_stage_events_on = true;
  return SERE_OK;
}

}  // extern "C"
