// params.cuh -- launch parameter blocks shared by the kernels and capi.cu.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "plan.cuh"

namespace sere {

enum : int { MODE_REROUTE = 1, MODE_ALIGN = 2 };
enum : int { EPI_SWIGLU = 0, EPI_STORE_F32 = 1 };

// Fused expert-parallel barrier (ep_p2p.cu): the kernel that ends a phase ARRIVES (its last
// CTA bumps this rank's epoch and release-stores it into every rank's flag slot), the first
// kernel of the next phase WAITS (one thread acquires every rank's slot >= its own epoch).
// world == 0: no fused barrier.
constexpr int kMaxEpRanks = 8;
struct EpSync {
  int world, rank;
  int32_t* flags[kMaxEpRanks];  // every rank's flag words (kEpFlagWords each)
  int32_t* epoch;               // this rank's epoch counter
  int32_t* status;              // this rank's barrier status word (SERE_ERR_CUDA on timeout / abort)
  long long timeout_ns;
  unsigned long long* wait_ns;  // optional: accumulated wait time [0] align side, [1] combine side
  int wait_slot;
};

struct AlignParams {
  const int32_t* ids_in;
  const double* sim;
  int T, K, M, S, n_shared;
  double rho;
  int flags, mode;
  // re-routing outputs (any may be null)
  int32_t* ids_out;
  uint8_t* expert_class;
  int32_t* reroute_map;
  int32_t* active_list;
  int32_t* n_active;
  int32_t* status_dev;
  // align outputs
  int32_t* plan;
  int32_t* row_token;  // padding rows are marked -1 here; the permute writes the token rows
  int tiles_gu, tiles_dn, ksplit_dn;  // FFN geometry (work units: plan.cuh group_units_*)
  int e_lo, m_local; // expert-parallel ownership: bank holds global experts [e_lo, e_lo+m_local)
  int r_max;         // rows of the permuted batch buffer (row_token is staged in smem when it fits)
  int ffn_ctas;      // grid of the fused FFN (its first wave of gate/up units)
  long long* dbg;    // optional phase timestamps (sere_debug_set_align_clocks)
  int32_t* ids_final;     // [T,K] the (re-routed) table the layer runs on (align mode; the permute reads it)
  uint16_t* blk_prefix;   // [TB][Et] cells of bank expert e in token blocks before tb (align mode)
  EpSync sync;            // expert parallel: wait for every rank's router rows before reading the table
  int stage_sim;          // set by launch_reroute_align: the sim is bulk-copied into shared memory
};

struct FfnParams {
  const uint8_t* w13;  // gate/up tiles (expert, mt, kt) at ((expert*tiles_gu+mt)*ktiles_gu+kt)*16KB
  const uint8_t* w2;   // down tiles   (expert, mt, kt) at ((expert*tiles_dn+mt)*ktiles_dn+kt)*16KB
  int tiles_gu, ktiles_gu, tiles_dn, ktiles_dn, ksplit_dn;
  const uint8_t* x_pack;  // gate/up B operand [ktiles_gu][r_max][128 B]
  uint8_t* h_pack;        // SwiGLU out = down B operand [ktiles_dn][r_max][128 B]
  float* y_perm;          // down out [ksplit_dn][r_max][d_h_pad]
  int r_max, d_h_pad;
  int32_t* plan;          // written by reroute_align; the ticket and dep counters are updated here
  int Et;
  int act;
  int dbg_mode;               // debug experiments (results invalid): bit0 skip weight copies, bit1 skip MMAs,
                              // bit2 skip the expert-output stores
  unsigned long long* trace;  // optional per-CTA unit timeline (sere_debug_set_ffn_trace), kFfnTraceStride u64 each
  EpSync sync;                // expert parallel: the last CTA out arrives (expert outputs final)
};
constexpr int kFfnTraceStride = 2048;
constexpr int kFfnTraceUnits = 200;

extern long long* g_route_dbg;

// launch with programmatic stream serialisation (PDL); `pdl` false = ordinary launch
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// The max-dynamic-shared-memory attribute is per device: each launcher keeps the largest
// size it has set for every device (a second GPU in the same process sets its own).
constexpr int kMaxDevices = 64;
struct SmemAttrCache {
  size_t configured[kMaxDevices] = {};
};
template <typename Kernel>
inline cudaError_t ensure_smem_attr(Kernel kernel, size_t smem, SmemAttrCache& cache, size_t default_cap = 48 * 1024) {
  if (smem <= default_cap) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < kMaxDevices && cache.configured[dev] >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess && dev >= 0 && dev < kMaxDevices) cache.configured[dev] = smem;
  return e;
}

// Expert-parallel group seen through NVLink peer memory (ep_p2p.cu; world == 0: single GPU).
// Every pointer array is indexed by rank; entry `rank` is this rank's own buffer.
struct EpPeers {
  int world, rank;
  int t0, T_all;                      // this rank's first global token; tokens of the whole batch
  int e_lo[kMaxEpRanks + 1];          // routed-expert blocks: rank r owns [e_lo[r], e_lo[r+1])
  int nsh[kMaxEpRanks];               // shared experts owned by rank r (s % world == r)
  int r_max[kMaxEpRanks];             // rank r's permuted-row capacity (its y_perm split stride / d_h_pad)
  const float* y_perm[kMaxEpRanks];   // rank r's down-GEMM outputs
  const int32_t* slot_row[kMaxEpRanks];
  __nv_bfloat16* h_all[kMaxEpRanks];  // rank r's gathered token states [T_all][d_h]
  int32_t* ids_all[kMaxEpRanks];      // rank r's gathered router ids [T_all][K]
  float* w_all[kMaxEpRanks];          // rank r's gathered router weights [T_all][K]
  int32_t* flags[kMaxEpRanks];        // rank r's barrier flags [kEpFlagWords]
  // this rank's fused-barrier state (epoch == nullptr: no fused barriers, sere_ep_barrier instead)
  int32_t* epoch;
  int32_t* status;
  int32_t* arrivals;                  // router CTAs done (the last one arrives)
  long long timeout_ns;
  unsigned long long* wait_ns;        // optional barrier wait accumulators (see EpSync)
};

// flags[r] holds kMaxEpRanks barrier slots followed by rank r's sticky ABORT word: a
// barrier that times out stores 1 into every rank's abort word; every later barrier fails
// fast and the kernels that touch peer memory (router dispatch stores, combine loads/stores)
// skip their peer accesses, so no rank proceeds on a half-synchronised step.
constexpr int kEpAbortSlot = kMaxEpRanks;
constexpr int kEpFlagWords = kMaxEpRanks + 1;
__device__ __forceinline__ void st_release_sys(int32_t* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool ep_aborted(const EpPeers& ep) {
  return ld_acquire_sys(ep.flags[ep.rank] + kEpAbortSlot) != 0;
}
__host__ __device__ inline EpSync ep_sync_dev(const EpPeers& ep) {
  EpSync s{};
  s.world = ep.world;
  s.rank = ep.rank;
  for (int r = 0; r < kMaxEpRanks; ++r) s.flags[r] = ep.flags[r];
  s.epoch = ep.epoch;
  s.status = ep.status;
  s.timeout_ns = ep.timeout_ns;
  s.wait_ns = ep.wait_ns;
  s.wait_slot = 1;  // the combine side
  return s;
}
inline EpSync ep_sync_of(const EpPeers& ep) {
  EpSync s{};
  if (ep.epoch == nullptr) return s;
  s.world = ep.world;
  s.rank = ep.rank;
  for (int r = 0; r < kMaxEpRanks; ++r) s.flags[r] = ep.flags[r];
  s.epoch = ep.epoch;
  s.status = ep.status;
  s.timeout_ns = ep.timeout_ns;
  s.wait_ns = ep.wait_ns;
  s.wait_slot = 0;  // the align side
  return s;
}
// one thread: this rank's writes so far (made system-visible by the caller's fences) are
// published to every rank under a new epoch
__device__ __forceinline__ void ep_arrive(const EpSync& s) {
  __threadfence_system();
  const int e = atomicAdd(s.epoch, 1) + 1;
  for (int p = 0; p < s.world; ++p) st_release_sys(s.flags[p] + s.rank, e);
}
// one thread: wait until every rank arrived at this rank's current epoch; false on a timeout
// (sticky abort raised on every rank) or when an abort is already raised
__device__ __forceinline__ bool ep_wait(const EpSync& s) {
  if (ld_acquire_sys(s.flags[s.rank] + kEpAbortSlot) != 0) {
    if (s.status) atomicExch(s.status, 6 /* SERE_ERR_CUDA */);
    return false;
  }
  const int e = *reinterpret_cast<volatile int32_t*>(s.epoch);
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int p = 0; p < s.world; ++p) {
    while (ld_acquire_sys(s.flags[s.rank] + p) < e) {
      __nanosleep(64);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > static_cast<unsigned long long>(s.timeout_ns)) {
        if (s.status) atomicExch(s.status, 6 /* SERE_ERR_CUDA */);
        for (int q = 0; q < s.world; ++q) st_release_sys(s.flags[q] + kEpAbortSlot, 1);
        return false;
      }
    }
  }
  if (s.wait_ns) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicAdd(s.wait_ns + s.wait_slot, t - t0);
  }
  __threadfence();
  return true;
}

// programmatic dependent launch per layer-chain kernel (sere_set_pdl bit mask)
enum : int { PDL_ALIGN = 1, PDL_PERMUTE = 2, PDL_FFN = 4, PDL_COMBINE = 8, PDL_RMSNORM = 16, PDL_ALL = 31 };
extern int g_pdl;  // capi.cu
// L2 policy for the per-layer scratch (sere_set_l2 bit mask). y_perm (the fp32 expert outputs)
// is rewritten every layer at the same addresses, so its dirty lines are dead once the combine
// has read them; written back to DRAM they cost ~30 MB of HBM writes per C4 layer, competing with
// the next layer's weight stream (profiles/r02_l2_scratch_discard.txt).
//   L2_DISCARD_Y: the next layer's permute CTAs drop the previous expert outputs from L2
//                 (discard.global.L2) before their PDL wait, while re-route/align runs
enum : int { L2_DISCARD_Y = 1, L2_ALL = 1 };
extern int g_l2;  // capi.cu

cudaError_t launch_reroute_align(const AlignParams& p, cudaStream_t stream);
size_t reroute_align_smem(int T, int K, int M, int Et);
cudaError_t launch_pack(const __nv_bfloat16* wg, const __nv_bfloat16* wu, const __nv_bfloat16* wd, int count,
                        const Dims& d, int Et, int first, uint8_t* bank, int unpack, cudaStream_t stream);
cudaError_t launch_permute(const __nv_bfloat16* x, const Dims& d, const int32_t* plan, int Et, int m_loc, int e_lo,
                           const int32_t* ids_final, const uint16_t* blk_prefix, int T, int K, int n_shared,
                           int32_t* slot_row, int32_t* row_token, int r_max, uint8_t* x_pack, cudaStream_t stream,
                           const float* y_dead = nullptr, long long y_lines = 0, bool x_early = false);
cudaError_t launch_combine(const float* y_perm, const Dims& d, int r_max, const int32_t* plan,
                           const int32_t* slot_row, const float* w, int T, int K, int n_shared, float* y,
                           __nv_bfloat16* y_bf16, float* x_res, __nv_bfloat16* h_next, float eps,
                           cudaStream_t stream, const EpPeers* ep = nullptr, const int32_t* ids_rr = nullptr);
cudaError_t launch_moe_ffn(const FfnParams& p, int num_sms, cudaStream_t stream);
size_t moe_ffn_smem(int Et);
cudaError_t launch_route_topk(const __nv_bfloat16* x, const __nv_bfloat16* w_router, const float* bias, int T,
                              int d_h, int M, int K, int32_t* ids, float* weights, float* logits_out,
                              cudaStream_t stream);
cudaError_t launch_route_mma(const __nv_bfloat16* x, const __nv_bfloat16* w_router, const float* bias, int T,
                             int d_h, int M, int K, int32_t* ids, float* weights, float* logits_out, void* ws,
                             cudaStream_t stream, const EpPeers* ep = nullptr);
cudaError_t launch_ep_barrier(const EpPeers& ep, int32_t* epoch, int32_t* status, long long timeout_ns,
                              cudaStream_t stream);
size_t route_workspace_bytes(int T, int d_h, int M);
bool route_fast_path(int M, int K, int d_h);
cudaError_t launch_residual_rmsnorm(float* x, const float* y, __nv_bfloat16* h_out, int T, int d_h, float eps,
                                    cudaStream_t stream);

}  // namespace sere
