/*
 * sere_b200.h -- C-ABI of the B200-native SERE batched-decode MoE path.
 *
 * The reference (`/root/reference/pkg/src/sere`) is pure Python; it has no FFI.
 * Its operator boundary is two module-level functions that `moe.model_forward`
 * resolves at call time (moe.py:368 and moe.py:375):
 *
 *   rerouting.apply_sere(assignment, sim, config) -> RerouteResult   (rerouting.py:130-171)
 *   moe.layer_forward(layer, x, assignment, activation) -> ndarray    (moe.py:280-310)
 *
 * Every entry point below replaces one of those (or a stage inside them) and is
 * what a ctypes binding of the reference would call.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers, caller-owned, dense row-major.
 *    The library never frees caller memory and keeps no pointer after the
 *    stream work completes. `stream` is a cudaStream_t (NULL = legacy stream).
 *  - Every call is asynchronous and stream-ordered; none synchronises the host.
 *  - Return value: host-side status (shape/config checks, launch errors).
 *    Data-dependent checks that the reference performs on every call (ids out
 *    of range, similarity outside [0,1]) run on the device and are reported
 *    through `status_dev` (one int32, device memory, SERE_OK on success); read
 *    it after the stream completes. Kernels downstream of a failed check do no
 *    work. Codes map 1:1 onto the reference exceptions (errors.py:9-34).
 *  - Expert ids are int32 (the reference uses int64; values are identical).
 *  - bf16 tensors are passed as uint16_t* (raw bf16 bits).
 */
#ifndef SERE_B200_H_
#define SERE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SERE_ABI_VERSION 2

/* status codes  (paper_2602_07616_b200/errors.py keeps the same numbers) */
enum {
  SERE_OK = 0,
  SERE_ERR_CONFIG = 1,      /* ConfigError    : S<1, S>K, rho outside [0,1], bad activation */
  SERE_ERR_DIMENSION = 2,   /* DimensionError : shapes; id outside [0,M) in re-routing (rerouting.py:111-114) */
  SERE_ERR_INPUT = 3,       /* InputError     : similarity outside [0,1] (rerouting.py:115-116) */
  SERE_ERR_ROUTING = 4,     /* RoutingError   : id outside [0,M) in layer_forward (moe.py:299-300) */
  SERE_ERR_DOMAIN = 5,      /* DomainError    : non-finite inputs */
  SERE_ERR_CUDA = 6,        /* CUDA launch / runtime failure */
  SERE_ERR_UNSUPPORTED = 7, /* device is not sm_100 / limits exceeded */
  SERE_ERR_WORKSPACE = 8    /* workspace too small */
};

/* per-expert classification written by sere_reroute (bit flags) */
enum {
  SERE_CLASS_PRIMARY = 1,  /* in the batch primary set (union of slots < S)      rerouting.py:147 */
  SERE_CLASS_CRITICAL = 2, /* secondary kept because best sim < rho (rho > 0)    rerouting.py:160-161 */
  SERE_CLASS_REROUTED = 4  /* secondary redirected; target in reroute_map[e]    rerouting.py:162-164 */
};

/* Expert id the router writes for a token whose logits are not all finite (a non-finite
 * token state; the reference's route_topk raises DomainError, moe.py:274-275). The
 * re-routing / align kernels report it as SERE_ERR_DOMAIN. */
#define SERE_ID_NONFINITE ((int32_t)0x80000000)

/* activations of moe.py:22 */
enum { SERE_ACT_SILU = 0, SERE_ACT_RELU = 1, SERE_ACT_GELU_TANH = 2 };

/* flags for sere_reroute / sere_moe_forward */
enum {
  SERE_FLAG_CHECK_SIM = 1 /* validate sim in [0,1] on the device (InputError); the Python
                             drop-in (apply_sere) sets it on every call, as the reference
                             validates on every call (rerouting.py:140); the device-level
                             API validates once per uploaded DeviceSimilarity */
};

int sere_abi_version(void);
const char* sere_status_string(int status);

/* Returns SERE_OK iff `device` is an sm_100 part the kernels were built for. */
int sere_device_check(int device);

/* ------------------------------------------------------------------------
 * (1) Re-routing.  Replaces rerouting.apply_sere (rerouting.py:130-171),
 *     equivalently the Alg. 2 kernel contract apply_sere_parallel (174-249).
 *
 *  ids_in     int32 [T,K]  top-k expert ids, slot 0 strongest (RoutingAssignment.indices)
 *  sim        f64   [M,M]  similarity, row = secondary u, column = candidate v
 *  S, rho     retain_count and threshold of RerouteConfig (rerouting.py:31-54)
 *  ids_out    int32 [T,K]  RerouteResult.new_indices, bit-exact
 *  expert_class u8 [M]     SERE_CLASS_* flags (0 = expert not routed to)
 *  reroute_map int32 [M]   target of a SERE_CLASS_REROUTED expert, else -1
 *                          (reference NaN quirk: a rerouted expert may map to -1)
 *  active_list int32 [M]   final_active, ascending; n_active int32[1] its length
 *  Weights are never read nor written (the reference leaves them untouched).
 * ------------------------------------------------------------------------ */
int sere_reroute(const int32_t* ids_in, const double* sim, int T, int K, int M, int S, double rho,
                 int flags, int32_t* ids_out, uint8_t* expert_class, int32_t* reroute_map,
                 int32_t* active_list, int32_t* n_active, int32_t* status_dev, void* stream);

/* ------------------------------------------------------------------------
 * (2) Expert bank: the layer's routed experts [0,M) followed by its shared
 *     experts [M, M+n_shared), bf16, in the tcgen05 tile layout.
 *     sere_pack_experts converts `count` experts from the reference orientation
 *     (ExpertWeights moe.py:70-77: w_gate,w_up [d_h,d_m], w_down [d_m,d_h],
 *     row-major, here bf16) into bank slots [first, first+count).
 * ------------------------------------------------------------------------ */
size_t sere_expert_bank_bytes(int n_experts_total, int d_h, int d_m);
int sere_pack_experts(const uint16_t* w_gate, const uint16_t* w_up, const uint16_t* w_down, int count,
                      int d_h, int d_m, void* bank, int n_experts_total, int first, void* stream);
/* Inverse of sere_pack_experts (for checkpoints / tests). */
int sere_unpack_experts(const void* bank, int n_experts_total, int first, int count, int d_h, int d_m,
                        uint16_t* w_gate, uint16_t* w_up, uint16_t* w_down, void* stream);

/* ------------------------------------------------------------------------
 * (3) MoE layer forward.  Replaces moe.layer_forward (moe.py:280-310):
 *     y[t] = sum_k w[t,k] * E_{ids[t,k]}(x[t])  (slot order 0..K-1)  + sum_s E_shared_s(x[t])
 *     E(x) = act(x Wg) * (x Wu) Wd.  Duplicate ids in a row contribute once per slot.
 *
 *  x          bf16 [T,d_h];  ids int32 [T,K];  weights f32 [T,K]
 *  y          f32  [T,d_h]   (required);  y_bf16 bf16 [T,d_h] (optional, may be NULL)
 *  workspace  >= sere_layer_workspace_bytes(...) bytes, 256-B aligned.
 *  Data-dependent error: id outside [0,M) -> SERE_ERR_ROUTING in status_dev.
 * ------------------------------------------------------------------------ */
size_t sere_layer_workspace_bytes(int T, int K, int M, int n_shared, int d_h, int d_m);
int sere_layer_forward(const void* bank, int M, int n_shared, int d_h, int d_m, int activation,
                       const uint16_t* x, const int32_t* ids, const float* weights, int T, int K,
                       float* y, uint16_t* y_bf16, void* workspace, size_t workspace_bytes,
                       int32_t* status_dev, void* stream);

/* ------------------------------------------------------------------------
 * (4) Fused SERE layer: sere_reroute + sere_layer_forward on the rewritten ids
 *     (the body of moe.model_forward's loop, moe.py:367-375) with the
 *     re-routing, count/align and permute fused into one launch pair.
 *     Pass S == K (or rho == 1 with off-diagonal sims < 1) for plain top-k on
 *     the same kernels.  Re-routing outputs as in sere_reroute (all optional
 *     except ids_out may be NULL too).
 * ------------------------------------------------------------------------ */
int sere_moe_forward(const void* bank, int M, int n_shared, int d_h, int d_m, int activation,
                     const double* sim, int S, double rho, int flags, const uint16_t* x,
                     const int32_t* ids_in, const float* weights, int T, int K, int32_t* ids_out,
                     uint8_t* expert_class, int32_t* reroute_map, int32_t* active_list,
                     int32_t* n_active, float* y, uint16_t* y_bf16, void* workspace,
                     size_t workspace_bytes, int32_t* status_dev, void* stream);

/* ------------------------------------------------------------------------
 * (4a) Decode block = (4) with the residual add and the next layer's RMSNorm fused
 *     into the combine pass: x_residual += MoE(h);  h_next = bf16(x_residual *
 *     rsqrt(mean(x_residual^2) + eps)).  y (f32 [T,d_h]) is optional (NULL skips it).
 *     The Qwen3-style pre-norm block of the 48-layer benchmark step.
 * ------------------------------------------------------------------------ */
int sere_moe_block_forward(const void* bank, int M, int n_shared, int d_h, int d_m, int activation,
                           const double* sim, int S, double rho, int flags, const uint16_t* h,
                           const int32_t* ids_in, const float* weights, int T, int K, int32_t* ids_out,
                           uint8_t* expert_class, int32_t* reroute_map, int32_t* active_list,
                           int32_t* n_active, float* x_residual, uint16_t* h_next, float eps, float* y,
                           void* workspace, size_t workspace_bytes, int32_t* status_dev, void* stream);

/* ------------------------------------------------------------------------
 * (4b) Expert-parallel shard of (4): the bank holds only global experts
 *     [expert_lo, expert_hi) (as bank slots 0..) plus n_shared_local shared
 *     experts. Re-routing runs on the FULL gathered [T,K] table (every rank
 *     computes the same bit-exact ids), then only this rank's experts are
 *     evaluated; y_partial [T,d_h] f32 = this rank's share of moe.layer_forward's
 *     sum (slot order kept). Ranks' partials are summed by the caller's
 *     reduce-scatter (paper_2602_07616_b200/ep.py). Workspace: size it with
 *     sere_layer_workspace_bytes(T, K, expert_hi-expert_lo, n_shared_local, ...).
 * ------------------------------------------------------------------------ */
int sere_moe_forward_ep(const void* bank, int M, int expert_lo, int expert_hi, int n_shared_local, int d_h,
                        int d_m, int activation, const double* sim, int S, double rho, int flags,
                        const uint16_t* x, const int32_t* ids_in, const float* weights, int T, int K,
                        int32_t* ids_out, uint8_t* expert_class, int32_t* reroute_map,
                        int32_t* active_list, int32_t* n_active, float* y_partial, void* workspace,
                        size_t workspace_bytes, int32_t* status_dev, void* stream);

/* ------------------------------------------------------------------------
 * (5) Router: logits = x W_r (fp32 accumulate), top-K with ties to the lower
 *     index, softmax over the K picks.  Replaces moe.route_topk / topk_softmax
 *     (moe.py:248-277).
 *  w_router_t bf16 [M, d_h]: RouterWeights.w_router TRANSPOSED (expert-major, K
 *     contiguous -- converted once at load, the router is static).
 *  bias f32 [M] (nullable) is added to the logits before selection: the benchmark's
 *     expert-popularity skew knob; NULL reproduces moe.route_topk.
 *  logits_out f32 [T,M] (nullable).  workspace: >= sere_route_workspace_bytes(T,d_h,M)
 *     bytes, ZERO-FILLED before its first use (it holds per-tile tickets that every
 *     launch leaves at zero again).
 * ------------------------------------------------------------------------ */
size_t sere_route_workspace_bytes(int T, int d_h, int M);
int sere_route_topk(const uint16_t* x, const uint16_t* w_router_t, const float* bias, int T, int d_h, int M,
                    int K, int32_t* ids, float* weights, float* logits_out, void* workspace,
                    size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * (6) Decode-block glue: x += y (fp32 residual stream, y nullable) and
 *     h = bf16(x * rsqrt(mean(x^2) + eps)) -- the pre-norm of a Qwen3-style MoE block
 *     used by the 48-layer benchmark step (not part of the reference model).
 * ------------------------------------------------------------------------ */
int sere_residual_rmsnorm(float* x, const float* y, uint16_t* h_out, int T, int d_h, float eps, void* stream);

/* Programmatic dependent launch on the layer-chain kernels: a kernel may become resident
 * while its predecessor drains and waits on-device (griddepcontrol) before touching shared
 * data. `enable` is a bit mask of the kernels launched that way: 1 re-route/align,
 * 2 permute, 4 FFN, 8 combine, 16 RMSNorm (31 = all; 0 = plain stream order). */
int sere_set_pdl(int enable);

/* L2 policy of the per-layer scratch (bit mask): 1 (default) the next layer's permute drops the
 * previous layer's expert outputs from L2 (discard.global.L2) before its programmatic-launch wait,
 * so their dead dirty lines are not written back to DRAM during the next weight stream
 * (single-GPU calls only). Results are identical for every value. */
int sere_set_l2(int flags);


/* Profiling hook: when n == 6, every following layer call on this host thread records
 * events[0..4] before its five stages (align, permute, gate/up GEMM, down GEMM,
 * combine) and events[5] after the last, on the launch stream (cudaEvent_t handles).
 * n == 0 disables. */
int sere_set_stage_events(void* const* events, int n);

/* Debug: when non-NULL, the re-routing/align kernel writes clock64() after each of its
 * barrier-separated phases into dev_buf[0..15] (device int64). NULL disables. */
int sere_debug_set_align_clocks(int64_t* dev_buf);

/* Debug: when non-NULL, the fused FFN kernel writes a per-CTA timeline (globaltimer ns)
 * into dev_buf[cta * 1024 .. +1024] (device uint64, >= num_SMs * 1024 entries):
 * [0] start, [1] producer slot-wait, [2] MMA operand-wait, [3] units, [4] producer
 * dependency-wait, [5] MMA accumulator-wait, [6] epilogue wait, [7] end,
 * [8+4i] unit i: ticket, t_ticket, t_first_copy, t_last_copy; [816+i] unit i epilogue done.
 * NULL disables. */
int sere_debug_set_ffn_trace(uint64_t* dev_buf);
/* Debug experiments on the fused FFN (outputs become INVALID): bit0 = skip the weight
 * copies, bit1 = skip the MMAs. 0 = normal operation. */
int sere_debug_set_ffn_mode(int mode);
/* Debug: router phase clocks (clock64) per CTA, dev_buf[cta * 8 + phase]. NULL disables. */
int sere_debug_set_route_clocks(int64_t* dev_buf);
/* Kernel-only timing: relaunch the fused expert FFN `reps` times on the plan and operands
 * the last sere_*forward call left in `workspace` (the FFN re-arms its ticket and
 * dependency counters when it finishes; outputs are rewritten with identical values). */
int sere_debug_replay_ffn(const void* bank, int M, int n_shared, int d_h, int d_m, int activation, int T, int K,
                          void* workspace, size_t workspace_bytes, int reps, void* stream);

/* ------------------------------------------------------------------------
 * (4c) Expert parallel over NVLink peer memory (replaces the NCCL
 *     all-gather / reduce-scatter choreography of (4b) -- the reference has no
 *     multi-GPU path, so these have no reference counterpart beyond moe.py:280-310).
 *     Each rank owns: gathered token states h_all bf16 [T_all,d_h], router ids_all
 *     i32 [T_all,K] and w_all f32 [T_all,K], barrier flags i32 [SERE_MAX_EP_RANKS + 1]
 *     (zeroed once; the last word is the rank's sticky abort word),
 *     and its layer workspace (y_perm / slot_row inside it, sere_layer_workspace_layout).
 *     All of them must be reachable from every rank (cudaIpcOpenMemHandle, see
 *     sere_ipc_*); sere_ep_peers lists every rank's pointers, entry `rank` = own.
 *     Per layer:  sere_route_topk_ep -> sere_ep_barrier -> sere_moe_ffn_ep ->
 *                 sere_ep_barrier -> sere_combine_ep,
 *     or, with the fused barriers (peers->epoch != NULL), 3 calls and no barrier kernels:
 *     the router's last CTA arrives, the re-route/align kernel of sere_moe_ffn_ep waits;
 *     the FFN's last CTA arrives, the combine waits.
 * ------------------------------------------------------------------------ */
#define SERE_MAX_EP_RANKS 8
typedef struct {
  int32_t world, rank;
  int32_t t0, T_all;                      /* this rank's first token; tokens of the batch       */
  int32_t e_lo[SERE_MAX_EP_RANKS + 1];    /* rank r owns routed experts [e_lo[r], e_lo[r+1])    */
  int32_t nsh[SERE_MAX_EP_RANKS];         /* shared experts s with s % world == r                */
  int32_t r_max[SERE_MAX_EP_RANKS];       /* sere_ws_layout.r_max of rank r's workspace          */
  const float* y_perm[SERE_MAX_EP_RANKS]; /* rank r: workspace + off_y_perm                      */
  const int32_t* slot_row[SERE_MAX_EP_RANKS]; /* rank r: workspace + off_slot_row               */
  uint16_t* h_all[SERE_MAX_EP_RANKS];
  int32_t* ids_all[SERE_MAX_EP_RANKS];
  float* w_all[SERE_MAX_EP_RANKS];
  int32_t* flags[SERE_MAX_EP_RANKS];
  /* this rank's fused-barrier state; epoch == NULL: no fused barriers (call sere_ep_barrier) */
  int32_t* epoch;    /* device epoch counter (zeroed once; shared with sere_ep_barrier)     */
  int32_t* status;   /* device status word: SERE_ERR_CUDA after a timeout / abort           */
  int32_t* arrivals; /* device counter of router CTAs (zeroed once)                          */
  int64_t timeout_ns;
  uint64_t* wait_ns; /* optional device [2]: ns spent waiting in the fused barriers, added by
                        the re-route/align kernel [0] and the combine [1] (NULL: not measured) */
} sere_ep_peers;

/* Router for this rank's T_local = T_all/world tokens (x_local = own h_all rows
 * [t0, t0+T_local)); ids/weights rows are stored into EVERY rank's ids_all/w_all. */
int sere_route_topk_ep(const sere_ep_peers* peers, const uint16_t* x_local, const uint16_t* w_router_t,
                       const float* bias, int T_local, int d_h, int M, int K, void* workspace,
                       size_t workspace_bytes, void* stream);
/* Flag barrier over the group (one warp). epoch_dev: this rank's device counter (zeroed
 * once). On a wait longer than timeout_ns: SERE_ERR_CUDA in status_dev, no hang, and the
 * abort word of EVERY rank is set: from then on every rank's barriers fail fast and its
 * router / combine skip their peer stores and loads (the step's outputs are invalid and
 * each rank's status says so). */
int sere_ep_barrier(const sere_ep_peers* peers, int32_t* epoch_dev, int32_t* status_dev, int64_t timeout_ns,
                    void* stream);
/* (4b) without its combine: re-route + align + permute + fused FFN of this rank's experts
 * over the whole gathered batch; the expert outputs stay in the workspace for the peers. */
int sere_moe_ffn_ep(const void* bank, int M, int expert_lo, int expert_hi, int n_shared_local, int d_h, int d_m,
                    int activation, const double* sim, int S, double rho, int flags, const uint16_t* x_all,
                    const int32_t* ids_all, const float* w_all, int T_all, int K, int32_t* ids_out,
                    uint8_t* expert_class, int32_t* reroute_map, int32_t* active_list, int32_t* n_active,
                    void* workspace, size_t workspace_bytes, int32_t* status_dev, const sere_ep_peers* peers,
                    void* stream);
/* Combine of this rank's tokens from the owners' expert outputs (peer loads), fixed slot
 * order: x_res[t] += y[t]; every rank's h_all row t0+t = bf16(RMSNorm(x_res[t])).
 * ids_rr = this rank's re-routed ids [T_all,K] (sere_moe_ffn_ep ids_out; identical on
 * every rank). y_local f32 [T_local,d_h] (nullable) receives y itself. */
int sere_combine_ep(const sere_ep_peers* peers, const int32_t* ids_rr, const void* workspace, int M_local,
                    int n_shared_local, int n_shared_total, int d_h, int d_m, int K, float* x_res, float* y_local,
                    float eps, void* stream);
/* CUDA IPC helpers: a 64-byte handle of a cudaMalloc'd base pointer (sere_alloc_peer),
 * opened in another process of the same node. */
int sere_alloc_peer(size_t bytes, void** out);
int sere_free_peer(void* ptr);
int sere_ipc_handle(void* base_ptr, uint8_t out_handle[64]);
int sere_ipc_open(const uint8_t handle[64], void** out_ptr);
int sere_ipc_close(void* ptr);

/* ------------------------------------------------------------------------
 * Introspection of the workspace (tests read the count/align plan back).
 * ------------------------------------------------------------------------ */
typedef struct {
  size_t off_plan_i32;   /* int32 plan header + arrays              */
  size_t off_slot_row;   /* int32 [T*(K+n_shared)] permuted row of every (token, slot) */
  size_t off_row_token;  /* int32 [R_max] source token of each permuted row, -1 = pad */
  size_t off_x_pack;     /* bf16 [d_h_pad/64][R_max][64] swizzled activations          */
  size_t off_h_pack;     /* bf16 [d_m_pad/64][R_max][64] swizzled SwiGLU output        */
  size_t off_y_perm;     /* f32  [ksplit][R_max][d_h_pad] expert outputs               */
  size_t total_bytes;
  int32_t r_max;         /* rows reserved for the permuted batch                        */
  int32_t d_h_pad, d_m_pad, ksplit_down;
  int32_t plan_groups_off; /* int32 offsets (in elements) inside the plan block: */
  int32_t plan_group_expert_off, plan_group_row0_off, plan_group_rows_off;
  int32_t plan_counts_off, plan_unit_off_gu, plan_unit_off_dn;
  size_t off_ids_final;  /* int32 [T*K] the (re-routed) table the layer runs on            */
  size_t off_blk_prefix; /* u16 [ceil(T/32)][Et] cells of each bank expert in earlier token blocks */
} sere_ws_layout;

int sere_layer_workspace_layout(int T, int K, int M, int n_shared, int d_h, int d_m,
                                sere_ws_layout* out);

#ifdef __cplusplus
}
#endif
#endif /* SERE_B200_H_ */
