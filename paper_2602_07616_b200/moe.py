"""GPU-backed mirror of the reference MoE layer path (`sere.moe`).

The reference layer (`/root/reference/pkg/src/sere/moe.py`) is a fp64 numpy
loop; here one MoE layer is five stream-ordered sm_100a launches behind the
C-ABI (`sere_layer_forward` / `sere_moe_forward`):

    count/align (+ re-routing)  ->  permute  ->  gate/up tcgen05 GEMM (+SwiGLU)
    ->  down tcgen05 GEMM  ->  fixed-order combine

Public API, matching the reference names and argument meaning:
  * `layer_forward(layer, x, assignment, activation)`  drop-in for moe.py:280
    (host arrays in/out; `layer` a reference MoELayer or an ExpertBank);
  * `route_topk(router, x)` / `topk_softmax` semantics on the GPU (moe.py:248-277);
  * `model_forward(model, batch, config, sims, router_override)`  (moe.py:329-377);
  * device-level: `ExpertBank`, `layer_forward_device`, `moe_forward_device`,
    `route_topk_device` on CUDA tensors, no host sync.
Precision: bf16 weights and activations, fp32 accumulation and fp32 layer output
(SURVEY Appendix B), intermediate h rounded to bf16.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Callable, Sequence

import numpy as np

from . import _lib
from . import rerouting as _rr
from .errors import ConfigError, DimensionError, DomainError, RoutingError, raise_for_status

ACTIVATIONS = ("silu", "relu", "gelu-tanh")
PHASES = ("prefill", "decode")
_ACT_CODE = {"silu": 0, "relu": 1, "gelu-tanh": 2}


def _torch():
    import torch

    return torch


def activation_code(kind: str) -> int:
    try:
        return _ACT_CODE[kind]
    except KeyError:
        raise ConfigError(f"unknown activation {kind!r}, expected one of {ACTIVATIONS}") from None


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _dev_index(device) -> int:
    torch = _torch()
    d = torch.device(device)
    return d.index if d.index is not None else torch.cuda.current_device()


# ---------------------------------------------------------------------------
# expert bank (packed weights of one layer)
# ---------------------------------------------------------------------------

class ExpertBank:
    """One layer's routed experts [0,M) and shared experts [M, M+n_shared) as bf16
    tcgen05 tiles in HBM. Built from reference-orientation weights
    (ExpertWeights: w_gate/w_up [d_h,d_m], w_down [d_m,d_h]) by `sere_pack_experts`."""

    def __init__(self, n_experts: int, n_shared: int, d_h: int, d_m: int, device=None):
        torch = _torch()
        if n_experts < 1 or n_shared < 0 or d_h < 1 or d_m < 1:
            raise ConfigError("bank needs n_experts >= 1, n_shared >= 0, d_h, d_m >= 1")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        _lib.ensure_device(_dev_index(self.device))
        self.M, self.n_shared, self.d_h, self.d_m = int(n_experts), int(n_shared), int(d_h), int(d_m)
        self.n_total = self.M + self.n_shared
        nbytes = _lib.load().sere_expert_bank_bytes(self.n_total, self.d_h, self.d_m)
        self.data = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)  # padding tiles stay 0

    @property
    def weight_bytes_per_expert(self) -> int:
        return 2 * 3 * self.d_h * self.d_m

    def pack(self, w_gate, w_up, w_down, first: int = 0, stream=None) -> None:
        """Pack `count` experts (bf16 CUDA tensors [count,d_h,d_m] x2, [count,d_m,d_h]) into slots first.."""
        torch = _torch()
        wg, wu, wd = (t.to(device=self.device, dtype=torch.bfloat16).contiguous() for t in (w_gate, w_up, w_down))
        count = int(wg.shape[0])
        if wg.shape != (count, self.d_h, self.d_m) or wu.shape != wg.shape or wd.shape != (count, self.d_m, self.d_h):
            raise DimensionError("expert weight shapes do not match the bank")
        _lib.call("sere_pack_experts", wg.data_ptr(), wu.data_ptr(), wd.data_ptr(), count, self.d_h, self.d_m,
                  self.data.data_ptr(), self.n_total, int(first), _stream_ptr(stream))

    def unpack(self, first: int = 0, count: int | None = None, stream=None):
        """bf16 (w_gate, w_up, w_down) of bank slots [first, first+count) in the reference orientation."""
        torch = _torch()
        count = self.n_total - first if count is None else count
        wg = torch.empty((count, self.d_h, self.d_m), dtype=torch.bfloat16, device=self.device)
        wu = torch.empty_like(wg)
        wd = torch.empty((count, self.d_m, self.d_h), dtype=torch.bfloat16, device=self.device)
        _lib.call("sere_unpack_experts", self.data.data_ptr(), self.n_total, int(first), int(count), self.d_h,
                  self.d_m, wg.data_ptr(), wu.data_ptr(), wd.data_ptr(), _stream_ptr(stream))
        return wg, wu, wd

    @classmethod
    def from_reference_layer(cls, layer: Any, device=None) -> "ExpertBank":
        """Convert a reference MoELayer (fp64 numpy ExpertWeights) to a bf16 bank."""
        torch = _torch()
        experts = list(layer.experts) + list(getattr(layer, "shared_experts", ()))
        n_shared = len(getattr(layer, "shared_experts", ()))
        d_h, d_m = experts[0].w_gate.shape
        bank = cls(len(experts) - n_shared, n_shared, d_h, d_m, device)

        def stack(name):
            a = np.stack([np.asarray(getattr(e, name), dtype=np.float32) for e in experts])
            return torch.from_numpy(a).to(device=bank.device, dtype=torch.bfloat16)

        bank.pack(stack("w_gate"), stack("w_up"), stack("w_down"))
        return bank

    @classmethod
    def random(cls, n_experts: int, n_shared: int, d_h: int, d_m: int, seed: int = 0, device=None,
               keep_raw: bool = False, chunk: int = 16, expert_ids=None, shared_ids=None) -> "ExpertBank":
        """Seeded N(0, 1/d_h) bf16 weights drawn on the device (moe.py:405-413 distribution).

        Every expert has its own generator seed derived from (seed, global id), so an
        expert-parallel shard (`expert_ids` = the global routed ids it owns, `shared_ids`
        = the shared experts it owns) holds exactly the tensors of the full model.
        Experts are drawn and packed `chunk` at a time so raw weights never all coexist."""
        torch = _torch()
        expert_ids = list(range(n_experts)) if expert_ids is None else list(expert_ids)
        shared_ids = list(range(n_shared)) if shared_ids is None else list(shared_ids)
        bank = cls(len(expert_ids), len(shared_ids), d_h, d_m, device)
        bank.expert_ids, bank.shared_ids = expert_ids, shared_ids
        seeds = [int(seed) * 1_000_003 + e for e in expert_ids] + \
                [int(seed) * 1_000_003 + 10_000_000 + s for s in shared_ids]
        gen = torch.Generator(device=bank.device)
        scale = 1.0 / float(np.sqrt(d_h))
        raw = [] if keep_raw else None
        n = len(seeds)
        for first in range(0, n, chunk):
            c = min(chunk, n - first)
            wg = torch.empty((c, d_h, d_m), dtype=torch.bfloat16, device=bank.device)
            wu = torch.empty_like(wg)
            wd = torch.empty((c, d_m, d_h), dtype=torch.bfloat16, device=bank.device)
            for j in range(c):
                gen.manual_seed(seeds[first + j])
                wg[j] = torch.randn((d_h, d_m), generator=gen, device=bank.device) * scale
                wu[j] = torch.randn((d_h, d_m), generator=gen, device=bank.device) * scale
                wd[j] = torch.randn((d_m, d_h), generator=gen, device=bank.device) * scale
            bank.pack(wg, wu, wd, first)
            if raw is not None:
                raw.append((wg, wu, wd))
        if raw is not None:
            bank.raw = tuple(torch.cat([r[i] for r in raw]) for i in range(3))
        return bank


# ---------------------------------------------------------------------------
# workspace cache
# ---------------------------------------------------------------------------

_WS: dict = {}
_WS_RETIRED: list = []  # grown-out buffers are kept alive: a captured graph may still point at them


def workspace_bytes(T: int, K: int, M: int, n_shared: int, d_h: int, d_m: int) -> int:
    return int(_lib.load().sere_layer_workspace_bytes(T, K, M, n_shared, d_h, d_m))


def new_workspace(T: int, K: int, M: int, n_shared: int, d_h: int, d_m: int, device) -> Any:
    """A caller-owned layer workspace (plan, permutation, x/h packs, expert outputs). Anything
    that captures a CUDA graph or runs on its own stream owns one (DecodeStep does)."""
    torch = _torch()
    return torch.empty(max(workspace_bytes(T, K, M, n_shared, d_h, d_m), 1), dtype=torch.uint8, device=device)


def workspace(T: int, K: int, M: int, n_shared: int, d_h: int, d_m: int, device) -> Any:
    """Shared per-device workspace for ad-hoc calls on the current stream (grown on demand;
    a replaced buffer is retired, never freed)."""
    nbytes = workspace_bytes(T, K, M, n_shared, d_h, d_m)
    key = (str(device),)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            _WS_RETIRED.append(buf)
        buf = new_workspace(T, K, M, n_shared, d_h, d_m, device)
        _WS[key] = buf
    return buf


@dataclass
class LayerOutput:
    y: Any                  # f32 [T,d_h]
    y_bf16: Any | None
    status: Any             # int32 [1]
    reroute: Any | None = None  # rerouting.DeviceReroute for the fused path

    def check(self) -> None:
        raise_for_status(int(self.status.item()), "layer")


def _check_layer_inputs(bank: ExpertBank, x, ids, weights):
    torch = _torch()
    if x.ndim != 2 or x.shape[1] != bank.d_h:
        raise DimensionError(f"input width {tuple(x.shape)} does not match d_h {bank.d_h}")
    if ids.ndim != 2 or ids.shape[0] != x.shape[0] or weights.shape != ids.shape:
        raise DimensionError(f"assignment covers {tuple(ids.shape)} tokens, batch has {x.shape[0]}")
    if ids.shape[1] > bank.M:
        raise ConfigError(f"top_k must satisfy 1 <= K <= M (got K={ids.shape[1]}, M={bank.M})")
    return (x.to(torch.bfloat16).contiguous(), ids.to(torch.int32).contiguous(),
            weights.to(torch.float32).contiguous())


def layer_forward_device(bank: ExpertBank, x, ids, weights, activation: str = "silu", y=None, y_bf16=None,
                         status=None, stream=None, want_bf16: bool = False, ws=None) -> LayerOutput:
    """moe.py:280-310 on CUDA tensors: x bf16 [T,d_h], ids int32 [T,K], weights f32 [T,K]."""
    torch = _torch()
    x, ids, weights = _check_layer_inputs(bank, x, ids, weights)
    T, K = int(ids.shape[0]), int(ids.shape[1])
    dev = bank.device
    y = torch.empty((T, bank.d_h), dtype=torch.float32, device=dev) if y is None else y
    if want_bf16 and y_bf16 is None:
        y_bf16 = torch.empty((T, bank.d_h), dtype=torch.bfloat16, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev) if status is None else status
    ws = workspace(T, K, bank.M, bank.n_shared, bank.d_h, bank.d_m, dev) if ws is None else ws
    _lib.call("sere_layer_forward", bank.data.data_ptr(), bank.M, bank.n_shared, bank.d_h, bank.d_m,
              activation_code(activation), x.data_ptr(), ids.data_ptr(), weights.data_ptr(), T, K, y.data_ptr(),
              y_bf16.data_ptr() if y_bf16 is not None else None, ws.data_ptr(), ws.numel(), status.data_ptr(),
              _stream_ptr(stream))
    return LayerOutput(y, y_bf16, status)


def moe_forward_device(bank: ExpertBank, sim, retain_count: int, threshold: float, x, ids, weights,
                       activation: str = "silu", stream=None, want_bf16: bool = False,
                       out: LayerOutput | None = None, ws=None) -> LayerOutput:
    """Fused SERE layer (moe.py:367-375): re-route `ids` against `sim`, then run the
    layer on the rewritten ids with the ORIGINAL weights (moe.py:369). S == K gives
    plain top-k on the same kernels."""
    torch = _torch()
    cfg = _rr.RerouteConfig(retain_count, threshold)
    x, ids, weights = _check_layer_inputs(bank, x, ids, weights)
    T, K = int(ids.shape[0]), int(ids.shape[1])
    if cfg.retain_count > K:
        raise ConfigError(f"retain_count must not exceed K (got S={cfg.retain_count}, K={K})")
    dsim = _rr.as_device_sim(sim, bank.device)
    if dsim.m != bank.M:
        raise DimensionError(f"similarity matrix has shape {(dsim.m, dsim.m)}, expected {(bank.M, bank.M)}")
    dev = bank.device
    if out is None:
        rr = _rr.DeviceReroute(
            new_indices=torch.empty((T, K), dtype=torch.int32, device=dev),
            expert_class=torch.empty(bank.M, dtype=torch.uint8, device=dev),
            reroute_map=torch.empty(bank.M, dtype=torch.int32, device=dev),
            active_list=torch.empty(bank.M, dtype=torch.int32, device=dev),
            n_active=torch.empty(1, dtype=torch.int32, device=dev),
            status=torch.zeros(1, dtype=torch.int32, device=dev),
        )
        out = LayerOutput(torch.empty((T, bank.d_h), dtype=torch.float32, device=dev),
                          torch.empty((T, bank.d_h), dtype=torch.bfloat16, device=dev) if want_bf16 else None,
                          rr.status, rr)
    rr = out.reroute
    flags = 0 if dsim.validated else _rr.FLAG_CHECK_SIM
    ws = workspace(T, K, bank.M, bank.n_shared, bank.d_h, bank.d_m, dev) if ws is None else ws
    _lib.call("sere_moe_forward", bank.data.data_ptr(), bank.M, bank.n_shared, bank.d_h, bank.d_m,
              activation_code(activation), dsim.values.data_ptr(), cfg.retain_count, cfg.threshold, flags,
              x.data_ptr(), ids.data_ptr(), weights.data_ptr(), T, K, rr.new_indices.data_ptr(),
              rr.expert_class.data_ptr(), rr.reroute_map.data_ptr(), rr.active_list.data_ptr(),
              rr.n_active.data_ptr(), out.y.data_ptr(),
              out.y_bf16.data_ptr() if out.y_bf16 is not None else None, ws.data_ptr(), ws.numel(),
              out.status.data_ptr(), _stream_ptr(stream))
    dsim.validated = True
    return out


def moe_block_forward_device(bank: ExpertBank, sim, retain_count: int, threshold: float, h, ids, weights,
                             x_residual, h_next, eps: float = 1e-6, activation: str = "silu", stream=None,
                             out: LayerOutput | None = None, want_y: bool = False, ws=None) -> LayerOutput:
    """Decode block (`sere_moe_block_forward`): x_residual += SERE-MoE(h) and
    h_next = bf16(RMSNorm(x_residual)) in the combine pass. h_next may alias h."""
    import ctypes

    torch = _torch()
    cfg = _rr.RerouteConfig(retain_count, threshold)
    T, K = int(ids.shape[0]), int(ids.shape[1])
    dsim = _rr.as_device_sim(sim, bank.device)
    dev = bank.device
    if out is None:
        rr = _rr.DeviceReroute(
            new_indices=torch.empty((T, K), dtype=torch.int32, device=dev),
            expert_class=torch.empty(bank.M, dtype=torch.uint8, device=dev),
            reroute_map=torch.empty(bank.M, dtype=torch.int32, device=dev),
            active_list=torch.empty(bank.M, dtype=torch.int32, device=dev),
            n_active=torch.empty(1, dtype=torch.int32, device=dev),
            status=torch.zeros(1, dtype=torch.int32, device=dev),
        )
        y = torch.empty((T, bank.d_h), dtype=torch.float32, device=dev) if want_y else None
        out = LayerOutput(y, None, rr.status, rr)
    rr = out.reroute
    flags = 0 if dsim.validated else _rr.FLAG_CHECK_SIM
    ws = workspace(T, K, bank.M, bank.n_shared, bank.d_h, bank.d_m, dev) if ws is None else ws
    _lib.call("sere_moe_block_forward", bank.data.data_ptr(), bank.M, bank.n_shared, bank.d_h, bank.d_m,
              activation_code(activation), dsim.values.data_ptr(), cfg.retain_count, cfg.threshold, flags,
              h.data_ptr(), ids.data_ptr(), weights.data_ptr(), T, K, rr.new_indices.data_ptr(),
              rr.expert_class.data_ptr(), rr.reroute_map.data_ptr(), rr.active_list.data_ptr(),
              rr.n_active.data_ptr(), x_residual.data_ptr(), h_next.data_ptr(), ctypes.c_float(eps),
              out.y.data_ptr() if out.y is not None else None, ws.data_ptr(), ws.numel(), out.status.data_ptr(),
              _stream_ptr(stream))
    dsim.validated = True
    return out


def moe_forward_ep_device(bank: ExpertBank, n_experts: int, expert_lo: int, sim, retain_count: int,
                          threshold: float, x, ids, weights, activation: str = "silu", stream=None,
                          out: LayerOutput | None = None, ws=None) -> LayerOutput:
    """Expert-parallel shard of `moe_forward_device` (`sere_moe_forward_ep`): re-route the
    full gathered [T,K] table against `sim` (global ids, M = n_experts), then evaluate only
    this bank's experts (global [expert_lo, expert_lo + bank.M) + its shared experts).
    out.y = this rank's partial layer output; the ranks' partials sum to moe.layer_forward."""
    torch = _torch()
    cfg = _rr.RerouteConfig(retain_count, threshold)
    x = x.to(torch.bfloat16).contiguous()
    ids = ids.to(torch.int32).contiguous()
    weights = weights.to(torch.float32).contiguous()
    T, K = int(ids.shape[0]), int(ids.shape[1])
    if x.shape != (T, bank.d_h) or weights.shape != ids.shape:
        raise DimensionError("x / ids / weights shapes disagree")
    if cfg.retain_count > K:
        raise ConfigError(f"retain_count must not exceed K (got S={cfg.retain_count}, K={K})")
    dsim = _rr.as_device_sim(sim, bank.device)
    if dsim.m != n_experts:
        raise DimensionError(f"similarity matrix is {dsim.m}x{dsim.m}, expected {n_experts}")
    dev = bank.device
    if out is None:
        rr = _rr.DeviceReroute(
            new_indices=torch.empty((T, K), dtype=torch.int32, device=dev),
            expert_class=torch.empty(n_experts, dtype=torch.uint8, device=dev),
            reroute_map=torch.empty(n_experts, dtype=torch.int32, device=dev),
            active_list=torch.empty(n_experts, dtype=torch.int32, device=dev),
            n_active=torch.empty(1, dtype=torch.int32, device=dev),
            status=torch.zeros(1, dtype=torch.int32, device=dev),
        )
        out = LayerOutput(torch.empty((T, bank.d_h), dtype=torch.float32, device=dev), None, rr.status, rr)
    rr = out.reroute
    flags = 0 if dsim.validated else _rr.FLAG_CHECK_SIM
    ws = workspace(T, K, bank.M, bank.n_shared, bank.d_h, bank.d_m, dev) if ws is None else ws
    _lib.call("sere_moe_forward_ep", bank.data.data_ptr(), int(n_experts), int(expert_lo),
              int(expert_lo) + bank.M, bank.n_shared, bank.d_h, bank.d_m, activation_code(activation),
              dsim.values.data_ptr(), cfg.retain_count, cfg.threshold, flags, x.data_ptr(), ids.data_ptr(),
              weights.data_ptr(), T, K, rr.new_indices.data_ptr(), rr.expert_class.data_ptr(),
              rr.reroute_map.data_ptr(), rr.active_list.data_ptr(), rr.n_active.data_ptr(), out.y.data_ptr(),
              ws.data_ptr(), ws.numel(), out.status.data_ptr(), _stream_ptr(stream))
    dsim.validated = True
    return out


_ROUTE_WS: dict = {}


def router_weight_t(w_router):
    """RouterWeights.w_router [d_h, M] -> the kernel's expert-major bf16 [M, d_h] (done once per layer)."""
    torch = _torch()
    return w_router.to(torch.bfloat16).t().contiguous()


def route_workspace(T: int, d_h: int, M: int, device) -> Any:
    """A caller-owned router workspace (zero-initialised: its tickets start at zero)."""
    torch = _torch()
    return torch.zeros(max(int(_lib.load().sere_route_workspace_bytes(T, d_h, M)), 1), dtype=torch.uint8,
                       device=device)


def route_topk_device(w_router_t, x, top_k: int, stream=None, logits: bool = False, bias=None, out=None, ws=None):
    """moe.py:268-277 on CUDA: w_router_t bf16 [M, d_h] (see `router_weight_t`), x bf16 [T,d_h]
    -> (ids int32 [T,K], weights f32 [T,K][, logits f32 [T,M]]).
    `bias` (f32 [M], optional) is the benchmark's popularity-skew knob added to the logits."""
    torch = _torch()
    x = x.to(torch.bfloat16).contiguous()
    w = w_router_t.to(torch.bfloat16).contiguous()
    T, d_h = int(x.shape[0]), int(x.shape[1])
    if w.shape[1] != d_h:
        raise DimensionError(f"input width {d_h} does not match router d_h {w.shape[1]}")
    M = int(w.shape[0])
    if not 1 <= top_k <= M:
        raise ConfigError(f"top_k must satisfy 1 <= K <= M (got K={top_k}, M={M})")
    if out is not None:
        ids, wts = out
    else:
        ids = torch.empty((T, top_k), dtype=torch.int32, device=x.device)
        wts = torch.empty((T, top_k), dtype=torch.float32, device=x.device)
    lg = torch.empty((T, M), dtype=torch.float32, device=x.device) if logits else None
    b = bias.to(torch.float32).contiguous() if bias is not None else None
    if ws is None:
        nbytes = _lib.load().sere_route_workspace_bytes(T, d_h, M)
        key = str(x.device)
        ws = _ROUTE_WS.get(key)
        if ws is None or ws.numel() < nbytes:
            if ws is not None:
                _WS_RETIRED.append(ws)
            ws = route_workspace(T, d_h, M, x.device)
            _ROUTE_WS[key] = ws
    _lib.call("sere_route_topk", x.data_ptr(), w.data_ptr(), b.data_ptr() if b is not None else None,
              T, d_h, M, int(top_k), ids.data_ptr(), wts.data_ptr(), lg.data_ptr() if lg is not None else None,
              ws.data_ptr(), ws.numel(), _stream_ptr(stream))
    return (ids, wts, lg) if logits else (ids, wts)


# ---------------------------------------------------------------------------
# reference-shaped drop-ins (host arrays in/out)
# ---------------------------------------------------------------------------

MAX_CELLS = 16384   # T*K of one layer call (the align kernel's u16 counters and smem ids; capi.cu kMaxCells)
MAX_EXPERTS = 256   # routed experts per layer (capi.cu kMaxExperts)
MAX_SHARED = 31     # shared experts per layer (capi.cu kMaxShared)


def device_supports(n_tokens: int, top_k: int, n_experts: int, n_shared: int = 0) -> bool:
    """Whether one layer call of this shape fits the device path's limits (the reference
    itself has none; `integration.install` falls back to the reference function beyond them)."""
    return (n_tokens * top_k <= MAX_CELLS and 1 <= n_experts <= MAX_EXPERTS and 0 <= n_shared <= MAX_SHARED
            and 1 <= top_k <= n_experts)


def _fingerprint(a: Any) -> tuple:
    """Content key of one weight array: shape, dtype, wrapping uint64 sum and xor of its
    words. Any single changed element changes the sum; read once at memory bandwidth,
    which is the same traffic the reference's own expert_forward spends on the array."""
    a = np.ascontiguousarray(np.asarray(a))
    b = a.reshape(-1).view(np.uint8)
    n8 = b.size // 8 * 8
    w = b[:n8].view(np.uint64)
    tail = bytes(b[n8:])
    return (a.shape, a.dtype.str, int(w.sum(dtype=np.uint64)), int(np.bitwise_xor.reduce(w)) if w.size else 0, tail)


def _expert_fingerprint(e: Any) -> tuple:
    return (_fingerprint(e.w_gate), _fingerprint(e.w_up), _fingerprint(e.w_down))


_BANKS: dict[int, tuple[Any, ExpertBank, list]] = {}


def bank_for(layer: Any, experts_used=None) -> ExpertBank:
    """ExpertBank of a reference MoELayer, packed once and kept in sync with the layer's
    CONTENT: every call fingerprints the experts it is about to use (`experts_used` = bank
    slots, default all) and re-packs any whose weights changed in place since they were
    packed. The reference reads the current arrays on every call (moe.py:243-245), so an
    edited weight must never be served from a stale device copy."""
    if isinstance(layer, ExpertBank):
        return layer
    if isinstance(getattr(layer, "bank", None), ExpertBank):  # io.GpuLayer
        return layer.bank
    experts = list(layer.experts) + list(getattr(layer, "shared_experts", ()))
    hit = _BANKS.get(id(layer))
    if hit is None or hit[0] is not layer:
        bank = ExpertBank.from_reference_layer(layer)
        if len(_BANKS) > 64:
            _BANKS.clear()
        _BANKS[id(layer)] = (layer, bank, [_expert_fingerprint(e) for e in experts])
        return bank
    _, bank, fps = hit
    torch = _torch()
    for j in (range(len(experts)) if experts_used is None else experts_used):
        fp = _expert_fingerprint(experts[j])
        if fp != fps[j]:
            e = experts[j]
            t = [torch.from_numpy(np.asarray(getattr(e, n), dtype=np.float32)[None]).to(bank.device, torch.bfloat16)
                 for n in ("w_gate", "w_up", "w_down")]
            bank.pack(*t, first=j)
            fps[j] = fp
    return bank


def invalidate(layer: Any | None = None) -> None:
    """Forget the packed copy of `layer` (or of every layer)."""
    if layer is None:
        _BANKS.clear()
    else:
        _BANKS.pop(id(layer), None)


def layer_forward(layer: Any, x: Any, assignment: Any, activation: str = "silu") -> np.ndarray:
    """Drop-in for moe.layer_forward (moe.py:280-310): weighted sum of routed experts in
    slot order plus every shared expert, on the GPU. Returns float64 [T,d_h] (the fp32
    device result widened)."""
    torch = _torch()
    activation_code(activation)
    idx = np.asarray(assignment.indices)
    n_routed = len(layer.experts) if not isinstance(layer, ExpertBank) and hasattr(layer, "experts") else None
    used = None
    if n_routed is not None and idx.size and idx.min() >= 0 and idx.max() < n_routed:
        n_sh = len(getattr(layer, "shared_experts", ()))
        used = sorted(set(np.unique(idx).tolist()) | set(range(n_routed, n_routed + n_sh)))
    bank = bank_for(layer, used)
    xa = np.asarray(x, dtype=np.float64)
    if xa.ndim != 2:
        raise DimensionError(f"x must be 2-D, got shape {xa.shape}")
    w = np.asarray(assignment.weights, dtype=np.float64)
    if idx.shape[0] != xa.shape[0]:
        raise DimensionError(f"assignment covers {idx.shape[0]} tokens, batch has {xa.shape[0]}")
    if xa.shape[1] != bank.d_h:
        raise DimensionError(f"input width {xa.shape[1]} does not match expert d_h {bank.d_h}")
    if idx.size and (idx.min() < 0 or idx.max() >= bank.M):
        raise RoutingError(f"assignment refers to experts outside [0, {bank.M})")
    dev = bank.device
    out = layer_forward_device(bank, torch.from_numpy(xa).to(dev), torch.from_numpy(idx.astype(np.int32)).to(dev),
                               torch.from_numpy(w.astype(np.float32)).to(dev), activation)
    out.check()
    return out.y.double().cpu().numpy()


@dataclass
class LayerTrace:
    """moe.py:313-320."""

    original: Any
    final: Any
    reroute: Any
    active: frozenset


@dataclass
class ForwardResult:
    """moe.py:323-326."""

    output: np.ndarray
    layers: list = field(default_factory=list)


@dataclass
class Assignment:
    """Host twin of RoutingAssignment (moe.py:193-232) used in traces."""

    indices: np.ndarray
    weights: np.ndarray

    @property
    def n_tokens(self) -> int:
        return self.indices.shape[0]

    @property
    def top_k(self) -> int:
        return self.indices.shape[1]


def route_topk(router: Any, x: Any) -> Assignment:
    """moe.py:268-277 on the GPU for a reference RouterWeights (bf16 weights, fp32 logits)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    xa = np.asarray(x, dtype=np.float64)
    if xa.ndim != 2:
        raise DimensionError(f"x must be 2-D, got shape {xa.shape}")
    if xa.shape[1] != np.shape(router.w_router)[0]:
        raise DimensionError(f"input width {xa.shape[1]} does not match router d_h {np.shape(router.w_router)[0]}")
    if not np.all(np.isfinite(xa)):  # moe.py:274-275
        raise DomainError("router input contains non-finite values")
    w = torch.as_tensor(np.asarray(router.w_router, dtype=np.float32)).to(dev)
    xt = torch.as_tensor(xa.astype(np.float32)).to(dev)
    ids, wts = route_topk_device(router_weight_t(w), xt, int(router.top_k))
    return Assignment(ids.cpu().numpy().astype(np.int64), wts.double().cpu().numpy())


def model_forward(model: Any, batch: Any, config: Any = None, sims: Sequence | None = None,
                  router_override: Callable | None = None) -> ForwardResult:
    """moe.py:329-377 with every layer on the GPU: route -> (phase-gated) fused
    re-route + layer. Routing uses the GPU router unless `router_override` is given."""
    torch = _torch()
    x_np = np.asarray(batch.x, dtype=np.float64)
    if x_np.shape[1] != model.d_h:
        raise DimensionError(f"batch width {x_np.shape[1]} does not match model d_h {model.d_h}")
    if config is not None:
        if sims is None or len(sims) != model.n_layers:
            raise DimensionError(f"rewriting needs one similarity matrix per layer ({model.n_layers})")
        for l, sim in enumerate(sims):
            m = model.layers[l].n_experts
            if np.shape(getattr(sim, "values", sim)) != (m, m):
                raise DimensionError(f"similarity matrix for layer {l} has wrong shape, expected {(m, m)}")
    apply_rewrite = config is not None and (config.phase_mode == "all_phases" or batch.phase == "decode")
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.from_numpy(x_np).to(dev)
    traces = []
    for l, layer in enumerate(model.layers):
        bank = bank_for(layer)
        if router_override is not None:
            a = router_override(l, x.double().cpu().numpy())
            ids = torch.as_tensor(np.asarray(a.indices).astype(np.int32)).to(dev)
            wts = torch.as_tensor(np.asarray(a.weights, dtype=np.float32)).to(dev)
            original = a
        else:
            wr = layer.router.w_router
            if not isinstance(wr, torch.Tensor):
                wr = torch.as_tensor(np.asarray(wr, dtype=np.float32))
            ids, wts = route_topk_device(router_weight_t(wr.to(dev)), x, int(layer.router.top_k))
            original = Assignment(ids.cpu().numpy().astype(np.int64), wts.double().cpu().numpy())
        if apply_rewrite:
            dsim = _rr.DeviceSimilarity(sims[l], dev)  # current values, validated on this call (rerouting.py:140)
            out = moe_forward_device(bank, dsim, config.retain_count, config.threshold, x, ids, wts,
                                     model.activation)
            out.check()
            res = out.reroute.to_result()
            final = Assignment(res.new_indices, np.asarray(original.weights, dtype=np.float64))
            active = res.final_active
        else:
            out = layer_forward_device(bank, x, ids, wts, model.activation)
            out.check()
            res = None
            final = original
            active = frozenset(np.unique(np.asarray(original.indices)).tolist())
        x = out.y
        traces.append(LayerTrace(original=original, final=final, reroute=res, active=active))
    return ForwardResult(output=x.double().cpu().numpy(), layers=traces)
