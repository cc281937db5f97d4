"""Multi-layer batched-decode step on the GPU (the C4 benchmark workload).

A decode step pushes T tokens (one per sequence) through L MoE layers. Each layer is
the reference's per-layer body (moe.model_forward, moe.py:362-375):

    ids, w = route_topk(layer.router, h)          (router kernel, fp32 logits)
    if SERE: ids = apply_sere(ids, sim_l, S, rho)  (fused into the layer launch)
    y = layer_forward(layer, h, ids, w)            (grouped tcgen05 FFN)

wrapped, for the benchmark, in the pre-norm residual block of a Qwen3 decoder layer
minus attention: h = RMSNorm(x); x = x + MoE(h). The reference chains raw outputs
(x <- MoE(x)); with N(0, 1/d_h) random weights that chain decays doubly
exponentially (sigma_{l+1} ~ 0.1 sigma_l^2) and by layer ~6 every token routes to the
same experts, which would make any SERE-vs-top-k number meaningless. The residual
stream keeps routing token-dependent at every depth. `block="plain"` runs the
reference chain instead (used by the parity tests).

The whole step is captured once into a CUDA graph (7 launches per layer, no host
sync, all data-dependent sizes stay on the device).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Any

import numpy as np

from . import _lib
from . import moe as _moe
from . import rerouting as _rr


def _torch():
    import torch

    return torch


def clustered_sim(rng: np.random.Generator, m: int, n_clusters: int = 8) -> np.ndarray:
    """Symmetric similarity with cluster structure: intra U[0.6,1], inter U[0,0.4], unit diagonal."""
    labels = rng.integers(0, n_clusters, size=m)
    r = rng.random((m, m))
    same = labels[:, None] == labels[None, :]
    v = np.where(same, 0.6 + 0.4 * r, 0.4 * r)
    v = (v + v.T) / 2.0
    np.fill_diagonal(v, 1.0)
    return v


def uniform_sim(rng: np.random.Generator, m: int) -> np.ndarray:
    """The reference tests' construction (tests/test_rerouting.py:23-29)."""
    r = rng.random((m, m))
    v = (r + r.T) / 2.0
    np.fill_diagonal(v, 1.0)
    return v


@dataclass
class DecodeLayer:
    bank: Any            # moe.ExpertBank
    w_router: Any        # bf16 [d_h, M] (reference orientation)
    bias: Any            # f32 [M] popularity skew (beta * N(0,1)); zeros for beta = 0
    sim: Any             # rerouting.DeviceSimilarity (fp64 [M,M])
    w_router_t: Any = None  # bf16 [M, d_h] kernel orientation


class DecodeModel:
    """L MoE layers with random-init weights of one architecture, resident in HBM."""

    def __init__(self, n_layers: int, M: int, K: int, d_h: int, d_m: int, n_shared: int = 0, seed: int = 0,
                 beta: float = 1.0, sim_kind: str = "uniform", device=None, keep_raw_layer: int | None = None,
                 expert_ids=None, shared_ids=None):
        """`expert_ids` / `shared_ids`: the experts this process holds (expert parallelism);
        default all. Routers, biases and sims are replicated and identical on every shard."""
        torch = _torch()
        self.L, self.M, self.K, self.d_h, self.d_m, self.n_shared = n_layers, M, K, d_h, d_m, n_shared
        self.beta, self.sim_kind, self.seed = float(beta), sim_kind, seed
        self.expert_ids = list(range(M)) if expert_ids is None else list(expert_ids)
        self.shared_ids = list(range(n_shared)) if shared_ids is None else list(shared_ids)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.layers: list[DecodeLayer] = []
        self.sims_host: list[np.ndarray] = []
        g = torch.Generator(device=self.device)
        for l in range(n_layers):
            bank = _moe.ExpertBank.random(M, n_shared, d_h, d_m, seed=seed * 100003 + l, device=self.device,
                                          keep_raw=(keep_raw_layer == l), expert_ids=self.expert_ids,
                                          shared_ids=self.shared_ids)
            g.manual_seed(seed * 100003 + 50000 + l)
            wr = (torch.randn((d_h, M), generator=g, device=self.device) / float(np.sqrt(d_h))).to(torch.bfloat16)
            bias = (self.beta * torch.randn(M, generator=g, device=self.device)).float()
            rng = np.random.default_rng([seed, l, 3])
            sim = clustered_sim(rng, M) if sim_kind == "clustered" else uniform_sim(rng, M)
            self.sims_host.append(sim)
            self.layers.append(DecodeLayer(bank, wr, bias, _rr.DeviceSimilarity(sim, self.device),
                                           _moe.router_weight_t(wr)))

    @property
    def weight_bytes_per_expert(self) -> int:
        return 2 * 3 * self.d_h * self.d_m


class StageEvents:
    """Per-layer CUDA events around the 5 stages of the layer launch (sere_set_stage_events)."""

    stage_events = None

    def enable_stage_events(self) -> None:
        """Record 6 timing events around the 5 stages of every layer (must precede capture)."""
        torch = _torch()
        self.stage_events = []
        for _ in range(self.model.L):
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            for e in evs:
                e.record()  # materialise the CUDA event handle
            self.stage_events.append(evs)
        torch.cuda.synchronize()

    def _events_on(self, l: int) -> None:
        if self.stage_events is not None:
            arr = (ctypes.c_void_p * 6)(*[e.cuda_event for e in self.stage_events[l]])
            _lib.load().sere_set_stage_events(arr, 6)

    def _events_off(self) -> None:
        if self.stage_events is not None:
            _lib.load().sere_set_stage_events(None, 0)

    def stage_times_ms(self) -> np.ndarray:
        """[L, 5] durations (ms) of align(+reroute), permute, gate/up GEMM, down GEMM, combine."""
        out = np.zeros((self.model.L, 5))
        for l, evs in enumerate(self.stage_events):
            for i in range(5):
                out[l, i] = evs[i].elapsed_time(evs[i + 1])
        return out


class DecodeStep(StageEvents):
    """Preallocated buffers + (optionally) a CUDA graph for one decode step.

    mode "sere": re-route every layer with (retain_count, threshold);
    mode "topk": the same kernels with S = K (identity re-routing, plain top-k)."""

    def __init__(self, model: DecodeModel, T: int, retain_count: int = 1, threshold: float = 0.5,
                 mode: str = "sere", block: str = "prenorm_residual", eps: float = 1e-6):
        torch = _torch()
        if mode not in ("sere", "topk"):
            raise ValueError(mode)
        self.model, self.T, self.mode, self.block, self.eps = model, T, mode, block, eps
        self.S = retain_count if mode == "sere" else model.K
        self.rho = threshold
        dev = model.device
        self.x_in = torch.zeros((T, model.d_h), dtype=torch.float32, device=dev)    # step input (embeddings)
        self.x = torch.zeros((T, model.d_h), dtype=torch.float32, device=dev)       # residual stream / output
        self.h = torch.zeros((T, model.d_h), dtype=torch.bfloat16, device=dev)      # layer input
        self.ids = torch.zeros((T, model.K), dtype=torch.int32, device=dev)
        self.w = torch.zeros((T, model.K), dtype=torch.float32, device=dev)
        self.outs = []
        for _ in range(model.L):
            rr = _rr.DeviceReroute(
                new_indices=torch.zeros((T, model.K), dtype=torch.int32, device=dev),
                expert_class=torch.zeros(model.M, dtype=torch.uint8, device=dev),
                reroute_map=torch.zeros(model.M, dtype=torch.int32, device=dev),
                active_list=torch.zeros(model.M, dtype=torch.int32, device=dev),
                n_active=torch.zeros(1, dtype=torch.int32, device=dev),
                status=torch.zeros(1, dtype=torch.int32, device=dev),
            )
            y = torch.zeros((T, model.d_h), dtype=torch.float32, device=dev) if block == "plain" else None
            self.outs.append(_moe.LayerOutput(y, None, rr.status, rr))
        self.graph = None
        self.stage_events = None
        self._trace_hook = None  # debug_ffn: called with the layer index before each layer launch
        # this step's own workspaces: its CUDA graph bakes in their addresses, so they live
        # (and are used) exactly as long as the step
        self.ws = _moe.new_workspace(T, model.K, len(model.expert_ids), len(model.shared_ids), model.d_h,
                                     model.d_m, dev)
        self.route_ws = _moe.route_workspace(T, model.d_h, model.M, dev)

    # ---------------------------------------------------------------- launches
    def _norm(self, y) -> None:
        _lib.call("sere_residual_rmsnorm", self.x.data_ptr(), y.data_ptr() if y is not None else None,
                  self.h.data_ptr(), self.T, self.model.d_h, ctypes.c_float(self.eps), _moe._stream_ptr())

    def _launch(self) -> None:
        m = self.model
        plain = self.block == "plain"
        self.x.copy_(self.x_in)
        if not plain:
            self._norm(None)
        for l, layer in enumerate(m.layers):
            if plain:
                # reference chain x <- MoE(x): the layer input is bf16(x)
                if l == 0:
                    self.h.copy_(self.x)
                else:
                    self.h.copy_(self.outs[l - 1].y)
            _moe.route_topk_device(layer.w_router_t, self.h, m.K, bias=layer.bias, out=(self.ids, self.w),
                                   ws=self.route_ws)
            if self._trace_hook is not None:
                self._trace_hook(l)
            self._events_on(l)
            if plain:
                _moe.moe_forward_device(layer.bank, layer.sim, self.S, self.rho, self.h, self.ids, self.w,
                                        out=self.outs[l], ws=self.ws)
            else:  # x += MoE(h); h = RMSNorm(x) fused into the combine pass
                _moe.moe_block_forward_device(layer.bank, layer.sim, self.S, self.rho, self.h, self.ids, self.w,
                                              self.x, self.h, self.eps, out=self.outs[l], ws=self.ws)
            self._events_off()
        if plain:
            self.x.copy_(self.outs[-1].y)

    @property
    def launches_per_step(self) -> int:
        """Kernels of this library per step: router + 4 layer kernels (re-route/align, permute,
        fused FFN, combine) per layer (+ the first RMSNorm)."""
        return self.model.L * 5 + (0 if self.block == "plain" else 1)

    def run(self) -> None:
        """One step on the current stream (graph replay if captured)."""
        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch()

    def capture(self) -> None:
        """Warm up eagerly once, then capture the step into a CUDA graph."""
        torch = _torch()
        self._launch()
        torch.cuda.synchronize()
        self.check()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launch()
        self.graph = g

    # ---------------------------------------------------------------- results
    def check(self) -> None:
        for o in self.outs:
            o.check()

    def active_counts(self) -> np.ndarray:
        """|final_active| per layer of the last step (routed experts streamed)."""
        torch = _torch()
        return torch.cat([o.reroute.n_active for o in self.outs]).cpu().numpy()

    def set_input(self, x) -> None:
        self.x_in.copy_(x)

    @property
    def workspace(self) -> tuple[int, int]:
        """(device pointer, bytes) of this step's layer workspace (kernel-only FFN replay)."""
        return self.ws.data_ptr(), self.ws.numel()

    def run_host(self, x_host, out_host) -> None:
        """Public end-to-end call: host (pinned) input -> step -> host output, stream-ordered."""
        self.x_in.copy_(x_host, non_blocking=True)
        self.run()
        out_host.copy_(self.x, non_blocking=True)
