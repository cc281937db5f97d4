"""Expert parallelism (EP) for the multi-layer decode step.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch). Rank r of N
owns a contiguous block of routed experts (`expert_range`) and the shared experts
s with s % N == r; routers and similarity matrices are replicated; the decode
batch is split into N equal token slices. Per layer:

  1. h_r = RMSNorm(x_r); (ids_r, w_r) = router(h_r)                   (local)
  2. all-gather of the packed rows [h | ids | w] -> the full batch     (NCCL)
  3. re-routing on the FULL [T,K] table -- every rank computes the same
     bit-exact ids the 1-GPU run computes, so no separate primary-mask
     exchange is needed (the batch-global union of rerouting.py:147 is local)
  4. grouped FFN over this rank's experts only -> partial y [T, d_h] (f32)
  5. reduce-scatter(sum) of the partials -> y_r; x_r += y_r           (NCCL)

Why all-gather rather than all-to-all: with K = 8 routed experts per token spread
over N <= 8 ranks, almost every token is needed by almost every rank, so the
dispatch volume of an all-to-all is within a few percent of an all-gather while
the all-gather needs no host-visible split sizes (no sync, CUDA-graph capturable).

`Exchange` is backend-agnostic: NCCL on the GPU path, gloo (CPU tensors) in the
world-size-2 tests, which drive the same choreography with the CPU oracle as the
per-rank compute.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Any

import numpy as np

from . import _lib
from . import moe as _moe
from . import rerouting as _rr
from .decode import StageEvents


def _torch():
    import torch

    return torch


def expert_range(M: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous routed-expert block [lo, hi) of `rank` (sizes differ by at most one)."""
    base, rem = divmod(M, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def shared_owned(n_shared: int, world: int, rank: int) -> list[int]:
    return [s for s in range(n_shared) if s % world == rank]


def token_slice(T: int, world: int, rank: int) -> tuple[int, int]:
    if T % world:
        raise ValueError(f"decode batch {T} must split evenly over {world} ranks")
    n = T // world
    return rank * n, (rank + 1) * n


class Exchange:
    """The two collectives of an EP layer over preallocated buffers.

    Rows are packed as bytes [h (2*d_h) | ids (4*K) | w (4*K)] so one all-gather moves
    everything; partial outputs are f32 and reduce-scattered with SUM."""

    def __init__(self, T_local: int, d_h: int, K: int, device, group=None, h_dtype=None, y_dtype=None):
        torch = _torch()
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)
        self.T_local, self.d_h, self.K = T_local, d_h, K
        self.h_dtype = h_dtype or torch.bfloat16
        hb = torch.tensor([], dtype=self.h_dtype).element_size() * d_h
        self.h_bytes = hb
        self.row_bytes = (hb + 8 * K + 15) // 16 * 16
        self.send = torch.zeros((T_local, self.row_bytes), dtype=torch.uint8, device=device)
        self.recv = torch.zeros((self.world * T_local, self.row_bytes), dtype=torch.uint8, device=device)
        T = self.world * T_local
        self.h_all = torch.zeros((T, d_h), dtype=self.h_dtype, device=device)
        self.ids_all = torch.zeros((T, K), dtype=torch.int32, device=device)
        self.w_all = torch.zeros((T, K), dtype=torch.float32, device=device)
        self.y_local = torch.zeros((T_local, d_h), dtype=y_dtype or torch.float32, device=device)

    def _views(self, buf):
        hb, K = self.h_bytes, self.K
        h = buf[:, :hb].view(self.h_dtype)
        ids = buf[:, hb:hb + 4 * K].view(_torch().int32)
        w = buf[:, hb + 4 * K:hb + 8 * K].view(_torch().float32)
        return h, ids, w

    def gather(self, h_local, ids_local, w_local):
        """All-gather the local rows; returns contiguous (h_all, ids_all, w_all) in rank order."""
        h, i, w = self._views(self.send)
        h.copy_(h_local)
        i.copy_(ids_local)
        w.copy_(w_local)
        if hasattr(self.dist, "all_gather_into_tensor") and self.backend == "nccl":
            self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        else:
            parts = list(self.recv.chunk(self.world, dim=0))
            self.dist.all_gather(parts, self.send, group=self.group)
            if parts[0].data_ptr() != self.recv.data_ptr():
                self.recv.copy_(_torch().cat(parts, 0))
        h, i, w = self._views(self.recv)
        self.h_all.copy_(h)
        self.ids_all.copy_(i)
        self.w_all.copy_(w)
        return self.h_all, self.ids_all, self.w_all

    def reduce_scatter(self, y_partial):
        """Sum the ranks' partial outputs and keep this rank's token slice."""
        if self.backend == "nccl":
            self.dist.reduce_scatter_tensor(self.y_local, y_partial, op=self.dist.ReduceOp.SUM, group=self.group)
        else:  # gloo has no reduce-scatter: all-reduce then slice (CPU tests only)
            buf = y_partial.clone()
            self.dist.all_reduce(buf, op=self.dist.ReduceOp.SUM, group=self.group)
            lo = self.rank * self.T_local
            self.y_local.copy_(buf[lo:lo + self.T_local])
        return self.y_local


class EPDecodeStep(StageEvents):
    """Expert-parallel decode step of a sharded `decode.DecodeModel` (one rank's view)."""

    def __init__(self, model, T: int, retain_count: int = 1, threshold: float = 0.5, mode: str = "sere",
                 group=None, eps: float = 1e-6):
        torch = _torch()
        import torch.distributed as dist

        self.model, self.T, self.mode, self.eps = model, T, mode, eps
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.lo, self.hi = expert_range(model.M, self.world, self.rank)
        if model.expert_ids != list(range(self.lo, self.hi)):
            raise ValueError("model shard does not match this rank's expert range")
        self.t0, self.t1 = token_slice(T, self.world, self.rank)
        self.T_local = self.t1 - self.t0
        self.S = retain_count if mode == "sere" else model.K
        self.rho = threshold
        dev = model.device
        self.x_in = torch.zeros((self.T_local, model.d_h), dtype=torch.float32, device=dev)
        self.x = torch.zeros_like(self.x_in)
        self.h = torch.zeros((self.T_local, model.d_h), dtype=torch.bfloat16, device=dev)
        self.ids = torch.zeros((self.T_local, model.K), dtype=torch.int32, device=dev)
        self.w = torch.zeros((self.T_local, model.K), dtype=torch.float32, device=dev)
        self.xch = Exchange(self.T_local, model.d_h, model.K, dev, group)
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
            self.outs.append(_moe.LayerOutput(torch.zeros((T, model.d_h), dtype=torch.float32, device=dev), None,
                                              rr.status, rr))
        self.graph = None
        self.graphed = False
        self.ws = _moe.new_workspace(T, model.K, len(model.expert_ids), len(model.shared_ids), model.d_h,
                                     model.d_m, dev)
        self.route_ws = _moe.route_workspace(self.T_local, model.d_h, model.M, dev)

    @property
    def workspace(self) -> tuple[int, int]:
        return self.ws.data_ptr(), self.ws.numel()

    def _norm(self, y) -> None:
        _lib.call("sere_residual_rmsnorm", self.x.data_ptr(), y.data_ptr() if y is not None else None,
                  self.h.data_ptr(), self.T_local, self.model.d_h, ctypes.c_float(self.eps), _moe._stream_ptr())

    def _launch(self) -> None:
        m = self.model
        self.x.copy_(self.x_in)
        self._norm(None)
        for l, layer in enumerate(m.layers):
            _moe.route_topk_device(layer.w_router_t, self.h, m.K, bias=layer.bias, out=(self.ids, self.w),
                                   ws=self.route_ws)
            h_all, ids_all, w_all = self.xch.gather(self.h, self.ids, self.w)
            self._events_on(l)
            _moe.moe_forward_ep_device(layer.bank, m.M, self.lo, layer.sim, self.S, self.rho, h_all, ids_all,
                                       w_all, out=self.outs[l], ws=self.ws)
            self._events_off()
            y_local = self.xch.reduce_scatter(self.outs[l].y)
            self._norm(y_local)

    @property
    def launches_per_step(self) -> int:
        """Kernels of this library per step: router, re-route/align, permute, fused FFN, combine and
        residual RMSNorm per layer, plus the first RMSNorm (NCCL and torch copies not counted)."""
        return self.model.L * 6 + 1

    def run(self) -> None:
        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch()

    def capture(self) -> bool:
        """Warm up, then try to capture the step (NCCL collectives included) in a CUDA graph.
        Falls back to eager launches if capture is not supported; returns whether graphed."""
        torch = _torch()
        self._launch()
        torch.cuda.synchronize()
        self.check()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch()
            self.graph = g
            self.graphed = True
        except Exception:  # pragma: no cover - depends on the NCCL/torch build
            self.graph = None
            self.graphed = False
            torch.cuda.synchronize()
        return self.graphed

    def check(self) -> None:
        for o in self.outs:
            o.check()

    def active_counts(self) -> np.ndarray:
        torch = _torch()
        return torch.cat([o.reroute.n_active for o in self.outs]).cpu().numpy()

    def run_host(self, x_host, out_host) -> None:
        self.x_in.copy_(x_host, non_blocking=True)
        self.run()
        out_host.copy_(self.x, non_blocking=True)
