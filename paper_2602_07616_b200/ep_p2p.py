"""Expert parallelism over NVLink peer memory (include/sere_b200.h (4c)).

Same sharding as `ep.py` (rank r owns a contiguous block of routed experts and the
shared experts s % N == r; routers and sims replicated; the batch split into N token
slices), but the two collectives are gone: every rank owns a peer-reachable region

    h_all bf16 [T,d_h] | ids_all i32 [T,K] | w_all f32 [T,K] | flags i32 [N] | workspace

and the kernels read and write the other ranks' regions directly:

  1. router (this rank's tokens)        -> ids/w rows stored into EVERY rank's ids_all/w_all
  2. flag barrier                          (everybody's rows landed)
  3. re-route + align + permute + fused FFN over the whole batch, this rank's experts;
     the expert outputs (y_perm) stay in this rank's workspace
  4. flag barrier                          (everybody's y_perm is final)
  5. combine of this rank's tokens: each slot's row is loaded from its OWNER's y_perm in
     slot order (bit-exact with one GPU), x += y, and h = RMSNorm(x) is stored into
     EVERY rank's h_all -- the reduce-scatter and the next layer's all-gather.

`PeerRegion` allocates a region with `sere_alloc_peer` (its own cudaMalloc, so one CUDA
IPC handle covers it); `connect_ipc` exchanges handles over a torch.distributed group
(any backend) and maps the peers' regions; `connect_local` wires "virtual ranks" of one
process on one device (the tests' single-GPU form of the same kernels).
"""

from __future__ import annotations

import ctypes
from typing import Any

import numpy as np

from . import _lib
from . import moe as _moe
from . import rerouting as _rr
from .decode import StageEvents
from .ep import expert_range, shared_owned, token_slice


def _torch():
    import torch

    return torch


def _align(x: int, a: int) -> int:
    return (x + a - 1) // a * a


class _CudaArray:
    """`__cuda_array_interface__` view of raw device memory (torch.as_tensor wraps it)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _view(ptr: int, shape: tuple, typestr: str, device):
    torch = _torch()
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=device)


class PeerRegion:
    """One rank's peer-reachable buffers (a single `sere_alloc_peer` allocation)."""

    def __init__(self, T_all: int, d_h: int, K: int, world: int, ws_bytes: int, device):
        self.T_all, self.d_h, self.K, self.world, self.device = T_all, d_h, K, world, device
        off = 0
        self.off_h = off
        off = _align(off + T_all * d_h * 2, 1024)
        self.off_ids = off
        off = _align(off + T_all * K * 4, 1024)
        self.off_w = off
        off = _align(off + T_all * K * 4, 1024)
        self.off_flags = off
        off = _align(off + 4 * (_lib.MAX_EP_RANKS + 1), 1024)  # barrier slots + the sticky abort word
        self.off_ws = off
        self.ws_bytes = ws_bytes
        self.nbytes = off + ws_bytes + 2048
        p = ctypes.c_void_p()
        _lib.call("sere_alloc_peer", ctypes.c_size_t(self.nbytes), ctypes.byref(p))
        self.base = int(p.value)
        self.owned = True
        self._bind(self.base)
        self.flags.zero_()

    @classmethod
    def mapped(cls, like: "PeerRegion", base: int) -> "PeerRegion":
        """A peer's region opened in this process (same geometry as `like`)."""
        r = cls.__new__(cls)
        r.__dict__.update({k: v for k, v in like.__dict__.items() if k.startswith(("off_", "T_all", "d_h", "K",
                                                                                   "world", "device", "ws_bytes",
                                                                                   "nbytes"))})
        r.owned = False
        r.base = int(base)
        r._bind(r.base)
        return r

    def _bind(self, base: int) -> None:
        torch = _torch()
        T, d_h, K, dev = self.T_all, self.d_h, self.K, self.device
        self.h_all = _view(base + self.off_h, (T, d_h), "<i2", dev).view(torch.bfloat16)
        self.ids_all = _view(base + self.off_ids, (T, K), "<i4", dev)
        self.w_all = _view(base + self.off_w, (T, K), "<f4", dev)
        self.flags = _view(base + self.off_flags, (_lib.MAX_EP_RANKS + 1,), "<i4", dev)
        self.ws_ptr = _align(base + self.off_ws, 1024)  # the library aligns its workspace base to 1 KB too

    def ipc_handle(self) -> bytes:
        buf = (ctypes.c_char * 64)()
        _lib.call("sere_ipc_handle", ctypes.c_void_p(self.base), buf)
        return bytes(buf)

    def close(self) -> None:
        if self.base:
            _lib.call("sere_free_peer" if self.owned else "sere_ipc_close", ctypes.c_void_p(self.base))
            self.base = 0


class P2PDecodeStep(StageEvents):
    """One rank's expert-parallel decode step over peer memory (prenorm-residual block,
    the same layer chain as `decode.DecodeStep`, whose output it reproduces bit for bit)."""

    def __init__(self, model, T: int, world: int, rank: int, retain_count: int = 1, threshold: float = 0.5,
                 mode: str = "sere", eps: float = 1e-6, timeout_s: float = 5.0, fused_barriers: bool = True):
        torch = _torch()
        self.model, self.T, self.world, self.rank, self.mode, self.eps = model, T, world, rank, mode, eps
        if not 1 <= world <= _lib.MAX_EP_RANKS:
            raise ValueError(f"world size {world} outside [1, {_lib.MAX_EP_RANKS}]")
        self.lo, self.hi = expert_range(model.M, world, rank)
        if model.expert_ids != list(range(self.lo, self.hi)):
            raise ValueError("model shard does not match this rank's expert range")
        self.n_shared_total = model.n_shared  # shared experts of the layer (this shard holds model.shared_ids)
        self.sh = shared_owned(self.n_shared_total, world, rank)
        if list(model.shared_ids) != self.sh:
            raise ValueError("model shard does not hold this rank's shared experts")
        self.t0, self.t1 = token_slice(T, world, rank)
        self.T_local = self.t1 - self.t0
        self.S = retain_count if mode == "sere" else model.K
        self.rho = threshold
        self.timeout_ns = int(timeout_s * 1e9)
        dev = model.device
        m_local = self.hi - self.lo
        ws_bytes = _lib.load().sere_layer_workspace_bytes(T, model.K, m_local, len(self.sh), model.d_h, model.d_m)
        self.region = PeerRegion(T, model.d_h, model.K, world, ws_bytes, dev)
        self.x_in = torch.zeros((self.T_local, model.d_h), dtype=torch.float32, device=dev)
        self.x = torch.zeros_like(self.x_in)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=dev)
        self.bar_status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.arrivals = torch.zeros(1, dtype=torch.int32, device=dev)
        self.wait_ns = torch.zeros(2, dtype=torch.int64, device=dev)  # fused-barrier waits: align, combine
        # fused barriers: the router's last CTA and the FFN's last CTA arrive, the align kernel and
        # the combine wait (5 launches per layer); False: two sere_ep_barrier kernels (7 launches)
        self.fused = bool(fused_barriers)
        self.route_ws = torch.zeros(max(_lib.load().sere_route_workspace_bytes(self.T_local, model.d_h, model.M), 1),
                                    dtype=torch.uint8, device=dev)
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
            self.outs.append(_moe.LayerOutput(None, None, rr.status, rr))
        self.peers = None
        self.peer_regions: list = []
        self.graph = None
        # virtual ranks (one device): callbacks around the FFN launch, see connect_local
        self._ffn_pre = None
        self._ffn_post = None
        self._combine_pre = None
        self._router_post = None

    # ------------------------------------------------------------------ wiring
    def _layout(self, m_local: int, n_sh: int):
        m = self.model
        return _lib.workspace_layout(self.T, m.K, m_local, n_sh, m.d_h, m.d_m)

    def _build_peers(self, regions: list) -> None:
        m = self.model
        p = _lib.EpPeers()
        p.world, p.rank, p.t0, p.T_all = self.world, self.rank, self.t0, self.T
        for r in range(self.world):
            p.e_lo[r] = expert_range(m.M, self.world, r)[0]
        p.e_lo[self.world] = m.M
        for r, reg in enumerate(regions):
            lo, hi = expert_range(m.M, self.world, r)
            n_sh = len(shared_owned(self.n_shared_total, self.world, r))
            L = self._layout(hi - lo, n_sh)
            p.nsh[r] = n_sh
            p.r_max[r] = L.r_max
            p.y_perm[r] = reg.ws_ptr + L.off_y_perm
            p.slot_row[r] = reg.ws_ptr + L.off_slot_row
            p.h_all[r] = reg.h_all.data_ptr()
            p.ids_all[r] = reg.ids_all.data_ptr()
            p.w_all[r] = reg.w_all.data_ptr()
            p.flags[r] = reg.flags.data_ptr()
        if self.fused:
            p.epoch = self.epoch.data_ptr()
            p.status = self.bar_status.data_ptr()
            p.arrivals = self.arrivals.data_ptr()
            p.timeout_ns = self.timeout_ns
            p.wait_ns = self.wait_ns.data_ptr()
        self.peers = p
        self.peer_regions = regions

    @staticmethod
    def connect_local(steps: list) -> None:
        """Virtual ranks of one process on one device: every step sees the others' regions.
        Their FFN launches are serialised in rank order by events (two persistent FFN grids
        of the same device must not wait on each other's residency)."""
        torch = _torch()
        regions = [s.region for s in steps]
        for s in steps:
            s._build_peers(regions)
        evs = [[torch.cuda.Event() for _ in range(s.model.L)] for s in steps]
        rev = [[torch.cuda.Event() for _ in range(s.model.L)] for s in steps]
        for r, s in enumerate(steps):
            # one device: a kernel spinning on a fused barrier (the align kernel, launched early by
            # PDL with the FFN grid queued behind it) must not hold the SMs another rank's router
            # needs, so every rank's FFN stage also waits for every rank's router
            s._router_post = (lambda l, r=r: rev[r][l].record())

            def ffn_pre(l, r=r):
                cur = torch.cuda.current_stream()
                if r > 0:
                    cur.wait_event(evs[r - 1][l])
                if steps[r].fused:
                    for q in range(len(steps)):
                        cur.wait_event(rev[q][l])

            s._ffn_pre = ffn_pre
            s._ffn_post = (lambda l, r=r: evs[r][l].record())
            # one device: a combine grid spinning on the fused barrier must not hold the SMs the
            # later ranks' persistent FFN grids need, so every combine also waits for every FFN
            s._combine_pre = (lambda l: [torch.cuda.current_stream().wait_event(evs[q][l])
                                         for q in range(len(steps))])

    def connect_ipc(self, group=None) -> None:
        """Multi-process: exchange CUDA IPC handles over `group` and map the peers' regions."""
        import torch.distributed as dist

        handles = [None] * self.world
        dist.all_gather_object(handles, self.region.ipc_handle(), group=group)
        regions = []
        for r, h in enumerate(handles):
            if r == self.rank:
                regions.append(self.region)
                continue
            buf = (ctypes.c_char * 64).from_buffer_copy(h)
            p = ctypes.c_void_p()
            _lib.call("sere_ipc_open", buf, ctypes.byref(p))
            regions.append(PeerRegion.mapped(self.region, p.value))
        self._build_peers(regions)

    # ------------------------------------------------------------------ launches
    def _barrier(self) -> None:
        _lib.call("sere_ep_barrier", ctypes.byref(self.peers), self.epoch.data_ptr(), self.bar_status.data_ptr(),
                  ctypes.c_int64(self.timeout_ns), _moe._stream_ptr())

    def _launch(self) -> None:
        for _ in self._phases():
            pass

    def _phases(self):
        """The step's launches, yielding after each phase (prologue; then per layer router,
        FFN stage, combine) so that virtual ranks sharing one device can be interleaved phase
        by phase (`run_local`): every cross-rank event is recorded before it is waited on."""
        if self.peers is None:
            raise RuntimeError("P2PDecodeStep is not connected (connect_local / connect_ipc)")
        m, reg = self.model, self.region
        K, d_h = m.K, m.d_h
        own_h = reg.h_all[self.t0:self.t1]
        self.x.copy_(self.x_in)
        _lib.call("sere_residual_rmsnorm", self.x.data_ptr(), None, own_h.data_ptr(), self.T_local, d_h,
                  ctypes.c_float(self.eps), _moe._stream_ptr())
        for r, peer in enumerate(self.peer_regions):  # first layer's input rows to every rank
            if r != self.rank:
                peer.h_all[self.t0:self.t1].copy_(own_h)
        yield
        ws_bytes = reg.ws_bytes
        for l, layer in enumerate(m.layers):
            b = layer.bias
            _lib.call("sere_route_topk_ep", ctypes.byref(self.peers), own_h.data_ptr(), layer.w_router_t.data_ptr(),
                      b.data_ptr() if b is not None else None, self.T_local, d_h, m.M, K,
                      self.route_ws.data_ptr(), self.route_ws.numel(), _moe._stream_ptr())
            if self._router_post is not None:
                self._router_post(l)
            if not self.fused:
                self._barrier()
            yield
            if self._ffn_pre is not None:
                self._ffn_pre(l)
            self._events_on(l)  # stages 0-3 inside sere_moe_ffn_ep, 4-5 around the combine
            out = self.outs[l]
            rr = out.reroute
            dsim = layer.sim
            flags = 0 if dsim.validated else _rr.FLAG_CHECK_SIM
            bank = layer.bank
            _lib.call("sere_moe_ffn_ep", bank.data.data_ptr(), m.M, self.lo, self.hi, bank.n_shared, d_h, m.d_m,
                      _moe.activation_code(getattr(m, "activation", "silu")), dsim.values.data_ptr(), self.S, float(self.rho), flags,
                      reg.h_all.data_ptr(), reg.ids_all.data_ptr(), reg.w_all.data_ptr(), self.T, K,
                      rr.new_indices.data_ptr(), rr.expert_class.data_ptr(), rr.reroute_map.data_ptr(),
                      rr.active_list.data_ptr(), rr.n_active.data_ptr(), reg.ws_ptr, ws_bytes,
                      out.status.data_ptr(), ctypes.byref(self.peers) if self.fused else None, _moe._stream_ptr())
            dsim.validated = True
            if self._ffn_post is not None:
                self._ffn_post(l)
            if not self.fused:
                self._barrier()
            yield
            if self.fused and self._combine_pre is not None:
                self._combine_pre(l)
            _lib.call("sere_combine_ep", ctypes.byref(self.peers), rr.new_indices.data_ptr(), reg.ws_ptr,
                      self.hi - self.lo, bank.n_shared, self.n_shared_total, d_h, m.d_m, K, self.x.data_ptr(), None,
                      ctypes.c_float(self.eps), _moe._stream_ptr())
            self._events_off()
            yield

    @staticmethod
    def run_local(steps: list, streams: list) -> None:
        """One eager step of virtual ranks on one device (connect_local), each on its own
        stream, launched phase by phase in rank order."""
        torch = _torch()
        gens = [st._phases() for st in steps]
        live = list(range(len(steps)))
        while live:
            for r in list(live):
                with torch.cuda.stream(streams[r]):
                    try:
                        next(gens[r])
                    except StopIteration:
                        live.remove(r)

    @property
    def launches_per_step(self) -> int:
        """Library kernels per step: router, re-route/align, permute, fused FFN and combine per
        layer (+ 2 barrier kernels without the fused barriers), plus the first RMSNorm (the first
        layer's row copies not counted)."""
        return self.model.L * (5 if self.fused else 7) + 1

    def run(self) -> None:
        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch()

    def capture(self) -> bool:
        """Warm up, then capture the whole step (barriers and peer loads/stores are plain
        kernels, so the graph replays on every rank in lockstep)."""
        torch = _torch()
        self._launch()
        torch.cuda.synchronize()
        self.check()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launch()
        self.graph = g
        return True

    def run_host(self, x_host, out_host) -> None:
        self.x_in.copy_(x_host, non_blocking=True)
        self.run()
        out_host.copy_(self.x, non_blocking=True)

    @property
    def workspace(self) -> tuple[int, int]:
        """(device pointer, bytes) of this rank's layer workspace (kernel-only FFN replay)."""
        return self.region.ws_ptr, self.region.ws_bytes

    def check(self) -> None:
        from .errors import raise_for_status

        raise_for_status(int(self.bar_status.item()), "peer barrier")
        for o in self.outs:
            o.check()

    def active_counts(self) -> np.ndarray:
        torch = _torch()
        return torch.cat([o.reroute.n_active for o in self.outs]).cpu().numpy()

    def close(self) -> None:
        for r, reg in enumerate(self.peer_regions):
            if r != self.rank:
                reg.close()
        self.region.close()


__all__ = ["PeerRegion", "P2PDecodeStep"]
