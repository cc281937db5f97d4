"""GPU-backed mirror of the reference `sere.rerouting` module.

Same names, argument meaning and error behaviour as
`/root/reference/pkg/src/sere/rerouting.py`; the computation runs in the
sm_100a re-routing kernel (`sere_reroute`, csrc/reroute_align.cu), bit-exact
with the reference on the same inputs.

Two levels:
  * `apply_sere(assignment, sim, config) -> RerouteResult` -- the drop-in
    (rerouting.py:130): host arrays in, host sets out; one device sync.
  * `reroute(ids, sim, retain_count, threshold) -> DeviceReroute` -- the
    device path used inside the layer pipeline: int32 CUDA tensors in and out,
    asynchronous; the Python sets are materialised lazily.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any

import numpy as np

from . import _lib
from .errors import ConfigError, DimensionError, InputError, SereError, raise_for_status

PHASE_MODES = ("all_phases", "decode_only")

CLASS_PRIMARY, CLASS_CRITICAL, CLASS_REROUTED = 1, 2, 4
FLAG_CHECK_SIM = 1


@dataclass(frozen=True)
class RerouteConfig:
    """rerouting.py:31-54: keep top `retain_count` slots, redirect the rest unless
    their best similarity falls below `threshold`."""

    retain_count: int
    threshold: float
    phase_mode: str = "all_phases"

    def __post_init__(self) -> None:
        if int(self.retain_count) < 1:
            raise ConfigError(f"retain_count must be >= 1, got {self.retain_count}")
        object.__setattr__(self, "retain_count", int(self.retain_count))
        if not 0.0 <= float(self.threshold) <= 1.0:
            raise ConfigError(f"threshold must lie in [0, 1], got {self.threshold}")
        object.__setattr__(self, "threshold", float(self.threshold))
        if self.phase_mode not in PHASE_MODES:
            raise ConfigError(f"phase_mode must be one of {PHASE_MODES}, got {self.phase_mode!r}")


@dataclass
class RerouteResult:
    """rerouting.py:57-65."""

    new_indices: np.ndarray
    primary_set: frozenset
    preserved_critical: frozenset
    final_active: frozenset
    reroute_map: dict


def _torch():
    import torch

    return torch


class DeviceSimilarity:
    """A layer's M x M similarity matrix resident in HBM as float64 (compared in fp64,
    SURVEY Appendix A item 5). Shape is checked on construction (DimensionError,
    rerouting.py:108-110); the [0,1] range is checked on the device at first use
    (InputError, rerouting.py:115-116; NaN passes exactly as in the reference)."""

    def __init__(self, values: Any, device=None):
        torch = _torch()
        if isinstance(values, torch.Tensor):
            t = values.detach()
        else:
            v = getattr(values, "values", values)
            t = torch.as_tensor(np.asarray(v, dtype=np.float64))
        if t.ndim != 2 or t.shape[0] != t.shape[1]:
            raise DimensionError(f"similarity matrix must be square, got {tuple(t.shape)}")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.values = t.to(device=dev, dtype=torch.float64).contiguous()
        self.m = int(t.shape[0])
        self.validated = False

    @property
    def device(self):
        return self.values.device


def as_device_sim(sim: Any, device=None) -> DeviceSimilarity:
    if isinstance(sim, DeviceSimilarity):
        return sim
    return DeviceSimilarity(sim, device)


@dataclass
class DeviceReroute:
    """Device-resident re-routing result (`sere_reroute` outputs)."""

    new_indices: Any          # int32 [T,K] cuda
    expert_class: Any         # uint8 [M]  (CLASS_* flags)
    reroute_map: Any          # int32 [M]  (-1 unless rerouted)
    active_list: Any          # int32 [M]  (first n_active valid, ascending)
    n_active: Any             # int32 [1]
    status: Any               # int32 [1]
    _host: dict = field(default_factory=dict)

    def check(self) -> None:
        """Sync on the status word and raise the reference exception if a device check failed."""
        raise_for_status(int(self.status.item()), "sere_reroute")

    def to_result(self) -> RerouteResult:
        """Materialise the reference RerouteResult (one D2H copy)."""
        self.check()
        ids = self.new_indices.cpu().numpy().astype(np.int64)
        cls = self.expert_class.cpu().numpy()
        rmap = self.reroute_map.cpu().numpy()
        primary = frozenset(np.flatnonzero(cls & CLASS_PRIMARY).tolist())
        critical = frozenset(np.flatnonzero(cls & CLASS_CRITICAL).tolist())
        rerouted = np.flatnonzero(cls & CLASS_REROUTED).tolist()
        return RerouteResult(
            new_indices=ids,
            primary_set=primary,
            preserved_critical=critical,
            final_active=primary | critical,
            reroute_map={int(e): int(rmap[e]) for e in rerouted},
        )


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def reroute(ids, sim: Any, retain_count: int, threshold: float, stream=None, out: DeviceReroute | None = None,
            check_sim: bool | None = None) -> DeviceReroute:
    """Device re-routing: `ids` int32 [T,K] CUDA tensor, `sim` DeviceSimilarity (or array).

    Host-side checks follow rerouting.py:45-54 and 104-110; id range and sim range
    are checked on the device (see DeviceReroute.check)."""
    torch = _torch()
    cfg = RerouteConfig(retain_count, threshold)  # ConfigError for S<1 / rho outside [0,1]
    if ids.ndim != 2:
        raise DimensionError(f"indices must be 2-D, got shape {tuple(ids.shape)}")
    T, K = int(ids.shape[0]), int(ids.shape[1])
    if cfg.retain_count > K:
        raise ConfigError(f"retain_count must not exceed K (got S={cfg.retain_count}, K={K})")
    dsim = as_device_sim(sim, ids.device)
    M = dsim.m
    dev = ids.device
    _lib.ensure_device(dev.index if dev.index is not None else torch.cuda.current_device())
    ids = ids.to(torch.int32).contiguous()
    if out is None:
        out = DeviceReroute(
            new_indices=torch.empty((T, K), dtype=torch.int32, device=dev),
            expert_class=torch.empty(M, dtype=torch.uint8, device=dev),
            reroute_map=torch.empty(M, dtype=torch.int32, device=dev),
            active_list=torch.empty(M, dtype=torch.int32, device=dev),
            n_active=torch.empty(1, dtype=torch.int32, device=dev),
            status=torch.empty(1, dtype=torch.int32, device=dev),
        )
    if check_sim is None:
        check_sim = not dsim.validated
    flags = FLAG_CHECK_SIM if check_sim else 0
    _lib.call("sere_reroute", ids.data_ptr(), dsim.values.data_ptr(), T, K, M, cfg.retain_count,
              cfg.threshold, flags, out.new_indices.data_ptr(), out.expert_class.data_ptr(),
              out.reroute_map.data_ptr(), out.active_list.data_ptr(), out.n_active.data_ptr(),
              out.status.data_ptr(), _stream_ptr(stream))
    if check_sim:
        dsim.validated = True  # provisional; apply_sere clears it again if the device rejects the matrix
    return out


MAX_CELLS = 16384  # T*K per call (capi.cu kMaxCells)
MAX_EXPERTS = 256  # capi.cu kMaxExperts


def device_supports(n_tokens: int, top_k: int, n_experts: int) -> bool:
    """Whether `sere_reroute` takes this shape (`integration.install` falls back beyond it)."""
    return n_tokens * top_k <= MAX_CELLS and 1 <= n_experts <= MAX_EXPERTS


def apply_sere(assignment: Any, sim: Any, config: RerouteConfig) -> RerouteResult:
    """Drop-in for rerouting.apply_sere (rerouting.py:130-171), computed on the GPU.

    `assignment` needs `.indices` [T,K] (a reference RoutingAssignment works),
    `sim` a reference SimilarityMatrix / ndarray / DeviceSimilarity, `config` any
    object with retain_count / threshold (reference or this module's RerouteConfig)."""
    torch = _torch()
    idx = np.asarray(getattr(assignment, "indices", assignment))
    if idx.ndim != 2:
        raise DimensionError(f"indices must be 2-D, got shape {idx.shape}")
    k = idx.shape[1]
    if int(config.retain_count) > k:  # order of _validate_inputs: config first
        raise ConfigError(f"retain_count must not exceed K (got S={config.retain_count}, K={k})")
    dev = torch.device("cuda", torch.cuda.current_device())
    # stateless like the reference: the CURRENT values are uploaded (M*M*8 B, 128 KiB at
    # M=128) and range-checked on every call (rerouting.py:140, _validate_inputs 108-116);
    # only the device-level API (`reroute` with a DeviceSimilarity) keeps a resident copy
    dsim = sim if isinstance(sim, DeviceSimilarity) else DeviceSimilarity(sim, dev)
    if idx.size and (idx.min() < np.iinfo(np.int32).min or idx.max() > np.iinfo(np.int32).max):
        raise DimensionError(f"similarity matrix of dimension {dsim.m} does not cover every routed index")
    ids = torch.as_tensor(idx.astype(np.int32)).to(dev)
    res = reroute(ids, dsim, int(config.retain_count), float(config.threshold), check_sim=True)
    try:
        return res.to_result()
    except InputError:
        dsim.validated = False
        raise


def select_primary(assignment: Any, retain_count: int) -> frozenset:
    """rerouting.py:68-75: union of every token's strongest `retain_count` ids (1 <= S < K)."""
    idx = np.asarray(getattr(assignment, "indices", assignment))
    k = idx.shape[1]
    if not 1 <= retain_count < k:
        raise ConfigError(f"retain_count must satisfy 1 <= S < K (got S={retain_count}, K={k})")
    torch = _torch()
    m = int(idx.max()) + 1 if idx.size else 1
    ident = torch.eye(m, dtype=torch.float64)
    res = reroute(torch.as_tensor(idx.astype(np.int32)).cuda(), ident, retain_count, 1.0)
    r = res.to_result()
    return r.primary_set


def final_active_set(result: RerouteResult) -> frozenset:
    """rerouting.py:252-254."""
    return result.primary_set | result.preserved_critical


# ---------------------------------------------------------------------------
# JSON forms (rerouting.py:261-288) -- trace I/O, identical format
# ---------------------------------------------------------------------------

def result_to_dict(result: RerouteResult) -> dict:
    return {
        "new_indices": np.asarray(result.new_indices).tolist(),
        "primary_set": sorted(result.primary_set),
        "preserved_critical": sorted(result.preserved_critical),
        "final_active": sorted(result.final_active),
        "reroute_map": {str(u): int(v) for u, v in sorted(result.reroute_map.items())},
    }


def result_from_dict(d: dict) -> RerouteResult:
    return RerouteResult(
        new_indices=np.asarray(d["new_indices"], dtype=np.int64),
        primary_set=frozenset(int(e) for e in d["primary_set"]),
        preserved_critical=frozenset(int(e) for e in d["preserved_critical"]),
        final_active=frozenset(int(e) for e in d["final_active"]),
        reroute_map={int(u): int(v) for u, v in d["reroute_map"].items()},
    )


def save_trace(layers: list, path) -> None:
    Path(path).write_text(json.dumps({"layers": layers}, indent=2) + "\n")


def load_trace(path) -> dict:
    return json.loads(Path(path).read_text())


__all__ = [
    "PHASE_MODES", "RerouteConfig", "RerouteResult", "DeviceSimilarity", "DeviceReroute", "reroute",
    "device_supports",
    "apply_sere", "select_primary", "final_active_set", "result_to_dict", "result_from_dict",
    "save_trace", "load_trace", "SereError",
]
