"""Reference file formats <-> the GPU layout.

The reference serialises a model as `model.json` plus one little-endian float32
file per tensor (`moe.py:428-512`): `layer{l}.expert{j}.{gate,up,down}.f32`,
`layer{l}.shared{j}.{gate,up,down}.f32`, `layer{l}.router.f32`, row-major in the
`x @ W` orientation. Similarity matrices are `sim.layer{l}.json` (+ an f32 twin,
`similarity.py:438-487`).

`load_model` streams every expert file straight into a bf16 `ExpertBank` on the
GPU (no fp64 copy of the whole model on the host, unlike the reference loader),
so reference model directories run on the B200 path; `save_model` writes the
same format back from the banks. The returned `GpuModel` is accepted by
`moe.model_forward` like a reference `MoEModel`.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Any

import numpy as np

from . import moe as _moe
from .errors import ConfigError, DimensionError, DomainError, InputError

MODEL_META_NAME = "model.json"  # moe.py:25


def _torch():
    import torch

    return torch


def _read_f32(path: Path, shape: tuple[int, ...]) -> np.ndarray:
    """moe.py:432-437 (float32 kept: the bank stores bf16)."""
    if not path.is_file():
        raise InputError(f"{path} not found")
    raw = np.fromfile(path, dtype="<f4")
    expected = int(np.prod(shape))
    if raw.size != expected:
        raise DimensionError(f"{path.name} holds {raw.size} values, expected {expected}")
    return raw.reshape(shape)


def _write_f32(path: Path, a) -> None:
    path.write_bytes(np.ascontiguousarray(np.asarray(a), dtype="<f4").tobytes())


@dataclass
class GpuRouter:
    w_router: Any  # bf16 CUDA tensor [d_h, M] (reference orientation)
    top_k: int


@dataclass
class GpuLayer:
    bank: Any  # moe.ExpertBank (routed experts then shared experts)
    router: GpuRouter

    @property
    def n_experts(self) -> int:
        return self.bank.M


@dataclass
class GpuModel:
    layers: list
    d_h: int
    activation: str
    seed: Any = None

    @property
    def n_layers(self) -> int:
        return len(self.layers)


def load_model(directory, device=None, chunk: int = 8) -> GpuModel:
    """moe.py:476-512 into GPU banks: experts are read `chunk` at a time, converted to
    bf16 on the device and packed (`sere_pack_experts`)."""
    torch = _torch()
    directory = Path(directory)
    meta_path = directory / MODEL_META_NAME
    if not meta_path.is_file():
        raise InputError(f"{meta_path} not found")
    meta = json.loads(meta_path.read_text())
    d_h, d_m = int(meta["d_h"]), int(meta["d_m"])
    M, K, n_sh = int(meta["n_experts"]), int(meta["top_k"]), int(meta["n_shared"])
    act = str(meta["activation"])
    _moe.activation_code(act)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    names = [f"expert{j}" for j in range(M)] + [f"shared{j}" for j in range(n_sh)]
    layers = []
    for l in range(int(meta["n_layers"])):
        bank = _moe.ExpertBank(M, n_sh, d_h, d_m, dev)
        for first in range(0, len(names), chunk):
            part = names[first:first + chunk]
            wg = np.stack([_read_f32(directory / f"layer{l}.{n}.gate.f32", (d_h, d_m)) for n in part])
            wu = np.stack([_read_f32(directory / f"layer{l}.{n}.up.f32", (d_h, d_m)) for n in part])
            wd = np.stack([_read_f32(directory / f"layer{l}.{n}.down.f32", (d_m, d_h)) for n in part])
            bank.pack(*(torch.from_numpy(a).to(dev, torch.bfloat16) for a in (wg, wu, wd)), first=first)
        wr = torch.from_numpy(_read_f32(directory / f"layer{l}.router.f32", (d_h, M))).to(dev, torch.bfloat16)
        layers.append(GpuLayer(bank, GpuRouter(wr, K)))
    return GpuModel(layers, d_h, act, meta.get("seed"))


def model_meta(seed, n_layers: int, n_experts: int, top_k: int, d_h: int, d_m: int, n_shared: int,
               activation: str) -> dict:
    """model.json of moe.py:445-454 (same keys, same order)."""
    return {"seed": seed, "n_layers": n_layers, "n_experts": n_experts, "top_k": top_k, "d_h": d_h, "d_m": d_m,
            "n_shared": n_shared, "activation": activation}


def write_model_dir(directory, meta: dict, layers) -> None:
    """The byte layout of the reference's save_model (moe.py:440-473): model.json, then per
    layer the routed experts' gate/up/down, the shared experts', and the router, each a
    little-endian float32 row-major file. `layers` yields (w_gate [E,d_h,d_m], w_up,
    w_down [E,d_m,d_h], w_router [d_h,M]) host arrays with the routed experts first."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    (directory / MODEL_META_NAME).write_text(json.dumps(meta, indent=2) + "\n")
    n_routed = int(meta["n_experts"])
    for l, (wg, wu, wd, w_router) in enumerate(layers):
        for j in range(len(wg)):
            name = f"expert{j}" if j < n_routed else f"shared{j - n_routed}"
            _write_f32(directory / f"layer{l}.{name}.gate.f32", wg[j])
            _write_f32(directory / f"layer{l}.{name}.up.f32", wu[j])
            _write_f32(directory / f"layer{l}.{name}.down.f32", wd[j])
        _write_f32(directory / f"layer{l}.router.f32", w_router)


def save_model(model: GpuModel, directory) -> None:
    """moe.py:440-473 from GPU banks (bf16 values written as float32), one layer's
    tensors on the host at a time."""
    first = model.layers[0]
    meta = model_meta(model.seed, model.n_layers, first.bank.M, first.router.top_k, model.d_h, first.bank.d_m,
                      first.bank.n_shared, model.activation)
    for layer in model.layers:
        b = layer.bank
        if (b.M, b.n_shared, b.d_m, layer.router.top_k) != (meta["n_experts"], meta["n_shared"], meta["d_m"],
                                                          meta["top_k"]):
            raise ConfigError("only homogeneous layer stacks can be serialized")

    def host_layers():
        for layer in model.layers:
            wg, wu, wd = (t.float().cpu().numpy() for t in layer.bank.unpack())
            yield wg, wu, wd, layer.router.w_router.float().cpu().numpy()

    write_model_dir(directory, meta, host_layers())


# ---------------------------------------------------------------------------
# similarity matrices (similarity.py:70-90, 438-487)
# ---------------------------------------------------------------------------

def sim_json_name(layer_index: int) -> str:
    return f"sim.layer{layer_index}.json"


def sim_f32_name(layer_index: int) -> str:
    return f"sim.layer{layer_index}.f32"


def validate_similarity(v: np.ndarray) -> None:
    """SimilarityMatrix.validate (similarity.py:82-91)."""
    if v.ndim != 2 or v.shape[0] != v.shape[1]:
        raise DimensionError(f"similarity matrix must be square, got {v.shape}")
    if not np.array_equal(v, v.T):
        raise DomainError("similarity matrix must be exactly symmetric")
    if v.min() < 0.0 or v.max() > 1.0:
        raise DomainError("similarity values must lie in [0, 1]")
    if not np.all(np.diag(v) == 1.0):
        raise DomainError("similarity diagonal must be exactly 1")


def load_similarity(path) -> np.ndarray:
    """similarity.py:468-476: fp64 values of sim.layer{l}.json (validated)."""
    payload = json.loads(Path(path).read_text())
    v = np.asarray(payload["values"], dtype=np.float64)
    validate_similarity(v)
    return v


def load_similarity_set(directory, n_layers: int) -> list:
    """similarity.py:479-487."""
    directory = Path(directory)
    sims = []
    for l in range(n_layers):
        path = directory / sim_json_name(l)
        if not path.is_file():
            raise InputError(f"missing similarity file {path}")
        sims.append(load_similarity(path))
    return sims


def save_similarity(values, directory, layer_index: int = 0, metric: str = "frobenius",
                    write_f32: bool = True) -> Path:
    """similarity.py:446-465."""
    v = np.asarray(values, dtype=np.float64)
    validate_similarity(v)
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    payload = {"metric": metric, "layer": layer_index, "n_experts": v.shape[0],
               "values": [[float(x) for x in row] for row in v]}
    path = directory / sim_json_name(layer_index)
    path.write_text(json.dumps(payload, indent=2) + "\n")
    if write_f32:
        (directory / sim_f32_name(layer_index)).write_bytes(np.ascontiguousarray(v, dtype="<f4").tobytes())
    return path


__all__ = ["GpuModel", "GpuLayer", "GpuRouter", "load_model", "save_model", "write_model_dir", "model_meta", "load_similarity",
           "load_similarity_set", "save_similarity", "validate_similarity", "MODEL_META_NAME"]
