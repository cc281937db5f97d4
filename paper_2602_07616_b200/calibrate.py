"""Expert-similarity calibration on the GPU (reference similarity.py:325-383).

Activation-based estimation, restating `similarity.estimate_similarity_raw`: for every
calibration batch and layer, every routed expert runs densely on the layer input, each
unordered expert pair is scored (Frobenius distance of the two output slabs, or the mean
row cosine), scores are averaged over batches, and the batch advances through the
routed forward (router top-K -> grouped FFN, this package's kernels) to the next layer.
`normalize_to_unit` maps the averaged matrix into [0, 1] exactly as the reference does.

This is the offline step that produces the `sim.layer{l}.json` files the decode path
consumes (`io.save_similarity`). The dense expert outputs are plain batched GEMMs
(cuBLAS, fp32); the pair scores come from one fp64 Gram matrix per layer,
||a-b||^2 = ||a||^2 + ||b||^2 - 2<a,b> (CKA metrics are not offered on the GPU).
The reference's Frobenius calibration costs 28 s on CPU.
"""

from __future__ import annotations

from typing import Any, Iterable

import numpy as np

from . import moe as _moe
from .errors import ConfigError, DimensionError, DomainError, InputError

METRICS = ("frobenius", "cosine")


def _torch():
    import torch

    return torch


def _layers(model: Any) -> list:
    """(bank, router weight [d_h, M], router bias or None, top_k) per layer of a
    `decode.DecodeModel` or an `io.GpuModel`."""
    out = []
    for layer in model.layers:
        if hasattr(layer, "router"):  # io.GpuLayer
            out.append((layer.bank, layer.router.w_router, None, int(layer.router.top_k)))
        else:  # decode.DecodeLayer (its benchmark bias is part of its router)
            out.append((layer.bank, layer.w_router, getattr(layer, "bias", None), int(model.K)))
    return out


def _act(kind: str):
    torch = _torch()
    if kind == "silu":
        return torch.nn.functional.silu
    if kind == "relu":
        return torch.relu
    if kind == "gelu-tanh":  # the reference's spelling (moe.py:22,42-45; moe.ACTIVATIONS)
        return lambda g: torch.nn.functional.gelu(g, approximate="tanh")
    raise ConfigError(f"unknown activation {kind!r}, expected one of {_moe.ACTIVATIONS}")


def _pair_scores(y, metric: str) -> np.ndarray:
    """[M, T, d_h] fp32 expert outputs -> [M, M] raw pair scores (similarity.py:127-152)."""
    torch = _torch()
    m = y.shape[0]
    if metric == "frobenius":
        f = y.reshape(m, -1).double()
        g = f @ f.t()
        sq = torch.diagonal(g)
        d = (sq[:, None] + sq[None, :] - 2.0 * g).clamp_min(0.0).sqrt()
        d.fill_diagonal_(0.0)  # ||a - a|| is exactly 0 in the reference
        d = (d + d.t()) / 2.0  # exact symmetry, as the reference fills both triangles from one score
        return d.cpu().numpy()
    yd = y.double()
    n = yd.norm(dim=2, keepdim=True)
    yn = torch.where(n > 0, yd / torch.where(n > 0, n, torch.ones_like(n)), torch.zeros_like(yd))
    f = yn.reshape(m, -1)
    c = (f @ f.t()) / float(y.shape[1])
    c = (c + c.t()) / 2.0
    return c.cpu().numpy()


def estimate_similarity_raw(model: Any, batches: Iterable[Any], metric: str = "frobenius",
                            activation: str = "silu") -> list[np.ndarray]:
    """similarity.py:325-371 on the GPU: averaged raw pair scores, one [M, M] per layer."""
    torch = _torch()
    if metric not in METRICS:
        raise ConfigError(f"unknown metric {metric!r} for GPU calibration, expected one of {METRICS}")
    layers = _layers(model)
    dev = layers[0][0].device
    d_h = layers[0][0].d_h
    blist = [torch.as_tensor(np.asarray(b) if not hasattr(b, "device") else b, dtype=torch.float32).to(dev)
             for b in batches]
    if not blist:
        raise InputError("no calibration batches supplied")
    for b in blist:
        if b.ndim != 2 or b.shape[1] != d_h:
            raise DimensionError(f"calibration batches must be T x d_h with d_h={d_h}, got {tuple(b.shape)}")
        if not bool(torch.isfinite(b).all()):
            raise DomainError("calibration batch contains non-finite values")
    act = _act(activation)
    raw = [np.zeros((bank.M, bank.M)) for bank, *_ in layers]
    for x in blist:
        for l, (bank, w_router, bias, k) in enumerate(layers):
            wg, wu, wd = bank.unpack(0, bank.M)  # routed experts only (shared ones are never scored)
            wg, wu, wd = wg.float(), wu.float(), wd.float()
            h = act(torch.matmul(x, wg)) * torch.matmul(x, wu)  # [M, T, d_m]
            y = torch.matmul(h, wd)                             # [M, T, d_h]
            del wg, wu, wd, h
            raw[l] += _pair_scores(y, metric)
            del y
            xb = x.to(torch.bfloat16)
            ids, w = _moe.route_topk_device(_moe.router_weight_t(w_router), xb, k, bias=bias)
            out = _moe.layer_forward_device(bank, xb, ids, w, activation)
            out.check()
            x = out.y
    return [r / len(blist) for r in raw]


def normalize_to_unit(raw: np.ndarray, metric: str) -> np.ndarray:
    """similarity.py:273-295 with frobenius_normalize 155-177: Frobenius distances flip and
    rescale by the off-diagonal maximum, cosines shift from [-1, 1]; diagonal exactly 1."""
    raw = np.asarray(raw, dtype=np.float64)
    if raw.ndim != 2 or raw.shape[0] != raw.shape[1]:
        raise DimensionError(f"raw matrix must be square, got {raw.shape}")
    if metric == "frobenius":
        off = raw[~np.eye(raw.shape[0], dtype=bool)]
        mx = float(off.max()) if off.size else 0.0
        values = np.ones_like(raw) if mx == 0.0 else 1.0 - raw / mx
    else:
        values = (raw + 1.0) / 2.0
    values = np.clip(values, 0.0, 1.0)
    np.fill_diagonal(values, 1.0)
    return values


def estimate_similarity(model: Any, batches: Iterable[Any], metric: str = "frobenius",
                        activation: str = "silu") -> list[np.ndarray]:
    """similarity.py:374-383: per-layer similarity matrices (fp64 [M, M], validated)."""
    from .io import validate_similarity

    sims = [normalize_to_unit(r, metric) for r in estimate_similarity_raw(model, batches, metric, activation)]
    for s in sims:
        validate_similarity(s)
    return sims


def calibrate_to_dir(model: Any, batches: Iterable[Any], directory, metric: str = "frobenius",
                     activation: str = "silu") -> list:
    """The reference CLI's `calibrate` output (cli.py -> similarity.save_similarity_set):
    one sim.layer{l}.json (+ .f32) per layer in `directory`; returns the written paths."""
    from .io import save_similarity

    sims = estimate_similarity(model, batches, metric, activation)
    return [save_similarity(s, directory, layer_index=l, metric=metric) for l, s in enumerate(sims)]


__all__ = ["METRICS", "estimate_similarity_raw", "estimate_similarity", "normalize_to_unit", "calibrate_to_dir"]
