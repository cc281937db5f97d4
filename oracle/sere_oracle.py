"""CPU oracle for the SERE batched-decode MoE path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference package's hot path
(`/root/reference/pkg/src/sere/`, pure Python + numpy). It exists to *check*
the CUDA path and to time the reference algorithm on the host; it is never
imported by the product package `paper_2602_07616_b200` (which fails loudly if
its CUDA library is missing). Allowed importers: `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py`.

Parity pin: every function here is checked against golden vectors produced by
running the real reference in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.json|npz`, checked by
`tests/test_oracle_golden.py`), including the reference's own fixtures
(Fig. 1 four-token batch, the CLI golden trace) and frozen values.

Each function cites the reference line range it restates. Arithmetic is
float64 with the reference's reduction order, so on identical inputs the
results are bit-identical to the reference (the golden tests assert equality,
not closeness, for ids and for the fp64 layer output).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2602_07616_b200.errors import (
    ConfigError,
    DimensionError,
    DomainError,
    InputError,
    RoutingError,
    SereError,
)

ACTIVATIONS = ("silu", "relu", "gelu-tanh")


# ---------------------------------------------------------------------------
# re-routing (reference: src/sere/rerouting.py)
# ---------------------------------------------------------------------------

@dataclass
class OracleReroute:
    """Field-for-field twin of `RerouteResult` (rerouting.py:57-65)."""

    new_indices: np.ndarray
    primary_set: frozenset
    preserved_critical: frozenset
    final_active: frozenset
    reroute_map: dict = field(default_factory=dict)


def validate_inputs(indices: np.ndarray, sim: np.ndarray, retain_count: int) -> None:
    """rerouting.py:100-116 (`_validate_inputs`), same check order."""
    k = indices.shape[1]
    if retain_count > k:
        raise ConfigError(f"retain_count must not exceed K (got S={retain_count}, K={k})")
    m = sim.shape[0]
    if sim.ndim != 2 or sim.shape != (m, m):
        raise DimensionError(f"similarity matrix must be square, got {sim.shape}")
    if indices.min(initial=0) < 0 or indices.max(initial=-1) >= m:
        raise DimensionError(f"similarity matrix of dimension {m} does not cover every routed index")
    if sim.min() < 0.0 or sim.max() > 1.0:
        raise InputError("similarity values must lie in [0, 1]")


def best_primary_match(expert: int, primary: frozenset, sim: np.ndarray) -> tuple[float, int]:
    """rerouting.py:78-97: ascending scan, strict `>`, ties to the lowest index."""
    if not primary:
        raise SereError("primary set is empty")
    best_s = -np.inf
    best_e = -1
    for cand in range(sim.shape[0]):
        if cand in primary:
            s = sim[expert, cand]
            if s > best_s:
                best_s = s
                best_e = cand
    return float(best_s), int(best_e)


def apply_sere(indices, sim, retain_count: int, threshold: float) -> OracleReroute:
    """rerouting.py:130-171 (`apply_sere`), including the S==K identity (119-127).

    `indices` int [T,K] (slot 0 strongest), `sim` float64 [M,M] (row = secondary,
    column = candidate). Weights are not an input: the reference never reads them.
    """
    idx = np.asarray(indices, dtype=np.int64)
    sim = np.asarray(sim, dtype=np.float64)
    if idx.ndim != 2:
        raise DimensionError("indices must be 2-D")
    if int(retain_count) < 1:
        raise ConfigError(f"retain_count must be >= 1, got {retain_count}")  # rerouting.py:45-46
    if not 0.0 <= float(threshold) <= 1.0:
        raise ConfigError(f"threshold must lie in [0, 1], got {threshold}")  # rerouting.py:48-49
    retain_count = int(retain_count)
    threshold = float(threshold)
    validate_inputs(idx, sim, retain_count)
    t_count, k = idx.shape
    if retain_count == k:
        everything = frozenset(np.unique(idx).tolist())
        return OracleReroute(idx.copy(), everything, frozenset(), everything, {})
    primary = frozenset(np.unique(idx[:, :retain_count]).tolist())
    new = idx.copy()
    matches: dict[int, tuple[float, int]] = {}
    preserved: set[int] = set()
    reroute_map: dict[int, int] = {}
    for kk in range(retain_count, k):
        for t in range(t_count):
            e = int(idx[t, kk])
            if e in primary:
                continue
            if e not in matches:
                matches[e] = best_primary_match(e, primary, sim)
            best_s, best_e = matches[e]
            if threshold > 0.0 and best_s < threshold:
                preserved.add(e)
            else:
                new[t, kk] = best_e
                reroute_map[e] = best_e
    return OracleReroute(new, primary, frozenset(preserved), primary | frozenset(preserved), reroute_map)


def apply_sere_set_algebra(indices, sim, retain_count: int, threshold: float):
    """Independent restatement: the reference test oracle (tests/test_rerouting.py:37-56).

    Returns (new_indices, primary, preserved, mapping). Only valid for S < K.
    """
    indices = np.asarray(indices, dtype=np.int64)
    k = indices.shape[1]
    primary = set(indices[:, :retain_count].ravel().tolist())
    secondary = sorted(set(indices[:, retain_count:].ravel().tolist()) - primary)
    preserved, mapping = set(), {}
    for e in secondary:
        best = min(sorted(primary), key=lambda c: (-sim[e, c], c))
        if threshold > 0.0 and sim[e, best] < threshold:
            preserved.add(e)
        else:
            mapping[e] = best
    new = indices.copy()
    for t in range(indices.shape[0]):
        for kk in range(retain_count, k):
            e = int(indices[t, kk])
            if e in mapping:
                new[t, kk] = mapping[e]
    return new, primary, preserved, mapping


# ---------------------------------------------------------------------------
# MoE math (reference: src/sere/moe.py)
# ---------------------------------------------------------------------------

def silu(x: np.ndarray) -> np.ndarray:
    """moe.py:28-35: x*sigmoid(x) split by sign."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = x[pos] / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = x[~pos] * ex / (1.0 + ex)
    return out


def relu(x: np.ndarray) -> np.ndarray:
    """moe.py:38-39."""
    return np.maximum(x, 0.0)


def gelu_tanh(x: np.ndarray) -> np.ndarray:
    """moe.py:42-45."""
    c = np.sqrt(2.0 / np.pi)
    return 0.5 * x * (1.0 + np.tanh(c * (x + 0.044715 * x**3)))


_ACT = {"silu": silu, "relu": relu, "gelu-tanh": gelu_tanh}


def activation_fn(kind: str):
    """moe.py:55-60."""
    try:
        return _ACT[kind]
    except KeyError:
        raise ConfigError(f"unknown activation {kind!r}, expected one of {ACTIVATIONS}") from None


@dataclass
class OracleExpert:
    """`ExpertWeights` (moe.py:70-101): w_gate/w_up [d_h,d_m], w_down [d_m,d_h], float64."""

    w_gate: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray


@dataclass
class OracleLayer:
    """`MoELayer` (moe.py:127-151) + `RouterWeights` (moe.py:104-124)."""

    experts: list
    w_router: np.ndarray
    top_k: int
    shared_experts: list = field(default_factory=list)

    @property
    def n_experts(self) -> int:
        return len(self.experts)


def expert_forward(e: OracleExpert, x: np.ndarray, activation: str = "silu") -> np.ndarray:
    """moe.py:235-245: act(x @ Wg) * (x @ Wu) @ Wd."""
    act = activation_fn(activation)
    gate = act(x @ e.w_gate)
    up = x @ e.w_up
    return (gate * up) @ e.w_down


def topk_softmax(logits: np.ndarray, k: int):
    """moe.py:248-265: stable descending argsort (ties -> lower index), softmax over the K picks."""
    logits = np.asarray(logits, dtype=np.float64)
    m = logits.shape[1]
    if not 1 <= k <= m:
        raise ConfigError(f"top_k must satisfy 1 <= K <= M (got K={k}, M={m})")
    order = np.argsort(-logits, axis=1, kind="stable")[:, :k]
    sel = np.take_along_axis(logits, order, axis=1)
    shifted = sel - sel.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    w = e / e.sum(axis=1, keepdims=True)
    return order.astype(np.int64), w


def route_topk(w_router: np.ndarray, top_k: int, x: np.ndarray):
    """moe.py:268-277."""
    return topk_softmax(x @ w_router, top_k)


def layer_forward(layer: OracleLayer, x: np.ndarray, indices, weights, activation: str = "silu") -> np.ndarray:
    """moe.py:280-310: fixed order (slot 0..K-1 per expert group, then shared experts)."""
    x = np.asarray(x, dtype=np.float64)
    idx = np.asarray(indices, dtype=np.int64)
    w = np.asarray(weights, dtype=np.float64)
    if idx.shape[0] != x.shape[0]:
        raise DimensionError(f"assignment covers {idx.shape[0]} tokens, batch has {x.shape[0]}")
    m = layer.n_experts
    if idx.min(initial=0) < 0 or idx.max(initial=-1) >= m:
        raise RoutingError(f"assignment refers to experts outside [0, {m})")
    y = np.zeros_like(x)
    for k in range(idx.shape[1]):
        col = idx[:, k]
        for e in np.unique(col):
            rows = np.flatnonzero(col == e)
            y[rows] += w[rows, k : k + 1] * expert_forward(layer.experts[e], x[rows], activation)
    for shared in layer.shared_experts:
        y += expert_forward(shared, x, activation)
    return y


def model_forward(layers, x, activation="silu", retain_count=None, threshold=None,
                  sims=None, phase="decode", phase_mode="all_phases", router_override=None):
    """moe.py:329-377 (per layer: route -> phase-gated apply_sere -> layer_forward).

    Returns (output, traces) with traces[l] = dict(original, weights, final, reroute, active).
    """
    apply_rewrite = retain_count is not None and (phase_mode == "all_phases" or phase == "decode")
    x = np.asarray(x, dtype=np.float64)
    traces = []
    for l, layer in enumerate(layers):
        if router_override is not None:
            idx, w = router_override(l, x)
        else:
            idx, w = route_topk(layer.w_router, layer.top_k, x)
        if apply_rewrite:
            res = apply_sere(idx, sims[l], retain_count, threshold)
            final = res.new_indices
            active = res.final_active
        else:
            res = None
            final = idx
            active = frozenset(np.unique(idx).tolist())
        x = layer_forward(layer, x, final, w, activation)
        traces.append(dict(original=idx, weights=w, final=final, reroute=res, active=active))
    return x, traces


def bf16_round(a) -> np.ndarray:
    """Round to bfloat16 (nearest-even, via float32) and widen back to float64: the values a
    bf16 tensor holds. Used to hand the oracle exactly what the device computes on."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def rms_norm(x: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    """x / sqrt(mean(x^2) + eps) per row (no gain): the pre-norm of the benchmark block."""
    x = np.asarray(x, dtype=np.float64)
    return x / np.sqrt((x * x).mean(axis=1, keepdims=True) + eps)


def block_forward(layers, x0, sims, retain_count, threshold, routes, eps: float = 1e-6,
                  activation: str = "silu"):
    """The pre-norm residual decode block the benchmark runs (decode.DecodeStep, block=
    "prenorm_residual"): per layer

        h = bf16(RMSNorm(x));  ids, w = routes[l];  ids' = apply_sere(ids, sims[l], S, rho)
        x = x + layer_forward(layer, h, ids', w)                    (moe.py:280-310, 362-375)

    The reference chains raw outputs (x <- layer_forward(x), moe.py:375); the block adds the
    residual stream and the RMSNorm around the same two reference operators. `routes[l]` are
    the router's (ids, weights) of layer l, teacher-forced from the device router exactly as
    `model_forward`'s router_override does (moe.py:334,363-364). `retain_count=None` skips
    the rewrite (plain top-k). Returns (x, traces) with traces[l] = dict(x, h, final, active).
    """
    x = np.asarray(x0, dtype=np.float64)
    traces = []
    for l, layer in enumerate(layers):
        h = bf16_round(rms_norm(x, eps))
        ids, w = routes[l]
        if retain_count is not None:
            res = apply_sere(ids, sims[l], retain_count, threshold)
            final, active = res.new_indices, res.final_active
        else:
            final = np.asarray(ids, dtype=np.int64)
            active = frozenset(np.unique(final).tolist())
        traces.append(dict(x=x, h=h, final=final, active=active))
        x = x + layer_forward(layer, h, final, w, activation)
    return x, traces


def gen_layers(seed: int, n_layers: int, n_experts: int, top_k: int, d_h: int, d_m: int,
               n_shared: int = 0) -> list:
    """moe.py:380-421 (`gen_model`): identical draw order, so the same seed gives the same tensors."""
    rng = np.random.default_rng(seed)
    scale = 1.0 / np.sqrt(d_h)

    def draw():
        return OracleExpert(
            w_gate=rng.standard_normal((d_h, d_m)) * scale,
            w_up=rng.standard_normal((d_h, d_m)) * scale,
            w_down=rng.standard_normal((d_m, d_h)) * scale,
        )

    layers = []
    for _ in range(n_layers):
        experts = [draw() for _ in range(n_experts)]
        shared = [draw() for _ in range(n_shared)]
        w_router = rng.standard_normal((d_h, n_experts)) * scale
        layers.append(OracleLayer(experts, w_router, top_k, shared))
    return layers


# ---------------------------------------------------------------------------
# input generators shared by tests and the bench (restating the reference tests)
# ---------------------------------------------------------------------------

def random_symmetric_sim(rng: np.random.Generator, m: int) -> np.ndarray:
    """tests/test_rerouting.py:23-29: (r + r.T)/2 with a unit diagonal."""
    r = rng.random((m, m))
    v = (r + r.T) / 2.0
    np.fill_diagonal(v, 1.0)
    return v


def random_assignment(rng: np.random.Generator, t: int, k: int, m: int):
    """tests/test_rerouting.py:32-34: top-k of a random 4-wide router."""
    w_router = rng.standard_normal((4, m))
    return route_topk(w_router, k, rng.standard_normal((t, 4)))


# ---------------------------------------------------------------------------
# similarity calibration (offline, activation-based)
# ---------------------------------------------------------------------------

def gaussian_batches(seed: int, n_batches: int, tokens_per_batch: int, d_h: int) -> list:
    """similarity.py:298-306: deterministic standard-normal calibration batches."""
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((tokens_per_batch, d_h)) for _ in range(n_batches)]


def _pair_raw(a: np.ndarray, b: np.ndarray, metric: str) -> float:
    """similarity.py:127-152, 262-270 (frobenius distance / mean row cosine)."""
    if metric == "frobenius":
        d = a - b
        return float(np.sqrt((d * d).sum()))
    if metric == "cosine":
        num = (a * b).sum(axis=1)
        na = np.sqrt((a * a).sum(axis=1))
        nb = np.sqrt((b * b).sum(axis=1))
        denom = na * nb
        safe = np.where(denom > 0.0, denom, 1.0)
        per_row = np.where(denom > 0.0, num / safe, 0.0)
        return float(per_row.sum() / a.shape[0])
    raise ValueError(metric)


def estimate_similarity_raw(layers, batches, metric: str, activation: str = "silu") -> list:
    """similarity.py:325-371: per batch and layer, every routed expert runs densely on the
    layer input, each unordered pair (diagonal once) is scored and accumulated, and the batch
    advances through the routed forward (route_topk + layer_forward); averaged over batches."""
    raw = [np.zeros((len(l.experts), len(l.experts))) for l in layers]
    for batch in batches:
        x = np.asarray(batch, dtype=np.float64)
        for li, layer in enumerate(layers):
            slabs = [expert_forward(e, x, activation) for e in layer.experts]
            m = len(slabs)
            for p in range(m):
                for q in range(p, m):
                    s = _pair_raw(slabs[p], slabs[q], metric)
                    if p == q:
                        raw[li][p, p] += s
                    else:
                        raw[li][p, q] += s
                        raw[li][q, p] += s
            ids, w = route_topk(layer.w_router, layer.top_k, x)
            x = layer_forward(layer, x, ids, w, activation)
    return [r / len(batches) for r in raw]


def normalize_to_unit(raw: np.ndarray, metric: str) -> np.ndarray:
    """similarity.py:273-295 (+ frobenius_normalize 155-177): distances -> 1 - d/max(offdiag),
    cosines -> (c+1)/2 clipped; diagonal exactly 1."""
    raw = np.asarray(raw, dtype=np.float64)
    if metric == "frobenius":
        off = raw[~np.eye(raw.shape[0], dtype=bool)]
        mx = float(off.max()) if off.size else 0.0
        values = np.ones_like(raw) if mx == 0.0 else 1.0 - raw / mx
    else:
        values = np.clip((raw + 1.0) / 2.0, 0.0, 1.0)
    np.fill_diagonal(values, 1.0)
    return values
