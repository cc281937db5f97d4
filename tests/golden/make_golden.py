"""Generate golden vectors by running the REAL reference package (build container only).

    python tests/golden/make_golden.py

Imports `sere` from /root/reference/pkg/src (read-only, pure Python + numpy)
and records its outputs on seeded inputs. The GPU box has no /root/reference,
so the results are committed here and the tests read only these files:

  reroute_cases.npz   apply_sere inputs/outputs: the Fig. 1 four-token batch
                      (tests/fixtures/four_token_*.json), both layers of the CLI
                      golden trace (tests/fixtures/golden/*), a C3-style random
                      sweep (tests/test_acceptance.py:93-115 generator) and
                      BASELINE-shape instances (M=8/64/128, K=2/6/8) over a rho
                      grid and S in {1,2}; sims of the large instances are stored
                      by seed (numpy PCG64 `random` is stream-stable) and
                      re-derived by `oracle.sere_oracle.random_symmetric_sim`.
  layer_cases.npz     layer_forward / model_forward outputs (fp64) for small
                      gen_model configs (weights re-derived from the seed by
                      `oracle.sere_oracle.gen_layers`, same draw order).
  topk_cases.npz      topk_softmax outputs incl. ties.
  calib_cases.npz     estimate_similarity_raw / estimate_similarity (frobenius, cosine)
                      of a small gen_model on gaussian_batches.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_FIX = Path("/root/reference/pkg/tests/fixtures")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF_SRC))

from sere import moe, rerouting, similarity  # noqa: E402  (the reference)


class Ragged:
    """Pack many small arrays of one dtype into a flat array + offsets + shapes."""

    def __init__(self, dtype):
        self.dtype = dtype
        self.parts, self.shapes = [], []

    def add(self, a):
        a = np.asarray(a, dtype=self.dtype)
        self.parts.append(a.ravel())
        self.shapes.append(a.shape + (1,) * (2 - a.ndim) if a.ndim < 2 else a.shape)

    def dump(self, prefix, out):
        flat = np.concatenate(self.parts) if self.parts else np.zeros(0, self.dtype)
        lens = np.array([p.size for p in self.parts], dtype=np.int64)
        out[prefix + "_flat"] = flat
        out[prefix + "_off"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        out[prefix + "_shape"] = np.array(self.shapes, dtype=np.int64).reshape(-1, 2)


def _sym(rng, m):
    r = rng.random((m, m))
    v = (r + r.T) / 2.0
    np.fill_diagonal(v, 1.0)
    return v


def _assign(rng, t, k, m):
    router = moe.RouterWeights(w_router=rng.standard_normal((4, m)), top_k=k)
    return moe.route_topk(router, rng.standard_normal((t, 4)))


def reroute_cases():
    ids_in, ids_out, sims = Ragged(np.int64), Ragged(np.int64), Ragged(np.float64)
    sets = []
    meta = []  # (S, rho, sim_kind, sim_seed, M, source)

    def record(idx, sim_values, s, rho, source, sim_seed=-1):
        a = moe.RoutingAssignment(indices=idx, weights=np.full(np.shape(idx), 1.0 / np.shape(idx)[1]))
        sm = similarity.SimilarityMatrix(values=sim_values, metric="cosine")
        res = rerouting.apply_sere(a, sm, rerouting.RerouteConfig(retain_count=s, threshold=rho))
        ids_in.add(idx)
        ids_out.add(res.new_indices)
        if sim_seed >= 0:
            sims.add(np.zeros((0, 0)))
        else:
            sims.add(sim_values)
        sets.append(dict(
            primary=sorted(res.primary_set),
            critical=sorted(res.preserved_critical),
            active=sorted(res.final_active),
            map={str(u): int(v) for u, v in sorted(res.reroute_map.items())},
        ))
        meta.append((s, rho, sim_seed, np.shape(sim_values)[0], source))

    # Fig. 1 (reference fixture, tests/test_rerouting.py:118-127)
    fa = json.loads((REF_FIX / "four_token_assignment.json").read_text())
    fs = json.loads((REF_FIX / "four_token_similarity.json").read_text())
    for rho in (0.5, 0.0, 0.2, 0.35, 1.0):
        for s in (1, 2):
            record(np.array(fa["indices"]), np.array(fs["values"]), s, rho, "fig1")

    # CLI golden trace: original_indices of both layers against the golden sims (S=1, rho=0.3)
    trace = json.loads((REF_FIX / "golden" / "reroute_trace.json").read_text())
    for layer in trace["layers"]:
        l = layer["layer"]
        sv = json.loads((REF_FIX / "golden" / f"calibrate_sim.layer{l}.json").read_text())["values"]
        record(np.array(layer["original_indices"]), np.array(sv), 1, 0.3, f"trace{l}")
        # sanity: the reference reproduces its own stored trace
        assert sets[-1]["map"] == layer["reroute_map"], "golden trace not reproduced"
        for rho in (0.0, 0.6, 0.9):
            record(np.array(layer["original_indices"]), np.array(sv), 1, rho, f"trace{l}")

    # C3-style sweep (tests/test_acceptance.py:93-115 generator)
    for i in range(400):
        rng = np.random.default_rng([200, i])
        m = int(rng.integers(6, 13))
        k = int(rng.integers(2, 5))
        t = int(rng.integers(1, 9))
        s = int(rng.integers(1, k))
        a = _assign(rng, t, k, m)
        sv = _sym(rng, m)
        rho = float(rng.random())
        record(a.indices, sv, s, rho, "c3")
        if i % 4 == 0:
            record(a.indices, sv, k, rho, "c3_identity")  # S == K
            record(a.indices, sv, s, 0.0, "c3_rho0")
            record(a.indices, sv, s, 1.0, "c3_rho1")

    # ties + exact-threshold cases (Appendix A items 3/4)
    v = np.full((6, 6), 0.5)
    np.fill_diagonal(v, 1.0)
    record(np.array([[0, 3], [1, 4], [2, 5]]), v, 1, 0.5, "ties_eq_rho")
    record(np.array([[0, 3], [1, 4], [2, 5]]), v, 1, 0.6, "ties_above_rho")
    q = np.round(_sym(np.random.default_rng(7), 10) * 4) / 4  # many exact ties
    np.fill_diagonal(q, 1.0)
    rng = np.random.default_rng(8)
    for _ in range(20):
        a = _assign(rng, 6, 4, 10)
        for rho in (0.25, 0.5, 0.75):
            record(a.indices, q, 1, rho, "quantised_ties")
            record(a.indices, q, 2, rho, "quantised_ties")

    # BASELINE shapes (sims by seed): C0 toy, C1 Mixtral, C2 Qwen3, C3 DSV2-Lite, C4 Qwen3 T=512
    shapes = [(8, 2, 16), (8, 2, 64), (8, 2, 256), (128, 8, 128), (64, 6, 256), (128, 8, 512)]
    for j, (m, k, t) in enumerate(shapes):
        for beta in (0.0, 2.0):
            seed = 1000 + 10 * j + int(beta)
            rng = np.random.default_rng(seed)
            logits = rng.standard_normal((t, m)) + beta * rng.standard_normal(m)[None, :]
            idx = np.argsort(-logits, axis=1, kind="stable")[:, :k]
            sv = _sym(np.random.default_rng(seed + 5000), m)
            for s in (1, 2):
                for rho in (0.0, 0.5, 0.9, 0.95, 1.0):
                    record(idx, sv, s, rho, f"shape_m{m}_k{k}_t{t}", sim_seed=seed + 5000)

    out = {}
    ids_in.dump("ids_in", out)
    ids_out.dump("ids_out", out)
    sims.dump("sim", out)
    out["retain"] = np.array([m[0] for m in meta], dtype=np.int64)
    out["rho"] = np.array([m[1] for m in meta], dtype=np.float64)
    out["sim_seed"] = np.array([m[2] for m in meta], dtype=np.int64)
    out["m"] = np.array([m[3] for m in meta], dtype=np.int64)
    out["source"] = np.array([m[4] for m in meta])
    out["sets_json"] = np.array(json.dumps(sets))
    np.savez_compressed(HERE / "reroute_cases.npz", **out)
    print(f"reroute_cases: {len(meta)} instances")


def calib_cases():
    out = {}
    seed, L, M, K, d_h, d_m = 21, 2, 8, 2, 64, 96
    model = moe.gen_model(seed=seed, n_layers=L, n_experts=M, top_k=K, d_h=d_h, d_m=d_m)
    batches = similarity.gaussian_batches(5, 2, 16, d_h)
    out["config"] = np.array([seed, L, M, K, d_h, d_m, 5, 2, 16], dtype=np.int64)
    for metric in ("frobenius", "cosine"):
        raw = similarity.estimate_similarity_raw(model, batches, metric)
        sims = similarity.estimate_similarity(model, batches, metric)
        out[f"{metric}_raw"] = np.stack(raw)
        out[f"{metric}_sim"] = np.stack([s.values for s in sims])
    np.savez_compressed(HERE / "calib_cases.npz", **out)
    print("calib_cases: frobenius, cosine")


def layer_cases():
    out = {}
    rows = []
    configs = [
        # name, seed, L, M, K, d_h, d_m, n_shared, T, act, S, rho
        ("c0_toy", 0, 1, 8, 2, 256, 512, 0, 16, "silu", 1, 0.5),
        ("small_shared", 3, 2, 6, 3, 32, 64, 2, 9, "silu", 1, 0.0),
        ("relu", 4, 1, 4, 2, 16, 48, 0, 5, "relu", 1, 0.3),
        ("gelu", 5, 1, 5, 2, 24, 40, 1, 7, "gelu-tanh", 1, 0.3),
        ("multi", 6, 3, 8, 4, 64, 128, 0, 12, "silu", 2, 0.4),
    ]
    for name, seed, L, M, K, d_h, d_m, n_sh, T, act, S, rho in configs:
        model = moe.gen_model(seed=seed, n_layers=L, n_experts=M, top_k=K, d_h=d_h, d_m=d_m,
                              n_shared=n_sh, activation=act)
        rng = np.random.default_rng([seed, 77])
        x = rng.standard_normal((T, d_h))
        sims = [similarity.SimilarityMatrix(values=_sym(rng, M), metric="cosine") for _ in range(L)]
        cfg = rerouting.RerouteConfig(retain_count=S, threshold=rho)
        plain = moe.model_forward(model, moe.TokenBatch(x, "decode"))
        sere = moe.model_forward(model, moe.TokenBatch(x, "decode"), config=cfg, sims=sims)
        out[f"{name}_x"] = x
        out[f"{name}_sims"] = np.stack([s.values for s in sims])
        out[f"{name}_plain_y"] = plain.output
        out[f"{name}_sere_y"] = sere.output
        out[f"{name}_plain_ids"] = np.stack([tr.original.indices for tr in plain.layers])
        out[f"{name}_plain_w"] = np.stack([tr.original.weights for tr in plain.layers])
        out[f"{name}_sere_ids"] = np.stack([tr.final.indices for tr in sere.layers])
        # single-layer layer_forward on layer 0 with the plain routing
        lay = model.layers[0]
        a0 = plain.layers[0].original
        out[f"{name}_layer0_y"] = moe.layer_forward(lay, x, a0, act)
        rows.append(dict(name=name, seed=seed, L=L, M=M, K=K, d_h=d_h, d_m=d_m, n_shared=n_sh,
                         T=T, act=act, S=S, rho=rho))
    out["configs_json"] = np.array(json.dumps(rows))
    np.savez_compressed(HERE / "layer_cases.npz", **out)
    print(f"layer_cases: {len(rows)} configs")


def topk_cases():
    out = {}
    rng = np.random.default_rng(11)
    logits = [rng.standard_normal((7, 9)), np.round(rng.standard_normal((6, 8)) * 2) / 2,
              np.zeros((3, 5)), np.array([[1.0, 3.0, 3.0, 2.0, 3.0]])]
    for i, lg in enumerate(logits):
        for k in (1, 2, lg.shape[1]):
            a = moe.topk_softmax(lg, k)
            out[f"l{i}_k{k}_logits"] = lg
            out[f"l{i}_k{k}_ids"] = a.indices
            out[f"l{i}_k{k}_w"] = a.weights
    np.savez_compressed(HERE / "topk_cases.npz", **out)
    print(f"topk_cases: {len(out) // 3} cases")


if __name__ == "__main__":
    reroute_cases()
    layer_cases()
    calib_cases()
    topk_cases()
