"""Reference file formats (moe.py:428-512, similarity.py:438-487) on the GPU path."""

import json
import pathlib
import sys

import numpy as np
import pytest

from oracle import sere_oracle as O

REF = pathlib.Path("/root/reference/pkg/src")


def _write_reference_layout(directory, layers, d_h, d_m, activation="silu", seed=7):
    """The byte layout of the reference's save_model (moe.py:440-473)."""
    directory.mkdir(parents=True, exist_ok=True)
    first = layers[0]
    meta = {"seed": seed, "n_layers": len(layers), "n_experts": len(first.experts), "top_k": first.top_k,
            "d_h": d_h, "d_m": d_m, "n_shared": len(first.shared_experts), "activation": activation}
    (directory / "model.json").write_text(json.dumps(meta, indent=2) + "\n")
    w = lambda p, a: (directory / p).write_bytes(np.ascontiguousarray(a, dtype="<f4").tobytes())
    for l, layer in enumerate(layers):
        for j, e in enumerate(layer.experts):
            w(f"layer{l}.expert{j}.gate.f32", e.w_gate)
            w(f"layer{l}.expert{j}.up.f32", e.w_up)
            w(f"layer{l}.expert{j}.down.f32", e.w_down)
        for j, e in enumerate(layer.shared_experts):
            w(f"layer{l}.shared{j}.gate.f32", e.w_gate)
            w(f"layer{l}.shared{j}.up.f32", e.w_up)
            w(f"layer{l}.shared{j}.down.f32", e.w_down)
        w(f"layer{l}.router.f32", layer.w_router)


@pytest.mark.skipif(not REF.is_dir(), reason="reference package not present (GPU box)")
def test_product_writer_matches_reference_save_model(tmp_path):
    """io.save_model's writer (io.write_model_dir + io.model_meta, the code save_model runs after
    unpacking the banks) produces files byte-identical to the reference's save_model."""
    from paper_2602_07616_b200 import io

    sys.path.insert(0, str(REF))
    try:
        from sere import moe as ref_moe
    finally:
        sys.path.remove(str(REF))
    model = ref_moe.gen_model(seed=3, n_layers=2, n_experts=4, top_k=2, d_h=16, d_m=24, n_shared=1)
    ref_moe.save_model(model, tmp_path / "ref")
    first = model.layers[0]
    meta = io.model_meta(model.seed, model.n_layers, first.n_experts, first.router.top_k, model.d_h,
                         first.experts[0].d_m, len(first.shared_experts), model.activation)
    host = [(np.stack([e.w_gate for e in L.experts + L.shared_experts]),
             np.stack([e.w_up for e in L.experts + L.shared_experts]),
             np.stack([e.w_down for e in L.experts + L.shared_experts]), L.router.w_router)
            for L in model.layers]
    io.write_model_dir(tmp_path / "ours", meta, host)
    ref_files = sorted(p.name for p in (tmp_path / "ref").iterdir())
    assert ref_files == sorted(p.name for p in (tmp_path / "ours").iterdir())
    for name in ref_files:
        assert (tmp_path / "ref" / name).read_bytes() == (tmp_path / "ours" / name).read_bytes(), name


@pytest.mark.skipif(not REF.is_dir(), reason="reference package not present (GPU box)")
def test_writer_matches_reference_save_model(tmp_path):
    """The tests' own layout helper (used by the GPU tests on the box, where the reference is
    absent) writes byte-identical files to the reference save_model."""
    sys.path.insert(0, str(REF))
    try:
        from sere import moe as ref_moe
    finally:
        sys.path.remove(str(REF))
    model = ref_moe.gen_model(seed=3, n_layers=2, n_experts=4, top_k=2, d_h=16, d_m=24, n_shared=1)
    ref_moe.save_model(model, tmp_path / "ref")
    layers = [O.OracleLayer([O.OracleExpert(e.w_gate, e.w_up, e.w_down) for e in L.experts], L.router.w_router,
                            L.router.top_k, [O.OracleExpert(e.w_gate, e.w_up, e.w_down) for e in L.shared_experts])
              for L in model.layers]
    _write_reference_layout(tmp_path / "ours", layers, 16, 24, model.activation, model.seed)
    ref_files = sorted(p.name for p in (tmp_path / "ref").iterdir())
    assert ref_files == sorted(p.name for p in (tmp_path / "ours").iterdir())
    for name in ref_files:
        assert (tmp_path / "ref" / name).read_bytes() == (tmp_path / "ours" / name).read_bytes(), name


def test_similarity_json_round_trip_and_validation(tmp_path):
    from paper_2602_07616_b200 import io
    from paper_2602_07616_b200.errors import DomainError, InputError

    v = O.random_symmetric_sim(np.random.default_rng(0), 6)
    io.save_similarity(v, tmp_path, layer_index=1)
    np.testing.assert_array_equal(io.load_similarity(tmp_path / "sim.layer1.json"), v)
    assert (tmp_path / "sim.layer1.f32").stat().st_size == 6 * 6 * 4
    with pytest.raises(InputError):
        io.load_similarity_set(tmp_path, 2)  # layer 0 missing
    bad = v.copy()
    bad[0, 1] = 0.3
    with pytest.raises(DomainError):
        io.save_similarity(bad, tmp_path / "x")


@pytest.mark.gpu
def test_reference_model_dir_runs_on_gpu(cuda_device, tmp_path):
    """A reference-format model directory loads into GPU banks; model_forward with the SERE
    rewrite (sims from sim.layer{l}.json) matches the oracle on the same bf16 values, and
    save_model round-trips the banks."""
    import torch

    from paper_2602_07616_b200 import io, moe, rerouting

    rnd = lambda a: torch.as_tensor(np.asarray(a, np.float32)).to(torch.bfloat16).double().numpy()
    L, M, K, d_h, d_m, ns, T = 2, 8, 2, 128, 256, 1, 24
    raw = O.gen_layers(11, L, M, K, d_h, d_m, ns)
    layers = [O.OracleLayer([O.OracleExpert(rnd(e.w_gate), rnd(e.w_up), rnd(e.w_down)) for e in lay.experts],
                            rnd(lay.w_router), K,
                            [O.OracleExpert(rnd(e.w_gate), rnd(e.w_up), rnd(e.w_down)) for e in lay.shared_experts])
              for lay in raw]
    _write_reference_layout(tmp_path / "m", layers, d_h, d_m)
    rng = np.random.default_rng(5)
    for l in range(L):
        io.save_similarity(O.random_symmetric_sim(rng, M), tmp_path / "m", layer_index=l)
    model = io.load_model(tmp_path / "m")
    sims = io.load_similarity_set(tmp_path / "m", L)
    x = rnd(np.random.default_rng(6).standard_normal((T, d_h)))
    # teacher-forced routing (the oracle's fp64 top-k on the GPU layer input, recorded so the
    # oracle chain below uses the very same assignment): ids after SERE then match exactly
    routed = []

    def override(l, xin):
        ids, w = O.route_topk(layers[l].w_router, K, xin)
        routed.append((ids, w, np.asarray(xin, dtype=np.float64)))
        return type("A", (), {"indices": ids, "weights": w})()

    cfg = rerouting.RerouteConfig(1, 0.5)
    batch = type("B", (), {"x": x, "phase": "decode"})
    got = moe.model_forward(model, batch, cfg, sims, router_override=override)
    # every layer's input is teacher-forced from the device chain (the override sees the
    # previous layer's fp32 output; the layer computes on its bf16 rounding), so each layer's
    # output is held to the absolute bar on its own
    from conftest import check_close

    for l in range(L):
        ids, w, xin = routed[l]
        res = O.apply_sere(ids, sims[l], 1, 0.5)
        np.testing.assert_array_equal(got.layers[l].final.indices, res.new_indices)
        y_ref = O.layer_forward(layers[l], rnd(xin), res.new_indices, w)
        y_dev = routed[l + 1][2] if l + 1 < L else got.output
        # the raw reference chain (x <- MoE(x), gen_model weights) grows to |y| ~ 7.5 by layer 1;
        # Appendix B's ideal bf16 kernel reaches 6.9e-3 at |y| ~ 4, so beyond |y| = 4 the bar
        # keeps that relative accuracy (stated here, not in the shared helper: every BASELINE
        # shape is held to the plain absolute 1e-2)
        atol = 1e-2 * max(1.0, float(np.abs(y_ref).max()) / 4.0)
        check_close(y_dev, y_ref, f"reference-format model dir, layer {l} output", atol=atol)
    io.save_model(model, tmp_path / "back")
    again = io.load_model(tmp_path / "back")
    for a, b in zip(model.layers, again.layers):
        assert torch.equal(a.bank.data, b.bank.data)  # zero-initialised banks: padding tiles agree too
        for ta, tb in zip(a.bank.unpack(), b.bank.unpack()):
            assert torch.equal(ta, tb)
        assert torch.equal(a.router.w_router, b.router.w_router)
