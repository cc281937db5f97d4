"""Pin the CPU oracle to the real reference's outputs (golden vectors), CPU only."""

import numpy as np
import pytest

from oracle import sere_oracle as O
from paper_2602_07616_b200.errors import ConfigError, DimensionError, InputError, RoutingError


def test_oracle_reroute_matches_reference_goldens(reroute_goldens):
    sources = set()
    for c in reroute_goldens:
        res = O.apply_sere(c["ids_in"], c["sim"], c["retain"], c["rho"])
        assert res.new_indices.tobytes() == c["ids_out"].astype(np.int64).tobytes(), c["source"]
        assert res.primary_set == c["primary"]
        assert res.preserved_critical == c["critical"]
        assert res.final_active == c["active"]
        assert res.reroute_map == c["map"]
        sources.add(c["source"].split("_")[0])
    # every family of golden vectors was exercised
    assert {"fig1", "trace0", "trace1", "c3", "shape", "ties", "quantised"} <= sources


def test_fig1_known_answer(reroute_goldens):
    c = next(c for c in reroute_goldens if c["source"] == "fig1" and c["retain"] == 1 and c["rho"] == 0.5)
    assert c["primary"] == {1, 4} and c["critical"] == {3} and c["map"] == {2: 1}
    np.testing.assert_array_equal(c["ids_out"], [[1, 1], [4, 1], [1, 3], [4, 3]])


def test_set_algebra_oracle_agrees(reroute_goldens):
    for c in reroute_goldens:
        if c["retain"] >= c["ids_in"].shape[1]:
            continue
        new, primary, preserved, mapping = O.apply_sere_set_algebra(c["ids_in"], c["sim"], c["retain"], c["rho"])
        np.testing.assert_array_equal(new, c["ids_out"])
        assert primary == c["primary"] and preserved == c["critical"] and mapping == c["map"]


def test_oracle_layer_and_model_forward_bit_identical(layer_goldens):
    z, configs = layer_goldens
    for c in configs:
        n = c["name"]
        layers = O.gen_layers(c["seed"], c["L"], c["M"], c["K"], c["d_h"], c["d_m"], c["n_shared"])
        x = z[f"{n}_x"]
        y, tr = O.model_forward(layers, x, c["act"])
        assert y.tobytes() == z[f"{n}_plain_y"].tobytes(), n
        sims = list(z[f"{n}_sims"])
        ys, trs = O.model_forward(layers, x, c["act"], retain_count=c["S"], threshold=c["rho"], sims=sims)
        assert ys.tobytes() == z[f"{n}_sere_y"].tobytes(), n
        for l in range(c["L"]):
            np.testing.assert_array_equal(trs[l]["final"], z[f"{n}_sere_ids"][l])
            np.testing.assert_array_equal(tr[l]["original"], z[f"{n}_plain_ids"][l])
        y0 = O.layer_forward(layers[0], x, tr[0]["original"], tr[0]["weights"], c["act"])
        assert y0.tobytes() == z[f"{n}_layer0_y"].tobytes()


def test_oracle_topk_softmax():
    from conftest import GOLDEN

    z = np.load(GOLDEN / "topk_cases.npz")
    keys = sorted({k.rsplit("_", 1)[0] for k in z.files})
    assert keys
    for key in keys:
        k = int(key.split("_k")[1])
        ids, w = O.topk_softmax(z[key + "_logits"], k)
        np.testing.assert_array_equal(ids, z[key + "_ids"])
        assert w.tobytes() == z[key + "_w"].tobytes()


def test_frozen_expert_value():
    # reference tests/test_moe.py:44-54 frozen straight-line value (atol 1e-15)
    e = O.OracleExpert(
        w_gate=np.array([[0.1257, -0.1321], [0.6404, 0.1049]]),
        w_up=np.array([[-0.5357, 0.3616], [1.304, 0.9471]]),
        w_down=np.array([[-0.7037, -1.2654], [-0.6233, 0.0413]]),
    )
    y = O.expert_forward(e, np.array([[-2.325, -0.2188]]), "silu")
    np.testing.assert_allclose(y, [[0.22088790489460558, 0.19973560809728075]], rtol=0, atol=1e-15)


def test_oracle_error_contract():
    rng = np.random.default_rng(0)
    ids, _ = O.random_assignment(rng, 4, 2, 6)
    sim = O.random_symmetric_sim(rng, 6)
    with pytest.raises(ConfigError):
        O.apply_sere(ids, sim, 3, 0.3)  # S > K (rerouting.py:104-107)
    with pytest.raises(DimensionError):
        O.apply_sere(ids, O.random_symmetric_sim(rng, 3), 1, 0.5)
    with pytest.raises(InputError):
        O.apply_sere(ids, np.full((6, 6), 1.5), 1, 0.5)
    with pytest.raises(ConfigError):
        O.apply_sere(ids, sim, 0, 0.5)
    with pytest.raises(ConfigError):
        O.apply_sere(ids, sim, 1, 1.5)
    layer = O.gen_layers(0, 1, 4, 2, 8, 16)[0]
    with pytest.raises(RoutingError):
        O.layer_forward(layer, np.zeros((1, 8)), [[0, 4]], [[0.5, 0.5]])


def test_nan_quirk_matches_reference_semantics():
    # Appendix A item 8: NaN passes validation; all-NaN candidates -> critical at rho>0, -1 at rho=0
    sim = np.full((4, 4), np.nan)
    np.fill_diagonal(sim, 1.0)
    ids = np.array([[0, 2], [1, 3]])
    r = O.apply_sere(ids, sim, 1, 0.5)
    assert r.preserved_critical == {2, 3}
    r0 = O.apply_sere(ids, sim, 1, 0.0)
    np.testing.assert_array_equal(r0.new_indices, [[0, -1], [1, -1]])
    assert r0.reroute_map == {2: -1, 3: -1}


def test_bf16_round_matches_torch():
    """oracle.bf16_round (nearest-even via float32) equals torch's bfloat16 conversion."""
    import torch

    rng = np.random.default_rng(0)
    a = np.concatenate([rng.standard_normal(100000) * s for s in (1e-3, 1.0, 37.0)])
    a = np.concatenate([a, [0.0, -0.0, 1.0, 1.00390625, 1.0078125 + 2 ** -9, 65504.0]])
    want = torch.as_tensor(a.astype(np.float32)).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(O.bf16_round(a), want)


def test_block_forward_reduces_to_layer_chain():
    """oracle.block_forward is the residual chain x += layer_forward(bf16(RMSNorm(x))) with the
    given routes; S == K leaves the ids untouched."""
    layers = O.gen_layers(1, 2, 8, 2, 16, 24, 1)
    rng = np.random.default_rng(2)
    x0 = rng.standard_normal((6, 16))
    routes = [O.route_topk(l.w_router, 2, x0) for l in layers]
    sims = [O.random_symmetric_sim(rng, 8) for _ in layers]
    x, tr = O.block_forward(layers, x0, sims, 2, 0.5, routes)
    want = x0.copy()
    for l, layer in enumerate(layers):
        h = O.bf16_round(O.rms_norm(want))
        np.testing.assert_array_equal(tr[l]["final"], routes[l][0])
        want = want + O.layer_forward(layer, h, routes[l][0], routes[l][1])
    np.testing.assert_array_equal(x, want)
