"""Re-routing kernel parity: bit-exact against the reference (goldens) and the oracle."""

import types

import numpy as np
import pytest

from oracle import sere_oracle as O

pytestmark = pytest.mark.gpu


def _dev_reroute(ids, sim, s, rho):
    import torch

    from paper_2602_07616_b200 import rerouting

    t = torch.as_tensor(np.asarray(ids, dtype=np.int32)).cuda()
    return rerouting.reroute(t, np.asarray(sim, dtype=np.float64), s, rho).to_result()


def _assert_same(res, want_ids, primary, critical, active, mapping, tag=""):
    assert res.new_indices.astype(np.int64).tobytes() == np.asarray(want_ids, dtype=np.int64).tobytes(), tag
    assert res.primary_set == primary, tag
    assert res.preserved_critical == critical, tag
    assert res.final_active == active, tag
    assert res.reroute_map == mapping, tag


def test_goldens_bit_exact(cuda_device, reroute_goldens):
    """Every golden vector recorded from the real reference (Fig. 1, CLI trace, C3 sweep,
    quantised ties, BASELINE shapes x rho grid x S)."""
    n = 0
    for c in reroute_goldens:
        res = _dev_reroute(c["ids_in"], c["sim"], c["retain"], c["rho"])
        _assert_same(res, c["ids_out"], c["primary"], c["critical"], c["active"], c["map"], c["source"])
        n += 1
    assert n == reroute_goldens.n


def test_fig1_through_dropin_api(cuda_device):
    from paper_2602_07616_b200 import rerouting

    a = types.SimpleNamespace(indices=np.array([[1, 2], [4, 2], [1, 3], [4, 3]]),
                              weights=np.array([[0.6, 0.4], [0.7, 0.3], [0.55, 0.45], [0.65, 0.35]]))
    v = np.array([[1.0, 0.0, 0.0, 0.0, 0.0], [0.0, 1.0, 0.9, 0.2, 0.4], [0.0, 0.9, 1.0, 0.35, 0.3],
                  [0.0, 0.2, 0.35, 1.0, 0.25], [0.0, 0.4, 0.3, 0.25, 1.0]])
    sim = types.SimpleNamespace(values=v)
    res = rerouting.apply_sere(a, sim, rerouting.RerouteConfig(retain_count=1, threshold=0.5))
    assert res.primary_set == {1, 4} and res.preserved_critical == {3} and res.final_active == {1, 3, 4}
    assert res.reroute_map == {2: 1}
    np.testing.assert_array_equal(res.new_indices, [[1, 1], [4, 1], [1, 3], [4, 3]])
    np.testing.assert_array_equal(a.weights[0], [0.6, 0.4])  # weights untouched


def test_c3_style_sweep_vs_oracle(cuda_device):
    """tests/test_acceptance.py:93-115 generator, 1000 instances (different seeds from the goldens)."""
    for i in range(1000):
        rng = np.random.default_rng([900, i])
        m = int(rng.integers(6, 13))
        k = int(rng.integers(2, 5))
        t = int(rng.integers(1, 9))
        s = int(rng.integers(1, k + 1))
        ids, _ = O.random_assignment(rng, t, k, m)
        sim = O.random_symmetric_sim(rng, m)
        rho = float(rng.random())
        want = O.apply_sere(ids, sim, s, rho)
        res = _dev_reroute(ids, sim, s, rho)
        _assert_same(res, want.new_indices, want.primary_set, want.preserved_critical, want.final_active,
                     want.reroute_map, f"i={i}")


@pytest.mark.parametrize("m,k,t", [(8, 2, 256), (128, 8, 128), (64, 6, 256), (128, 8, 512), (256, 8, 2048)])
def test_baseline_shapes_vs_oracle(cuda_device, m, k, t):
    for beta in (0.0, 1.0, 2.0):
        rng = np.random.default_rng([m, k, t, int(beta)])
        logits = rng.standard_normal((t, m)) + beta * rng.standard_normal(m)[None, :]
        ids = np.argsort(-logits, axis=1, kind="stable")[:, :k]
        for kind in ("uniform", "quantised"):
            sim = O.random_symmetric_sim(rng, m)
            if kind == "quantised":  # exact ties everywhere: lowest-index rule decides
                sim = np.round(sim * 8) / 8
                np.fill_diagonal(sim, 1.0)
            for s in (1, 2, k):
                for rho in (0.0, 0.3, 0.7, 0.9, 0.97, 1.0):
                    want = O.apply_sere(ids, sim, s, rho)
                    res = _dev_reroute(ids, sim, s, rho)
                    _assert_same(res, want.new_indices, want.primary_set, want.preserved_critical,
                                 want.final_active, want.reroute_map, f"{kind} S={s} rho={rho}")


def test_threshold_equal_reroutes_and_fp64_compare(cuda_device):
    # s* == rho re-routes (strict <); fp64 compare: fp32(0.7) < 0.7 must stay critical
    v = np.full((4, 4), 0.5)
    np.fill_diagonal(v, 1.0)
    res = _dev_reroute([[0, 2], [1, 3]], v, 1, 0.5)
    assert res.reroute_map == {2: 0, 3: 0}
    v2 = np.full((4, 4), float(np.float32(0.7)))
    np.fill_diagonal(v2, 1.0)
    res = _dev_reroute([[0, 2], [1, 3]], v2, 1, 0.7)
    assert res.preserved_critical == {2, 3} and res.reroute_map == {}


def test_nan_quirk(cuda_device):
    sim = np.full((4, 4), np.nan)
    np.fill_diagonal(sim, 1.0)
    r = _dev_reroute([[0, 2], [1, 3]], sim, 1, 0.5)
    assert r.preserved_critical == {2, 3}
    r0 = _dev_reroute([[0, 2], [1, 3]], sim, 1, 0.0)
    np.testing.assert_array_equal(r0.new_indices, [[0, -1], [1, -1]])
    assert r0.reroute_map == {2: -1, 3: -1}


def test_error_contract(cuda_device):
    from paper_2602_07616_b200 import rerouting
    from paper_2602_07616_b200.errors import ConfigError, DimensionError, InputError

    rng = np.random.default_rng(1)
    ids, _ = O.random_assignment(rng, 4, 2, 6)
    sim = O.random_symmetric_sim(rng, 6)
    a = types.SimpleNamespace(indices=ids)
    with pytest.raises(ConfigError):
        rerouting.apply_sere(a, sim, rerouting.RerouteConfig(retain_count=3, threshold=0.3))
    with pytest.raises(DimensionError):
        rerouting.apply_sere(a, O.random_symmetric_sim(rng, 3), rerouting.RerouteConfig(1, 0.5))
    with pytest.raises(InputError):
        rerouting.apply_sere(a, np.full((6, 6), 1.5), rerouting.RerouteConfig(1, 0.5))
    with pytest.raises(DimensionError):
        rerouting.apply_sere(types.SimpleNamespace(indices=np.array([[0, 9]])), sim, rerouting.RerouteConfig(1, 0.5))
    with pytest.raises(ConfigError):
        rerouting.RerouteConfig(retain_count=0, threshold=0.5)
    with pytest.raises(ConfigError):
        rerouting.RerouteConfig(retain_count=1, threshold=1.5)


def test_deterministic_and_idempotent(cuda_device):
    rng = np.random.default_rng(5)
    logits = rng.standard_normal((512, 128)) + 2 * rng.standard_normal(128)[None, :]
    ids = np.argsort(-logits, axis=1, kind="stable")[:, :8]
    sim = O.random_symmetric_sim(rng, 128)
    a = _dev_reroute(ids, sim, 1, 0.9)
    b = _dev_reroute(ids, sim, 1, 0.9)
    assert a.new_indices.tobytes() == b.new_indices.tobytes()
    again = _dev_reroute(a.new_indices, sim, 1, 0.9)  # rewrite is idempotent (test_rerouting.py:161-171)
    np.testing.assert_array_equal(again.new_indices, a.new_indices)
    assert again.reroute_map == {} and again.final_active == a.final_active


def test_empty_batch(cuda_device):
    res = _dev_reroute(np.zeros((0, 2), dtype=np.int64), O.random_symmetric_sim(np.random.default_rng(0), 4), 1, 0.5)
    assert res.new_indices.shape == (0, 2) and res.final_active == frozenset()
