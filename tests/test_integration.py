"""Drop-in integration: patch a module namespace shaped like the
reference's `sere.rerouting` / `sere.moe` and drive it the way moe.model_forward does
(module-attribute lookup at moe.py:368 and moe.py:375)."""

import types
from dataclasses import dataclass

import numpy as np
import pytest

from oracle import sere_oracle as O


@dataclass(frozen=True)
class RefRerouteResult:  # field set of rerouting.py:57-65
    new_indices: np.ndarray
    primary_set: frozenset
    preserved_critical: frozenset
    final_active: frozenset
    reroute_map: dict


def _oracle_apply_sere(assignment, sim, config):
    r = O.apply_sere(np.asarray(assignment.indices), np.asarray(getattr(sim, "values", sim)),
                     config.retain_count, config.threshold)
    return RefRerouteResult(r.new_indices, r.primary_set, r.preserved_critical, r.final_active, r.reroute_map)


def _fake_reference():
    rr = types.ModuleType("sere_fake.rerouting")
    rr.RerouteResult = RefRerouteResult
    rr.apply_sere = _oracle_apply_sere
    moe = types.ModuleType("sere_fake.moe")
    moe.rerouting = rr

    def layer_forward(layer, x, assignment, activation="silu"):
        return O.layer_forward(layer, x, np.asarray(assignment.indices), np.asarray(assignment.weights), activation)

    moe.layer_forward = layer_forward

    def model_layer(layer, x, assignment, sim, config):  # moe.py:367-375, same lookups
        result = moe.rerouting.apply_sere(assignment, sim, config)
        final = types.SimpleNamespace(indices=result.new_indices, weights=assignment.weights)
        return result, moe.layer_forward(layer, x, final, "silu")

    moe.model_layer = model_layer
    return rr, moe


def test_install_uninstall_restores_attributes():
    from paper_2602_07616_b200 import integration

    rr, moe = _fake_reference()
    orig_a, orig_l = rr.apply_sere, moe.layer_forward
    h = integration.install(rr, moe)
    assert rr.apply_sere is not orig_a and moe.layer_forward is not orig_l
    h.uninstall()
    assert rr.apply_sere is orig_a and moe.layer_forward is orig_l


@pytest.mark.gpu
def test_patched_reference_runs_on_gpu(cuda_device):
    import torch

    from paper_2602_07616_b200 import integration

    M, K, d_h, d_m, T = 8, 2, 256, 512, 16
    layer = O.gen_layers(3, 1, M, K, d_h, d_m, 1)[0]
    rnd = lambda a: torch.as_tensor(a, dtype=torch.float32).to(torch.bfloat16).double().numpy()
    layer = O.OracleLayer([O.OracleExpert(rnd(e.w_gate), rnd(e.w_up), rnd(e.w_down)) for e in layer.experts],
                          layer.w_router, K,
                          [O.OracleExpert(rnd(e.w_gate), rnd(e.w_up), rnd(e.w_down)) for e in layer.shared_experts])
    rng = np.random.default_rng(7)
    x = rnd(rng.standard_normal((T, d_h)))
    ids, w = O.route_topk(layer.w_router, K, x)
    sim = types.SimpleNamespace(values=O.random_symmetric_sim(rng, M))
    cfg = types.SimpleNamespace(retain_count=1, threshold=0.5, phase_mode="all_phases")
    a = types.SimpleNamespace(indices=ids, weights=w)

    rr, moe = _fake_reference()
    want_res, want_y = moe.model_layer(layer, x, a, sim, cfg)
    h = integration.install(rr, moe)
    try:
        got_res, got_y = moe.model_layer(layer, x, a, sim, cfg)
    finally:
        h.uninstall()
    assert isinstance(got_res, RefRerouteResult)
    assert (got_res.primary_set, got_res.preserved_critical, got_res.final_active, got_res.reroute_map) == \
        (want_res.primary_set, want_res.preserved_critical, want_res.final_active, want_res.reroute_map)
    np.testing.assert_array_equal(got_res.new_indices, want_res.new_indices)
    err = float(np.abs(got_y - want_y).max())
    assert err <= 1e-2 * max(1.0, float(np.abs(want_y).max()))
    cos = float((got_y * want_y).sum() / np.linalg.norm(got_y) / np.linalg.norm(want_y))
    assert cos >= 0.9999
