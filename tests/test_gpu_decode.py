"""Multi-layer decode step, router kernel, CUDA-graph replay and expert-parallel shards on one GPU."""

import os
import socket

import numpy as np
import pytest

from oracle import sere_oracle as O

pytestmark = pytest.mark.gpu


def _bf16(a):
    import torch

    return torch.as_tensor(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def test_router_matches_fp64_topk_on_same_inputs(cuda_device):
    """moe.py:248-277: ids identical to the fp64 stable top-k wherever the K-th/K+1-th logit gap
    exceeds the fp32 accumulation error; softmax weights within 1e-5."""
    import torch

    from paper_2602_07616_b200.moe import route_topk_device, router_weight_t

    for (T, d_h, M, K) in [(512, 2048, 128, 8), (256, 4096, 8, 2), (256, 2048, 64, 6), (7, 24, 5, 2)]:
        g = torch.Generator(device="cuda")
        g.manual_seed(T + M)
        x = torch.randn(T, d_h, device="cuda", generator=g).to(torch.bfloat16)
        w = (torch.randn(d_h, M, device="cuda", generator=g) / d_h ** 0.5).to(torch.bfloat16)
        bias = torch.randn(M, device="cuda", generator=g)
        ids, wts, lg = route_topk_device(router_weight_t(w), x, K, logits=True, bias=bias)
        logits64 = x.double().cpu().numpy() @ w.double().cpu().numpy() + bias.double().cpu().numpy()[None, :]
        np.testing.assert_allclose(lg.double().cpu().numpy(), logits64, atol=2e-4, rtol=1e-4)
        ref_ids, ref_w = O.topk_softmax(logits64, K)
        srt = -np.sort(-logits64, axis=1)
        gap = srt[:, K - 1] - srt[:, K] if K < M else np.full(T, np.inf)
        safe = gap > 1e-3
        got = ids.cpu().numpy()
        np.testing.assert_array_equal(got[safe], ref_ids[safe])
        np.testing.assert_allclose(wts.double().cpu().numpy()[safe], ref_w[safe], atol=1e-5)
        assert safe.mean() > 0.9
        # rows with a near-tie at the K-th logit: the device may pick either side of the tie, but
        # every id it picks must be within the fp32 accumulation error of the fp64 top-K
        picked = np.take_along_axis(logits64, got.astype(np.int64), axis=1)
        assert np.all(picked >= srt[:, K - 1:K] - 1e-3)
        assert np.all([len(set(r)) == K for r in got])


def test_decode_plain_chain_vs_oracle(cuda_device):
    """block='plain' is the reference model_forward chain (x <- MoE(x)). Every layer's router
    ids/weights are teacher-forced from the device router into the oracle (router_override,
    moe.py:334,363-364): ids after SERE bit-exact on EVERY layer, output within the absolute bar."""
    import torch

    from conftest import check_close
    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

    L, M, K, d_h, d_m, T = 3, 16, 4, 256, 128, 24
    model = DecodeModel(L, M, K, d_h, d_m, n_shared=1, seed=3, beta=0.0, keep_raw_layer=None)
    step = DecodeStep(model, T, retain_count=1, threshold=0.6, block="plain")
    x0 = torch.randn(T, d_h, device="cuda")
    routes = []
    step._trace_hook = lambda l: routes.append((step.ids.cpu().numpy().astype(np.int64),
                                                step.w.double().cpu().numpy(), step.h.double().cpu().numpy()))
    step.set_input(x0)
    step.run()
    torch.cuda.synchronize()
    step.check()
    x = _bf16(x0.cpu().numpy())
    for l, layer in enumerate(model.layers):
        wg, wu, wd = [t.double().cpu().numpy() for t in layer.bank.unpack()]
        ol = O.OracleLayer([O.OracleExpert(wg[e], wu[e], wd[e]) for e in range(M)], None, K,
                           [O.OracleExpert(wg[M], wu[M], wd[M])])
        ids, w, h_gpu = routes[l]
        res = O.apply_sere(ids, model.sims_host[l], 1, 0.6)
        np.testing.assert_array_equal(step.outs[l].reroute.new_indices.cpu().numpy(), res.new_indices)
        y = O.layer_forward(ol, x, res.new_indices, w)
        got = step.outs[l].y.double().cpu().numpy()
        check_close(got, y, f"plain chain layer {l}")
        x = _bf16(got)  # the chain feeds bf16(y) forward, as the device does
        if l + 1 < L:
            np.testing.assert_array_equal(routes[l + 1][2], x)


def test_graph_replay_bit_identical_to_eager(cuda_device):
    import torch

    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

    model = DecodeModel(4, 32, 4, 512, 256, seed=1, beta=1.0)
    eager = DecodeStep(model, 64, 1, 0.5)
    graphed = DecodeStep(model, 64, 1, 0.5)
    x0 = torch.randn(64, 512, device="cuda")
    eager.set_input(x0)
    graphed.set_input(x0)
    eager.run()
    graphed.capture()
    graphed.run()
    torch.cuda.synchronize()
    assert torch.equal(eager.x, graphed.x)
    assert np.array_equal(eager.active_counts(), graphed.active_counts())


def test_stage_events_inside_graph(cuda_device):
    import torch

    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

    model = DecodeModel(2, 64, 6, 1024, 512, seed=2)
    st = DecodeStep(model, 128, 1, 0.5)
    st.enable_stage_events()
    st.capture()
    st.run()
    torch.cuda.synchronize()
    t = st.stage_times_ms()
    assert t.shape == (2, 5) and np.all(t > 0) and np.all(t < 50)


def test_ep_shards_sum_to_full_layer(cuda_device):
    """Virtual ranks on one GPU: each shard's sere_moe_forward_ep partial, summed, equals the
    full-bank layer; every shard reports the same bit-exact re-routed ids."""
    import torch

    from paper_2602_07616_b200 import ep
    from paper_2602_07616_b200.moe import ExpertBank, moe_forward_device, moe_forward_ep_device

    M, ns, K, d_h, d_m, T = 64, 2, 6, 1024, 512, 96
    full = ExpertBank.random(M, ns, d_h, d_m, seed=5)
    x = torch.randn(T, d_h, device="cuda").to(torch.bfloat16)
    top = torch.topk(torch.randn(T, M, device="cuda") + 1.5 * torch.randn(M, device="cuda"), K, dim=1)
    ids, w = top.indices.to(torch.int32), torch.softmax(top.values, 1)
    sim = O.random_symmetric_sim(np.random.default_rng(1), M)
    ref = moe_forward_device(full, sim, 1, 0.5, x, ids, w)
    ref.check()
    for world in (2, 4):
        total = torch.zeros(T, d_h, device="cuda")
        for r in range(world):
            lo, hi = ep.expert_range(M, world, r)
            bank = ExpertBank.random(M, ns, d_h, d_m, seed=5, expert_ids=range(lo, hi),
                                     shared_ids=ep.shared_owned(ns, world, r))
            out = moe_forward_ep_device(bank, M, lo, sim, 1, 0.5, x, ids, w)
            out.check()
            assert torch.equal(out.reroute.new_indices, ref.reroute.new_indices)
            total += out.y
        err = (total - ref.y).abs().max().item()
        assert err <= 1e-5 * max(1.0, ref.y.abs().max().item()), (world, err)


def test_ep_step_single_rank_nccl_equals_decode_step(cuda_device):
    """EPDecodeStep over a 1-rank NCCL group (all-gather / reduce-scatter are identities) must
    reproduce DecodeStep bit for bit, eager and CUDA-graph captured (NCCL inside the graph)."""
    import torch
    import torch.distributed as dist

    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep
    from paper_2602_07616_b200.ep import EPDecodeStep

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        model = DecodeModel(3, 32, 4, 512, 256, seed=4, beta=1.0)
        ref = DecodeStep(model, 64, 1, 0.5)
        epstep = EPDecodeStep(model, 64, 1, 0.5)
        x0 = torch.randn(64, 512, device="cuda")
        ref.set_input(x0)
        epstep.x_in.copy_(x0)
        ref.run()
        epstep.run()
        torch.cuda.synchronize()
        assert torch.equal(ref.x, epstep.x)
        graphed = epstep.capture()
        epstep.run()
        torch.cuda.synchronize()
        assert torch.equal(ref.x, epstep.x)
        print("EP graph capture:", graphed)
    finally:
        dist.destroy_process_group()


def test_nonfinite_token_state_raises_domain_error(cuda_device):
    """A non-finite token state: the reference's route_topk raises DomainError (moe.py:274-275).
    The device router flags the token (SERE_ID_NONFINITE) instead of emitting colliding ids,
    the fused layer reports DomainError, and the host drop-in raises before launching."""
    import torch

    from paper_2602_07616_b200 import moe
    from paper_2602_07616_b200.errors import DomainError

    M, K, d_h, d_m, T = 32, 4, 256, 128, 40
    bank = moe.ExpertBank.random(M, 0, d_h, d_m, seed=2)
    w = (torch.randn(d_h, M, device="cuda") / d_h ** 0.5).to(torch.bfloat16)
    x = torch.randn(T, d_h, device="cuda").to(torch.bfloat16)
    x[7, 3] = float("nan")
    ids, wts = moe.route_topk_device(moe.router_weight_t(w), x, K)
    got = ids.cpu().numpy()
    assert np.all(got[7] == np.iinfo(np.int32).min)
    assert np.all((got[np.arange(T) != 7] >= 0) & (got[np.arange(T) != 7] < M))
    out = moe.moe_forward_device(bank, O.random_symmetric_sim(np.random.default_rng(0), M), 1, 0.5, x, ids, wts)
    with pytest.raises(DomainError):
        out.check()
    router = type("R", (), {"w_router": w.float().cpu().numpy(), "top_k": K})()
    xh = x.float().cpu().numpy()
    with pytest.raises(DomainError):
        moe.route_topk(router, xh)


def test_launch_and_l2_knobs_do_not_change_results(cuda_device):
    """sere_set_pdl (programmatic dependent launch per kernel) and sere_set_l2 (dead expert outputs
    dropped from L2 before the next layer's permute) change timing only: the C4-shaped step's
    residual stream is bit-identical under every setting (graph replay, 2 steps each)."""
    import torch

    from paper_2602_07616_b200 import _lib
    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

    model = DecodeModel(3, 128, 8, 2048, 768, seed=4, beta=1.0)
    x0 = torch.randn(512, 2048, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4))
    outs = {}
    try:
        for pdl, l2 in ((31, 1), (0, 0), (31, 0), (0, 1)):
            _lib.call("sere_set_pdl", pdl)
            _lib.call("sere_set_l2", l2)
            st = DecodeStep(model, 512, 1, 0.5)
            st.set_input(x0)
            st.capture()
            st.run()
            st.set_input(x0)
            st.run()
            torch.cuda.synchronize()
            st.check()
            outs[(pdl, l2)] = st.x.clone()
    finally:
        _lib.call("sere_set_pdl", 31)
        _lib.call("sere_set_l2", 1)
    ref = outs[(31, 1)]
    for k, v in outs.items():
        assert torch.equal(v, ref), k
