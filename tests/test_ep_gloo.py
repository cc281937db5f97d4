"""Expert-parallel choreography on CPU: world_size 2 over gloo (127.0.0.1).

Each rank owns half the routed experts and a subset of the shared experts, routes its
own token slice, all-gathers the packed rows (ep.Exchange), re-routes the FULL table,
evaluates only its experts (the CPU oracle stands in for the GPU kernels here) and
reduce-scatters the partial outputs. The assembled result must equal the
single-process reference model_forward."""

import os
import socket

import numpy as np
import pytest

from oracle import sere_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CFG = dict(seed=5, L=3, M=8, K=3, d_h=16, d_m=24, n_shared=3, T=8, S=1, rho=0.4)


def _setup():
    c = CFG
    layers = O.gen_layers(c["seed"], c["L"], c["M"], c["K"], c["d_h"], c["d_m"], c["n_shared"])
    rng = np.random.default_rng(9)
    sims = [O.random_symmetric_sim(rng, c["M"]) for _ in range(c["L"])]
    x0 = rng.standard_normal((c["T"], c["d_h"]))
    return layers, sims, x0


def _partial(layer, x, ids, w, lo, hi, shared):
    """This rank's share of moe.layer_forward (moe.py:302-309): owned experts only."""
    y = np.zeros_like(x)
    for k in range(ids.shape[1]):
        col = ids[:, k]
        for e in np.unique(col):
            if lo <= e < hi:
                rows = np.flatnonzero(col == e)
                y[rows] += w[rows, k:k + 1] * O.expert_forward(layer.experts[e], x[rows])
    for s in shared:
        y += O.expert_forward(layer.shared_experts[s], x)
    return y


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2602_07616_b200 import ep

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = CFG
        layers, sims, x0 = _setup()
        lo, hi = ep.expert_range(c["M"], world, rank)
        sh = ep.shared_owned(c["n_shared"], world, rank)
        t0, t1 = ep.token_slice(c["T"], world, rank)
        xch = ep.Exchange(t1 - t0, c["d_h"], c["K"], "cpu", h_dtype=torch.float64, y_dtype=torch.float64)
        x = x0[t0:t1]
        all_ids = []
        for l, layer in enumerate(layers):
            ids, w = O.route_topk(layer.w_router, c["K"], x)
            h_all, ids_all, w_all = xch.gather(torch.from_numpy(x), torch.from_numpy(ids.astype(np.int32)),
                                               torch.from_numpy(w.astype(np.float32)))
            ids_all = ids_all.numpy().astype(np.int64)
            res = O.apply_sere(ids_all, sims[l], c["S"], c["rho"])  # full table on every rank
            all_ids.append(res.new_indices)
            part = _partial(layer, h_all.numpy(), res.new_indices, w_all.numpy().astype(np.float64), lo, hi, sh)
            x = xch.reduce_scatter(torch.from_numpy(part)).numpy().copy()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), x=x, ids=np.stack(all_ids), t0=t0, t1=t1)
    finally:
        dist.destroy_process_group()


def test_ep_world2_matches_single_process(tmp_path):
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    c = CFG
    layers, sims, x0 = _setup()
    # single process: same per-token routing (fp32-rounded weights as exchanged), reference semantics
    x = x0.copy()
    ref_ids = []
    for l, layer in enumerate(layers):
        ids, w = O.route_topk(layer.w_router, c["K"], x)
        w = w.astype(np.float32).astype(np.float64)
        res = O.apply_sere(ids, sims[l], c["S"], c["rho"])
        ref_ids.append(res.new_indices)
        x = O.layer_forward(layer, x, res.new_indices, w)
    got = np.zeros_like(x)
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        got[int(z["t0"]):int(z["t1"])] = z["x"]
        for l in range(c["L"]):
            np.testing.assert_array_equal(z["ids"][l], ref_ids[l])  # every rank: bit-exact global ids
    np.testing.assert_allclose(got, x, rtol=1e-10, atol=1e-12)


def test_partition_helpers():
    from paper_2602_07616_b200 import ep

    for M in (8, 64, 128, 130):
        for world in (1, 2, 3, 4, 8):
            spans = [ep.expert_range(M, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    owned = sorted(s for r in range(3) for s in ep.shared_owned(5, 3, r))
    assert owned == list(range(5))
    assert ep.token_slice(512, 8, 7) == (448, 512)
    with pytest.raises(ValueError):
        ep.token_slice(10, 4, 0)
