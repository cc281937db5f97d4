"""Expert parallelism over peer memory (ep_p2p.py, include/sere_b200.h (4c)) as virtual
ranks on one GPU: the ranks' kernels load/store each other's regions exactly as they
would over NVLink, and the step must reproduce the single-GPU decode step bit for bit."""

import pytest


def _shards(L, M, K, d_h, d_m, n_shared, world):
    from paper_2602_07616_b200.decode import DecodeModel
    from paper_2602_07616_b200.ep import expert_range, shared_owned

    return [DecodeModel(L, M, K, d_h, d_m, n_shared=n_shared, seed=4, beta=1.0,
                        expert_ids=range(*expert_range(M, world, r)), shared_ids=shared_owned(n_shared, world, r))
            for r in range(world)]


def _run(steps, streams):
    import torch

    from paper_2602_07616_b200.ep_p2p import P2PDecodeStep

    P2PDecodeStep.run_local(steps, streams)
    torch.cuda.synchronize()
    for st in steps:
        st.check()


@pytest.mark.gpu
@pytest.mark.parametrize("world,n_shared,mode,shape,fused", [(2, 0, "sere", "small", True),
                                                             (4, 2, "sere", "small", True),
                                                             (2, 1, "topk", "small", True),
                                                             (2, 0, "sere", "c4", True),
                                                             (4, 2, "sere", "small", False)])
def test_p2p_virtual_ranks_bit_exact_with_decode_step(cuda_device, world, n_shared, mode, shape, fused):
    """fused: the barriers live in the router / FFN (arrive) and align / combine (wait) kernels;
    otherwise two sere_ep_barrier kernels per layer."""
    import torch

    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep
    from paper_2602_07616_b200.ep_p2p import P2PDecodeStep

    if shape == "c4":  # the Qwen3-30B-A3B layer shape (2 layers, half the decode batch)
        L, M, K, d_h, d_m, T = 2, 128, 8, 2048, 768, 256
    else:
        L, M, K, d_h, d_m, T = 3, 32, 4, 512, 256, 64
    ref = DecodeStep(DecodeModel(L, M, K, d_h, d_m, n_shared=n_shared, seed=4, beta=1.0), T, 1, 0.5, mode)
    steps = [P2PDecodeStep(m, T, world, r, 1, 0.5, mode, fused_barriers=fused)
             for r, m in enumerate(_shards(L, M, K, d_h, d_m, n_shared, world))]
    P2PDecodeStep.connect_local(steps)
    streams = [torch.cuda.Stream() for _ in steps]
    try:
        for it in range(2):  # the second step runs on advanced barrier epochs
            x0 = torch.randn(T, d_h, device="cuda")
            ref.set_input(x0)
            ref.run()
            for st in steps:
                st.x_in.copy_(x0[st.t0:st.t1])
            torch.cuda.synchronize()
            _run(steps, streams)
            ref.check()
            for l in range(L):
                for st in steps:
                    assert torch.equal(st.outs[l].reroute.new_indices, ref.outs[l].reroute.new_indices), (it, l)
            got = torch.cat([st.x for st in steps])
            assert torch.equal(got, ref.x), (it, (got - ref.x).abs().max().item())
        assert all(int(st.epoch.item()) == 2 * 2 * L for st in steps)
        del ref
    finally:
        for st in steps:
            st.close()


@pytest.mark.gpu
def test_p2p_barrier_times_out_instead_of_hanging(cuda_device):
    """A rank whose peers never arrive reports SERE_ERR_CUDA through the status word."""
    import ctypes

    import torch

    from paper_2602_07616_b200 import _lib
    from paper_2602_07616_b200.ep_p2p import P2PDecodeStep
    from paper_2602_07616_b200.errors import SereError

    steps = [P2PDecodeStep(m, 32, 2, r, timeout_s=0.05) for r, m in enumerate(_shards(1, 8, 2, 256, 128, 0, 2))]
    P2PDecodeStep.connect_local(steps)
    try:
        st = steps[0]
        _lib.call("sere_ep_barrier", ctypes.byref(st.peers), st.epoch.data_ptr(), st.bar_status.data_ptr(),
                  ctypes.c_int64(st.timeout_ns), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        with pytest.raises(SereError):
            st.check()
        # the timeout is sticky and visible to every rank: both abort words are raised, and the
        # peer's next barrier fails at once (it would otherwise wait out its own 5 s timeout)
        assert [int(s.region.flags[_lib.MAX_EP_RANKS].item()) for s in steps] == [1, 1]
        peer = steps[1]
        peer.timeout_ns = int(5e9)
        import time

        t0 = time.perf_counter()
        _lib.call("sere_ep_barrier", ctypes.byref(peer.peers), peer.epoch.data_ptr(), peer.bar_status.data_ptr(),
                  ctypes.c_int64(peer.timeout_ns), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert time.perf_counter() - t0 < 1.0
        with pytest.raises(SereError):
            peer.check()
    finally:
        for st in steps:
            st.close()


def _ipc_worker(rank, world, port, out_dir):
    import os

    import torch
    import torch.distributed as dist

    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep
    from paper_2602_07616_b200.ep_p2p import P2PDecodeStep

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    L, M, K, d_h, d_m, T = 2, 16, 4, 256, 256, 32
    st = P2PDecodeStep(_shards(L, M, K, d_h, d_m, 0, world)[rank], T, world, rank, timeout_s=20.0)
    st.connect_ipc()
    g = torch.Generator(device="cuda").manual_seed(11)
    x0 = torch.randn(T, d_h, device="cuda", generator=g)
    st.x_in.copy_(x0[st.t0:st.t1])
    dist.barrier()
    st.run()
    torch.cuda.synchronize()
    st.check()
    ref = DecodeStep(DecodeModel(L, M, K, d_h, d_m, seed=4, beta=1.0), T, 1, 0.5)
    ref.set_input(x0)
    ref.run()
    torch.cuda.synchronize()
    ok = torch.equal(st.x, ref.x[st.t0:st.t1])
    (out_dir / f"rank{rank}.txt").write_text("ok" if ok else f"mismatch {(st.x - ref.x[st.t0:st.t1]).abs().max()}")
    dist.barrier()
    st.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_p2p_two_processes_ipc(cuda_device, tmp_path):
    """Two processes (time-sliced on one GPU here, one per GPU in production): CUDA IPC
    handles exchanged over a gloo group, peer regions mapped, one step bit-exact."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_ipc_worker, args=(2, port, tmp_path), nprocs=2, join=True)
    assert [(tmp_path / f"rank{r}.txt").read_text() for r in range(2)] == ["ok", "ok"]
