"""Kernel-only FFN timing on C4-shaped layers (sere_debug_replay_ffn on the step's own workspace),
median of several batches, optionally under a debug mode (1 skip weight copies, 2 skip MMAs,
4 skip the expert-output stores; results invalid, timing only).

    python scripts/ffn_replay.py [sere|topk] [dbg_mode ...]
"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2602_07616_b200 import _lib, build
from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

build.build()
mode = sys.argv[1] if len(sys.argv) > 1 else "sere"
dbg_modes = [int(v) for v in sys.argv[2:]] or [0]
model = DecodeModel(4, 128, 8, 2048, 768, seed=0, beta=1.0)
step = DecodeStep(model, 512, 1, 0.5, mode)
step.set_input(torch.randn(512, 2048, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)))
step.run()
torch.cuda.synchronize()
bank = model.layers[-1].bank
ws_ptr, ws_bytes = step.workspace
act = int(step.outs[-1].reroute.n_active.item())
st = torch.cuda.current_stream()
args = (bank.data.data_ptr(), bank.M, bank.n_shared, 2048, 768, 0, 512, 8, ws_ptr, ws_bytes)
lib = _lib.load()
for dm in dbg_modes:
    lib.sere_debug_set_ffn_mode(dm)
    _lib.call("sere_debug_replay_ffn", *args, 3, st.cuda_stream)
    res = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.call("sere_debug_replay_ffn", *args, 10, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 10 * 1e3)
    us = float(np.median(res))
    b = 2 * 3 * 2048 * 768 * act + 6 * 512 * 2048 + 8 * 512 * 8
    print(f"ffn {mode} dbg_mode {dm}: active {act}, {us:.1f} us, {b / us / 1e3:.0f} GB/s  "
          f"(batches: {' '.join(f'{r:.1f}' for r in res)})")
lib.sere_debug_set_ffn_mode(0)
