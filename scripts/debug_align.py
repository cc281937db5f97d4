"""Phase timing of the re-routing/align kernel (clock64 after each barrier phase).

    python scripts/debug_align.py [--T 512 --M 128 --K 8]
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import argparse


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=512)
    ap.add_argument("--M", type=int, default=128)
    ap.add_argument("--K", type=int, default=8)
    ap.add_argument("--beta", type=float, default=1.0)
    a = ap.parse_args()

    import numpy as np
    import torch

    from paper_2602_07616_b200 import _lib, build
    from paper_2602_07616_b200.decode import uniform_sim
    from paper_2602_07616_b200.rerouting import DeviceSimilarity, reroute

    build.build()
    T, M, K = a.T, a.M, a.K
    logits = torch.randn(T, M, device="cuda") + a.beta * torch.randn(M, device="cuda")
    ids = torch.topk(logits, K, dim=1).indices.to(torch.int32)
    sim = DeviceSimilarity(uniform_sim(np.random.default_rng(0), M))  # validated once, like the decode step
    dbg = torch.zeros(16, dtype=torch.int64, device="cuda")
    for _ in range(3):
        reroute(ids, sim, 1, 0.5).check()
    _lib.load().sere_debug_set_align_clocks(dbg.data_ptr())
    reroute(ids, sim, 1, 0.5).check()
    torch.cuda.synchronize()
    _lib.load().sere_debug_set_align_clocks(None)
    c = dbg.cpu().numpy()
    print("reroute-only (cycles): argmax", int(c[4] - c[1]), "final table", int(c[5] - c[4]), "total", int(c[5] - c[0]))

    from paper_2602_07616_b200.moe import ExpertBank, moe_forward_device

    bank = ExpertBank.random(M, 0, 256, 128, seed=0)  # small dims: only the align kernel matters here
    x = torch.randn(T, 256, device="cuda").to(torch.bfloat16)
    w = torch.full((T, K), 1.0 / K, device="cuda")
    for _ in range(3):
        moe_forward_device(bank, sim, 1, 0.5, x, ids, w).check()
    acc = np.zeros(16)
    for _ in range(20):
        dbg.zero_()
        _lib.load().sere_debug_set_align_clocks(dbg.data_ptr())
        moe_forward_device(bank, sim, 1, 0.5, x, ids, w).check()
        torch.cuda.synchronize()
        _lib.load().sere_debug_set_align_clocks(None)
        cc = dbg.cpu().numpy().astype(np.float64)
        acc += cc - cc[0]
    c = acc / 20
    names = {0: "init", 1: "load ids", 4: "argmax", 5: "final table+counts",
             7: "block prefix", 10: "group layout", 11: "schedule sort", 8: "unit prefix"}
    order = [0, 1, 4, 5, 7, 10, 11, 8]
    prev = c[0]
    parts = []
    for i in order[1:]:
        parts.append(f"{names[i]} {int(c[i] - prev)}")
        prev = c[i]
    print("reroute+align phase cycles:", ", ".join(parts), "| total", int(c[8] - c[0]))


if __name__ == "__main__":
    main()
