"""Profiling driver: a short C4-shaped decode run bracketed by cudaProfilerStart/Stop.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py
    ncu --profile-from-start off --set full --import-source on -k regex:moe_ffn -c 2 \
        -o gpurun_out/prof python scripts/profile_step.py --layers 2

Only the profiled steps are inside the profiler range (weight generation, packing and
warm-up are not), launched eagerly so every kernel appears as its own launch.
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import argparse


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--T", type=int, default=512)
    ap.add_argument("--mode", choices=["sere", "topk"], default="sere")
    ap.add_argument("--beta", type=float, default=1.0)
    a = ap.parse_args()

    import torch

    from paper_2602_07616_b200 import build
    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

    build.build()
    model = DecodeModel(a.layers, 128, 8, 2048, 768, seed=0, beta=a.beta)
    step = DecodeStep(model, a.T, 1, 0.5, a.mode)
    step.set_input(torch.randn(a.T, 2048, device="cuda"))
    for _ in range(3):
        step.run()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.steps):
        step.run()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    step.check()
    print("active experts per layer:", step.active_counts().tolist())


if __name__ == "__main__":
    main()
