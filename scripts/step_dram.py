"""DRAM traffic of the graph-replayed C4 decode step (one graph launch in the profiler range).

    ncu --profile-from-start off --graph-profiling graph --cache-control none --clock-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum python scripts/step_dram.py
"""
import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=48)
    ap.add_argument("--mode", default="sere")
    ap.add_argument("--l2", type=int, default=None)
    a = ap.parse_args()
    import torch

    from paper_2602_07616_b200 import build
    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

    build.build()
    if a.l2 is not None:
        from paper_2602_07616_b200 import _lib

        _lib.call("sere_set_l2", a.l2)
    model = DecodeModel(a.layers, 128, 8, 2048, 768, seed=0, beta=1.0)
    step = DecodeStep(model, 512, 1, 0.5, a.mode)
    step.set_input(torch.randn(512, 2048, device="cuda"))
    step.capture()
    for _ in range(3):
        step.run()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    step.run()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ws = step.model  # noqa: F841
    print("weights bytes per step (algorithmic):", sum(step.active_counts().tolist()) * 3 * 2048 * 768 * 2)


if __name__ == "__main__":
    main()
