"""Per-kernel device time of the graph-replayed C4 decode step (torch.profiler / CUPTI).

    python scripts/kernel_times.py [--layers 48 --mode sere --steps 3]
"""
import argparse
import pathlib
import sys
from collections import defaultdict

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=48)
    ap.add_argument("--mode", default="sere")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--T", type=int, default=512)
    ap.add_argument("--pdl", type=int, default=-1, help="sere_set_pdl mask (-1: library default)")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2602_07616_b200 import build
    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

    build.build()
    from paper_2602_07616_b200 import _lib
    if a.pdl >= 0:
        _lib.load().sere_set_pdl(a.pdl)
    model = DecodeModel(a.layers, 128, 8, 2048, 768, seed=0, beta=1.0)
    step = DecodeStep(model, a.T, 1, 0.5, a.mode)
    step.set_input(torch.randn(a.T, 2048, device="cuda"))
    step.capture()
    for _ in range(3):
        step.run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            step.run()
        torch.cuda.synchronize()
    agg = defaultdict(list)
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    for e in evs:
        agg[e.name.split("(")[0]].append(e.device_time if hasattr(e, "device_time") else e.cuda_time)
    tot = sum(sum(v) for v in agg.values())
    per_step = tot / a.steps
    print(f"{a.mode}: {len(evs)} kernels, device-busy {per_step / 1e3:.3f} ms/step, {per_step / a.layers:.1f} us/layer")
    for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {n[:40]:40s} n={len(v):5d} avg {sum(v) / len(v):8.2f} us  per-layer {sum(v) / a.steps / a.layers:7.2f} us  share {sum(v) / tot:.3f}")
    # timeline gaps: first start to last end per step
    starts = sorted((e.time_range.start, e.time_range.end) for e in evs)
    span = (starts[-1][1] - starts[0][0]) / a.steps
    print(f"  wall span per step {span / 1e3:.3f} ms (gaps+launch {(span - per_step) / a.layers:.1f} us/layer)")
    # chain view: for each kernel, start minus the previous kernel's end (negative = PDL overlap)
    seq = sorted(((e.time_range.start, e.time_range.end, e.name.split("(")[0]) for e in evs))
    gap = defaultdict(list)
    for (s0, e0, n0), (s1, e1, n1) in zip(seq, seq[1:]):
        gap[n1].append(s1 - e0)
    for n, v in sorted(gap.items(), key=lambda kv: -len(kv[1])):
        v = sorted(v)
        print(f"  gap before {n[:40]:40s} n={len(v):5d} avg {sum(v) / len(v):7.2f} us  median {v[len(v) // 2]:7.2f} us")


if __name__ == "__main__":
    main()
