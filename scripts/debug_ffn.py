"""Per-CTA timeline of the fused FFN kernel (sere_debug_set_ffn_trace) on C4-shaped layers.

    python scripts/debug_ffn.py [--layers 4 --mode sere --out gpurun_out/ffn_trace.npz]

Prints, per traced layer: kernel span, the spread of CTA start/end times (tail),
and the average per-CTA wait split (producer slot-wait = ring full, MMA operand
wait = bytes not landed, dependency wait, accumulator wait, epilogue wait).
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import argparse


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--T", type=int, default=512)
    ap.add_argument("--mode", choices=["sere", "topk"], default="sere")
    ap.add_argument("--beta", type=float, default=1.0)
    ap.add_argument("--out", default="")
    ap.add_argument("--dbg-mode", type=int, default=0, help="1: skip weight copies, 2: skip MMAs (invalid output)")
    a = ap.parse_args()

    import numpy as np
    import torch

    from paper_2602_07616_b200 import _lib, build
    from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

    build.build()
    lib = _lib.load()
    model = DecodeModel(a.layers, 128, 8, 2048, 768, seed=0, beta=a.beta)
    step = DecodeStep(model, a.T, 1, 0.5, a.mode)
    step.set_input(torch.randn(a.T, 2048, device="cuda"))
    for _ in range(3):
        step.run()
    torch.cuda.synchronize()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    traces = []
    bufs = [torch.zeros(sms * 2048, dtype=torch.int64, device="cuda") for _ in range(a.layers)]

    def hook(i):  # eager step: point the kernel at layer i's trace buffer before its launch
        lib.sere_debug_set_ffn_trace(bufs[i].data_ptr())

    step._trace_hook = hook
    lib.sere_debug_set_ffn_mode(a.dbg_mode)
    step.run()
    torch.cuda.synchronize()
    lib.sere_debug_set_ffn_mode(0)
    lib.sere_debug_set_ffn_trace(None)
    acts = step.active_counts()
    unit_bytes = {}  # filled per layer below (weights per unit from the plan is not exported: approximate)
    for l in range(a.layers):
        tr = bufs[l].view(sms, 2048).cpu().numpy().astype(np.int64)
        if tr[:, 0].max() == 0:
            continue
        t0 = tr[:, 0].min()
        start, end = tr[:, 0] - t0, tr[:, 7] - t0
        span = end.max()
        nunits = tr[:, 3]
        ns_per_cyc = (tr[:, 7] - tr[:, 0]).sum() / max((tr[:, 814] - tr[:, 813]).sum(), 1)
        w = {k: tr[:, i].mean() * ns_per_cyc / 1e3 for k, i in (("slot_wait", 1), ("operand_wait", 2), ("dep_wait", 4),
                                                    ("acc_wait", 5), ("epi_wait", 6),
                                                    ("queue_wait", 809), ("mma_issue", 811),
                                                    ("mma_queue_wait", 812), ("mma_commit", 1016),
                                                    ("mma_fence", 1017), ("mma_loop_total", 815))}
        units = []
        for c in range(sms):
            for i in range(min(int(nunits[c]), 200)):
                u, tt, tf, tl = tr[c, 8 + 4 * i: 12 + 4 * i]
                units.append((c, int(u), (tt - t0) / 1e3, (tf - t0) / 1e3, (tl - t0) / 1e3,
                              (tr[c, 816 + i] - t0) / 1e3))
        units = np.array(units)
        bytes_ = 2 * 3 * 2048 * 768 * int(acts[l])
        print(f"layer {l}: active {int(acts[l])}, span {span/1e3:.1f} us, {bytes_/span:.0f} GB/s, "
              f"units {int(nunits.sum())} ({nunits.min()}..{nunits.max()} per CTA), "
              f"start spread {start.max()/1e3:.1f} us, end spread {(end.max()-end.min())/1e3:.1f} us "
              f"(end p10 {np.percentile(end,10)/1e3:.1f} p50 {np.percentile(end,50)/1e3:.1f})")
        print("   mean per-CTA waits (us): " + ", ".join(f"{k} {v:.1f}" for k, v in w.items())
              + f"; clock {1 / ns_per_cyc:.2f} GHz; k-steps/CTA {tr[:, 810].mean():.0f} -> {span / max(tr[:, 810].mean(), 1):.0f} ns each")
        traces.append(tr)
        # bandwidth profile: each unit's weight bytes spread uniformly over [first copy, last copy]
        if len(units):
            ub = np.zeros(len(units))
            for i, (c, u, tt, tf, tl, te) in enumerate(units):
                ub[i] = float((int(u) >> 24) & 0xFFFFF) * 1024.0
            edges = np.arange(0.0, span / 1e3 + 5.0, 5.0)
            hist = np.zeros(len(edges) - 1)
            for (c, u, tt, tf, tl, te), b in zip(units, ub):
                if tl <= tf:
                    continue
                lo = np.clip((edges[:-1] - tf) / (tl - tf), 0, 1)
                hi = np.clip((edges[1:] - tf) / (tl - tf), 0, 1)
                hist += (hi - lo) * b
            print("   issue-rate TB/s per 5us:", " ".join(f"{h / 5e-6 / 1e12:.1f}" for h in hist))
            cyc = ns_per_cyc / 1e3
            print(f"   down-phase waits (us/CTA): slot {tr[:, 1018].mean() * cyc:.1f} of {tr[:, 1].mean() * cyc:.1f}, "
                  f"operand {tr[:, 1019].mean() * cyc:.1f} of {tr[:, 2].mean() * cyc:.1f}, "
                  f"tmem {tr[:, 1020].mean() * cyc:.1f} of {tr[:, 5].mean() * cyc:.1f}; "
                  f"down k-steps {tr[:, 1021].mean():.0f} of {tr[:, 810].mean():.0f}")
            kind = np.array([(int(u) >> 53) & 1 for u in units[:, 1]])
            nm = np.array([(int(u) >> 44) & 0x1FF for u in units[:, 1]])
            dur = units[:, 4] - units[:, 3]
            for dn in (0, 1):
                for lo_n, hi_n in ((0, 48), (48, 96), (96, 160), (160, 257)):
                    m = (kind == dn) & (nm > lo_n) & (nm <= hi_n)
                    if m.sum():
                        print(f"   {'dn' if dn else 'gu'} N({lo_n},{hi_n}]: {int(m.sum())} units, issue span "
                              f"{dur[m].mean():.1f} us, {ub[m].sum() / max(dur[m].sum(), 1e-9) / 1e3:.1f} GB/s per SM, "
                              f"ticket->first {(units[m, 3] - units[m, 2]).mean():.2f} us")
        if l == 0 and len(units):
            last = units[np.argsort(units[:, 5])[-8:]]
            print("   last units (cta, ticket, t_ticket, t_first, t_last_copy, t_epi):")
            for r in last:
                print("     ", [round(float(v), 1) for v in r])
    if a.out:
        np.savez(a.out, *traces)


if __name__ == "__main__":
    main()
