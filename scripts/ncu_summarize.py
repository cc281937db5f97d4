"""Summaries for profiles/ from a gpu_round.sh capture (run here, on the copied-back files).

    python scripts/ncu_summarize.py TAG [--round r02] [--rep gpurun_out/prof_ffn.ncu-rep] [--launches gpurun_out/launches.csv]

Writes profiles/RR_ncu_summary_TAG.txt, profiles/RR_ncu_traffic_TAG.json (per-launch DRAM
bytes of moe_ffn_kernel next to its algorithmic bytes) and profiles/RR_launches_TAG.csv /
_summary.txt (the serialised launch list's per-kernel share)."""
import argparse
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
           "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__cycles_active.avg", "gpc__cycles_elapsed.max",
           "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           # tensor pipe (tcgen05 UTCHMMA) utilisation of the grouped GEMM
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum",
           "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "smsp__mem_tensor_writes_op_utcmma.sum", "smsp__sass_inst_executed_op_tmem_ldt.sum",
           "dram__bytes_read.sum.pct_of_peak_sustained_elapsed"]
D_H, D_M = 2048, 768


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return [dict(zip(hdr, r)) for r in data], dict(zip(hdr, units))


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--rep", default="gpurun_out/prof_ffn.ncu-rep")
    ap.add_argument("--launches", default="gpurun_out/launches.csv")
    ap.add_argument("--note", default="")
    ap.add_argument("--round", default="r02")
    ap.add_argument("--layers", type=int, default=4, help="profile_step --layers of the capture")
    ap.add_argument("--skip", type=int, default=1, help="ncu -s: FFN launches skipped before the capture")
    a = ap.parse_args()
    rows, units = raw(a.rep)
    lines = [f"# {a.round} ncu summary {a.tag}: ncu --set full --clock-control none --import-source on; "
             f"profile_step --layers {a.layers} (captured launches from index {a.skip}; C4, SERE S=1 rho=0.5 beta=1). {a.note}"]
    launches = []
    for i, r in enumerate(rows):
        if "moe_ffn" not in r.get("Kernel Name", ""):
            continue
        for m in METRICS:
            if m in r:
                lines.append(f"{i} moe_ffn_kernel {m} {r[m]} {units.get(m, '')}")
        rd, wr = num(r["dram__bytes_read.sum"]), num(r["dram__bytes_write.sum"])
        # byte units as reported (ncu raw pages report bytes; scale if it says Mbyte etc.)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
        wr *= scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
        dur = num(r["gpu__time_duration.sum"]) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(
            units.get("gpu__time_duration.sum", "nsecond"), 1e-3)
        launches.append({"dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "duration_us": round(dur, 3)})
    prof_log = ROOT / "gpurun_out/prof.log"
    actives = []
    if prof_log.exists():
        for ln in prof_log.read_text().splitlines():
            if ln.startswith("active experts per layer:"):
                actives = [int(v) for v in ln.split(":", 1)[1].strip(" []").split(",")]
    for i, L in enumerate(launches):
        if i + a.skip < len(actives):
            L["active_experts"] = actives[i + a.skip]
            L["algorithmic_bytes"] = (2 * 3 * D_H * D_M * actives[i + a.skip] + 2 * 512 * D_H + 4 * 512 * D_H
                                      + 8 * 512 * 8)
    (ROOT / f"profiles/{a.round}_ncu_summary_{a.tag}.txt").write_text("\n".join(lines) + "\n")
    if launches and all("algorithmic_bytes" in L for L in launches):
        (ROOT / f"profiles/{a.round}_ncu_traffic_{a.tag}.json").write_text(json.dumps(
            {"kernel": "moe_ffn_kernel", "source": f"profiles/{a.round}_ncu_summary_{a.tag}.txt", "launches": launches,
             "note": "ncu flushes L2 before each replay, so activation/h reads that are L2 hits in the graph-replayed "
                     "step count as DRAM here"}, indent=1) + "\n")
    print("\n".join(lines))
    print(json.dumps(launches))
    # launch list
    if Path(a.launches).exists():
        txt = Path(a.launches).read_text()
        rows = [r for r in csv.reader(io.StringIO(txt[txt.index('"ID"'):]))] if '"ID"' in txt else []
        if rows:
            hdr = rows[0]
            ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
            agg = defaultdict(list)
            for r in rows[1:]:
                if len(r) > vi:
                    agg[r[ki].split("(")[0].replace("sere::", "")].append(num(r[vi]) / 1e3)
            tot = sum(sum(v) for v in agg.values())
            out = [f"ncu --metrics gpu__time_duration.sum --clock-control none, profile_step --layers 4 (C4), eager, cold/serialised ({a.tag})"]
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
                out.append(f"{k:32s} launches={len(v):3d} avg_us={sum(v)/len(v):8.2f} share={sum(v)/tot:.3f}")
            out.append(f"total us {tot:.1f}")
            (ROOT / f"profiles/{a.round}_launches_{a.tag}_summary.txt").write_text("\n".join(out) + "\n")
            (ROOT / f"profiles/{a.round}_launches_{a.tag}.csv").write_text(txt)
            print("\n".join(out))


if __name__ == "__main__":
    sys.exit(main())
