"""Aggregate ncu source-page stall samples per CUDA source line (ncu -i X --page source --csv --print-source cuda,sass).

    python scripts/ncu_lines.py rep.ncu-rep [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = {}
cur = None
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 6 or r[0] == "Line No":
        continue
    if r[0] != "":
        cur = (fname, int(r[0]), r[1][:90])
        continue
    if cur is None:
        continue
    try:
        s = int(r[4]); n = int(r[7])
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += s
    a[1] += n
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln, src), (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100.0 * s / tot:5.1f}%  {s:6d}  inst {n:7d}  {f}:{ln}  {src}")
