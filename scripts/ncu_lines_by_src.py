"""Aggregate ncu source-page warp-stall samples per CUDA source line (ncu -i X --page source --csv
--print-source cuda,sass > f.csv; python scripts/ncu_lines_by_src.py f.csv [top])."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, hdr, agg, src = None, None, collections.Counter(), {}
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0] not in ("", "-"):
        line = (cur_file, int(r[0]))
        src[line] = r[1].strip()[:100]
    try:
        agg[line] += int(r[4] or 0)
    except ValueError:
        pass
tot = sum(agg.values())
print("total samples", tot)
for k, v in agg.most_common(top):
    print(f"{v:6d} {100 * v / max(tot, 1):5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')}")
