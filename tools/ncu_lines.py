"""Warp-stall samples per CUDA source line from an
`ncu --page source --csv --print-source cuda,sass` export (developer tool)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur, curfile = None, None
agg, src = collections.Counter(), {}
for r in rows:
    if r and r[0] == "File Path":
        curfile = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] not in ("", "Line No"):
        cur = (curfile, int(r[0]))
        src[cur] = r[1].strip()[:70]
    if len(r) > 4 and r[0] == "" and r[2].startswith("0x"):
        try:
            agg[cur] += int(r[4] or 0)
        except ValueError:
            pass
tot = sum(agg.values())
print("total", tot)
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{v:7d} {100 * v / tot:5.1f}% {k[0]}:{k[1]:4d} {src.get(k, '')}")
