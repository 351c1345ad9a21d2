"""Top SASS instructions by warp-stall samples from an
`ncu --page source --csv --print-source sass` export (developer tool)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
data = []
for r in rows[2:]:
    try:
        n = int(r[si])
    except (ValueError, IndexError):
        continue
    data.append((n, r))
tot = sum(n for n, _ in data)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot)
for n, r in sorted(data, key=lambda x: -x[0])[:top]:
    st = sorted(((int(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{n:6d} {100 * n / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:60]:60s} {st}")
