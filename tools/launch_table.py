"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launches, mean duration and share of the captured time
(developer tool; used for profiles/README.md)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
agg = collections.defaultdict(list)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v = v / 1000 if r[ui] == "ns" else (v * 1000 if r[ui] == "ms" else v)
    name = r[ki].split("(")[0].replace("qadc::<unnamed>::", "").replace("void ", "")
    agg[name].append(v)
tot = sum(sum(v) for v in agg.values())
print(f"| kernel | launches | avg us | share |\n|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.3f} |")
print(f"\ncaptured: {sum(len(v) for v in agg.values())} launches, {tot / 1000:.2f} ms")
