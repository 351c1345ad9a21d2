"""Developer tool: executed-instruction mix by SASS opcode of an ncu report
(source page), and the share of the hottest address ranges.

    python tools/ncu_opmix.py gpurun_out/r2a/scan_prmt_cfg4.ncu-rep [lookups]
"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
lookups = float(sys.argv[2]) if len(sys.argv) > 2 else None
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}


def f(r, k):
    try:
        return float(r[idx[k]].replace(",", ""))
    except Exception:
        return 0.0


ops = Counter()
tot = 0.0
for r in rows[2:]:
    if len(r) < len(h) - 2:
        continue
    n = f(r, "Instructions Executed")
    text = r[1].strip()
    if not text:
        continue
    tok = text.split()
    op = tok[0]
    if op.startswith("@"):
        op = tok[1]
    ops[op.split(".")[0]] += n
    tot += n
print(f"total warp-instructions {tot:.4g}")
for op, n in ops.most_common(25):
    extra = f"  {n * 32 / lookups:.3f} lane-instr/lookup" if lookups else ""
    print(f"  {op:10s} {n / tot * 100:6.2f}%{extra}")
if lookups:
    print(f"  all        {tot * 32 / lookups:.3f} lane-instr/lookup")
