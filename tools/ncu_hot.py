"""Developer tool: stall reasons and SASS hotspots of an ncu report.

    python tools/ncu_hot.py gpurun_out/s13/tc_cfg1.ncu-rep [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
d = dict(zip(rows[0], rows[2]))
print("duration", d.get("gpu__time_duration.sum"), "inst", d.get("smsp__inst_executed.sum"),
      "issue%", d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
      "tensor%", d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"))
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
      for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
      and not k.endswith("not_issued") and v.replace(",", "").replace(".", "").isdigit()}
tot = sum(st.values())
print(" ".join(f"{k}={v / tot * 100:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]))
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


data = [(f(r, "Instructions Executed"), f(r, "Warp Stall Sampling (All Samples)"), i, r[1])
        for i, r in enumerate(rows[2:]) if len(r) >= len(h) - 2]
ti = sum(x[0] for x in data) or 1
ts = sum(x[1] for x in data) or 1
for x in sorted(data, key=lambda x: -x[1])[:N]:
    print(f"{x[0] / ti * 100:5.2f}%i {x[1] / ts * 100:5.2f}%s #{x[2]} {x[3][:80]}")
