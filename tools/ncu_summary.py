"""Write profiles/scan_ncu_<config>.json from an `ncu --set full` report of
the scan kernel (developer tool; bench.py reads that config's DRAM traffic
per launch from it).

    python tools/ncu_summary.py gpurun_out/r2g/scan_prmt_cfg4.ncu-rep "<kernel label>" "<command>" cfg4
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

rep, label, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
config = sys.argv[4] if len(sys.argv) > 4 else "cfg1"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
units = dict(zip(h, u))


def num(k):
    x = d.get(k)
    if x is None:
        return None
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def nbytes(k):
    x, un = num(k), units.get(k, "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(un, 1)
    return None if x is None else int(x * scale)


def ms(k):
    x, un = num(k), units.get(k, "")
    return None if x is None else x * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                                        "msecond": 1.0, "nsecond": 1e-6}.get(un, 1.0)


rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
out = {
    "kernel": label,
    "source": f"{cmd} ({Path(rep).name})",
    "duration_ms": round(ms("gpu__time_duration.sum"), 4),
    "dram_bytes_read_per_launch": rd,
    "dram_bytes_write_per_launch": wr,
    "dram_bytes_per_launch": (rd or 0) + (wr or 0),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "tensor_pipe_active_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "int8_tensor_ops_pct_of_peak": num(
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed"),
    "alu_pipe_active_pct": num("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "shared_pipe_active_pct": num("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "block_size": num("launch__block_size"),
    "grid": num("launch__grid_size"),
    "dram_throughput_pct": num("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    "fmaheavy_pipe_active_pct": num("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    "lsu_shared_wavefronts_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "instructions_executed": num("smsp__inst_executed.sum"),
    "achieved_warps_per_sm": num("sm__warps_active.avg.per_cycle_active"),
}
json.dump(out, open(Path(__file__).resolve().parents[1] / "profiles" / f"scan_ncu_{config}.json",
               "w"), indent=1)
print(json.dumps(out, indent=1))
