mkdir -p gpurun_out/s3
python tools/phase_times.py cfg2 100000000 10000 > gpurun_out/s3/phase_cfg2.txt 2>&1
QADC_B200_VARIANT_STATS=1 python tools/phase_times.py cfg1 10000000 1000 > gpurun_out/s3/phase_cfg1.txt 2>&1
python - > gpurun_out/s3/phase_cfg2_np64.txt 2>&1 <<'PY'
import sys, runpy
sys.argv=["x","cfg2","100000000","10000"]
import paper_1704_07355_b200.workload as w
import dataclasses
w.IVF_CONFIGS["cfg2"]=dataclasses.replace(w.IVF_CONFIGS["cfg2"], nprobe=64)
runpy.run_path("tools/phase_times.py", run_name="__main__")
PY
cat gpurun_out/s3/*.txt
