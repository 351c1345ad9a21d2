D=gpurun_out/s12; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu.log
timeout 600 python tools/phase_times.py cfg2 100000000 10000 > $D/phase_cfg2_tc.txt 2>&1
QADC_B200_TC=0 timeout 600 python tools/phase_times.py cfg2 100000000 10000 > $D/phase_cfg2_prmt.txt 2>&1
QADC_B200_TC=0 timeout 600 python tools/phase_times.py cfg1 10000000 1000 > $D/phase_cfg1_prmt.txt 2>&1
head -8 $D/phase_*.txt
