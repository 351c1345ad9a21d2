D=gpurun_out/s14; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $D/pytest_gpu.log
timeout 300 python tools/phase_times.py cfg1 10000000 1000 > $D/phase_cfg1_g4.txt 2>&1
QADC_B200_TC_GROUPS=2 timeout 300 python tools/phase_times.py cfg1 10000000 1000 > $D/phase_cfg1_g2.txt 2>&1
timeout 300 python tools/phase_times.py cfg0 1000000 100 > $D/phase_cfg0.txt 2>&1
timeout 300 python tools/phase_times.py cfg3 1000000 1000 > $D/phase_cfg3.txt 2>&1
head -7 $D/phase_*.txt
