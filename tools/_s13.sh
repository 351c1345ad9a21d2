D=gpurun_out/s13; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $D/smoke.log
timeout 300 python tools/phase_times.py cfg1 10000000 1000 > $D/phase_cfg1_tc.txt 2>&1
head -8 $D/phase_cfg1_tc.txt
