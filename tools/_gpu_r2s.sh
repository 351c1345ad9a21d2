O=gpurun_out/r2s; mkdir -p $O
tools/tc_mma_bench > $O/mma_bench.txt 2>&1; tail -25 $O/mma_bench.txt
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
KNOB_LIST_STATS=1 timeout 1200 python tools/knob_sweep.py cfg4 "" 2>&1 | tail -16
