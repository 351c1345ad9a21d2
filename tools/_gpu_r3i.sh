O=gpurun_out/r3i; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
KNOB_PROFILE=1 timeout 1500 python tools/knob_sweep.py cfg4 "" > $O/sweep0.txt 2>&1; grep -E "^\[| ms x" $O/sweep0.txt | cut -c1-200 | head -14
