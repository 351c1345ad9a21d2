O=gpurun_out/r2t; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "tc or tensor or scan or ivf" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
KNOB_COMPARE=1 timeout 1500 python tools/knob_sweep.py cfg4 "" 2>&1 | tail -4
