O=gpurun_out/r2u; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "ivf or opq or cfg2" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
KNOB_COMPARE=1 timeout 1500 python tools/knob_sweep.py cfg4 "" 2>&1 | tail -4
timeout 1500 python tools/knob_sweep.py cfg4 "QADC_B200_TC_DEBUG=256" "QADC_B200_TC_DEBUG=2" "QADC_B200_TC_DEBUG=128" "QADC_B200_TC_DEBUG=130" "QADC_B200_TC_DEBUG=1" 2>&1 | tail -6
