O=gpurun_out/r3d; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "warpgroup or ivf_search_vs_oracle or tensor_core_scan" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
KNOB_COMPARE=1 timeout 1500 python tools/knob_sweep.py cfg4 "" > $O/sweep0.txt 2>&1; grep "^\[" $O/sweep0.txt | cut -c1-400
