O=gpurun_out/r3n; mkdir -p $O
KNOB_COMPARE=1 timeout 1500 python tools/knob_sweep.py cfg4 "" > $O/sweep0.txt 2>&1; grep "^\[" $O/sweep0.txt | cut -c1-400
KNOB_PROFILE=1 timeout 1500 python tools/knob_sweep.py cfg4 "QADC_B200_BOUND_PREFIX_DIV=64" "QADC_B200_BOUND_PREFIX=65536" "QADC_B200_BOUND_PREFIX=4096" > $O/sweep.txt 2>&1; grep -E "^\[|k_prefix|k_scan_tcw" $O/sweep.txt | cut -c1-160
