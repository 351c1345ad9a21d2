O=gpurun_out/r3b; mkdir -p $O
timeout 1500 python tools/knob_sweep.py cfg4 "" "QADC_B200_BOUND_EVERY=8" "QADC_B200_BOUND_EVERY=16" "QADC_B200_BOUND_EVERY=64" "QADC_B200_BOUND_PREFIX=65536" "QADC_B200_BOUND_PREFIX=4096" "QADC_B200_RANK_BUCKETS=16" "QADC_B200_RANK_BUCKETS=1" > $O/sweep.txt 2>&1; grep "^\[" $O/sweep.txt | cut -c1-200
