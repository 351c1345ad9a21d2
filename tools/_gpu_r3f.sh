O=gpurun_out/r3f; mkdir -p $O
timeout 1500 python tools/knob_sweep.py cfg4 "QADC_B200_TC_DEBUG=1" "QADC_B200_TC_DEBUG=513" "QADC_B200_TC_DEBUG=1025" "QADC_B200_TC_DEBUG=3" "QADC_B200_TC_DEBUG=129" > $O/sweep.txt 2>&1; grep "^\[" $O/sweep.txt | cut -c1-200
