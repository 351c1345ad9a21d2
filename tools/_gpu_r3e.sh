O=gpurun_out/r3e; mkdir -p $O
KNOB_PROFILE=1 timeout 1500 python tools/knob_sweep.py cfg4 "" > $O/sweep0.txt 2>&1; cat $O/sweep0.txt | cut -c1-200 | tail -30
