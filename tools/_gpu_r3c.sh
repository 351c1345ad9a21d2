O=gpurun_out/r3c; mkdir -p $O
timeout 900 python tools/knob_sweep.py cfg4 "" > $O/sweep0.txt 2>&1; grep "^\[" $O/sweep0.txt | cut -c1-400
KNOB_CHILD=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tcw$" -s 2 -c 1 -o $O/scan_tcw_cfg4 python tools/knob_sweep.py cfg4 "" > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $O/ncu.log
