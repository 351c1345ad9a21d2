O=gpurun_out/r2v; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "warpgroup or ivf_search_vs_oracle" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 1500 python tools/knob_sweep.py cfg4 "QADC_B200_TC_DEBUG=1" "QADC_B200_TC_DEBUG=3" "QADC_B200_TC_DEBUG=129" "QADC_B200_TC_DEBUG=131" "QADC_B200_TC_DEBUG=257" > $O/sweep.txt 2>&1; grep "^\[" $O/sweep.txt | cut -c1-200
KNOB_CHILD=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tcw$" -s 2 -c 1 -o $O/scan_tcw_cfg4 python tools/knob_sweep.py cfg4 "" > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $O/ncu.log
