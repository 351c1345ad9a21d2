D=gpurun_out/s20; mkdir -p $D
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tc$" -s 1 -c 1 -o $D/scan_tc_cfg1 python tools/phase_times.py cfg1 10000000 1000 > $D/ncu.log 2>&1
QADC_B200_TC_DEBUG=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tc$" -s 1 -c 1 -o $D/scan_tc_cfg1_dbg1 python tools/phase_times.py cfg1 10000000 1000 > $D/ncu_dbg1.log 2>&1
ls -la $D
