D=gpurun_out/s15; mkdir -p $D
for dbg in 0 1 2 4 7; do
QADC_B200_TC_DEBUG=$dbg timeout 300 python tools/phase_times.py cfg1 10000000 1000 2>&1 | grep -m1 "k_scan_tc" | sed "s/^/dbg=$dbg /"
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tc$" -s 1 -c 1 -o $D/scan_tc_g4 python tools/phase_times.py cfg1 10000000 1000 > $D/ncu.log 2>&1
tail -2 $D/ncu.log
