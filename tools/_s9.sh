mkdir -p gpurun_out/s9
python tools/phase_times.py cfg1 2000000 1000 2>&1 | grep -v Warn | head -4
ncu --set full --import-source on --clock-control none -k regex:k_scan_tc -s 1 -c 1 -o gpurun_out/s9/tc_cfg1 python tools/phase_times.py cfg1 2000000 1000 > gpurun_out/s9/ncu.log 2>&1
tail -3 gpurun_out/s9/ncu.log
ls -la gpurun_out/s9
