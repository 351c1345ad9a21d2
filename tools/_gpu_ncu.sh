# Developer script: one full ncu capture of the TC scan kernel at cfg1 (gpurun_out/$TAG).
TAG=${TAG:-n}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tc2?$" -s 3 -c 1 -o $O/scan_tc_cfg1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 $O/ncu_full.log
