# Round-2 profiles of the headline config (run after bench.py exited 0 without ncu)
O=gpurun_out/${TAG:-r2p}; mkdir -p $O
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_short.json 2> $O/bench_cfg4_short.err; echo "bench rc=$?"
RX='regex:^k_(scan|nn_|residual|prefix|quantize|qmax|select|slot|emit|scatter|count|item|init|tables)'
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function --kernel-name "$RX" -c 120 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tcw$" -s 2 -c 1 -o $O/scan_tcw_cfg4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -c 600 $O/bench_cfg4_short.json; ls -la $O
