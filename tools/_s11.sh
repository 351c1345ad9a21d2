set -x
D=gpurun_out/s11; mkdir -p $D
timeout 300 python bench.py --config cfg0 --steps 10 --warmup 3 > $D/bench_cfg0.json 2> $D/bench_cfg0.err
timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 > $D/bench_cfg3.json 2> $D/bench_cfg3.err
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 > $D/bench_cfg2.json 2> $D/bench_cfg2.err
timeout 600 python bench.py --config cfg2 --nprobe 64 --steps 3 --warmup 3 --no-cpu-baseline > $D/bench_cfg2_np64.json 2> $D/bench_cfg2_np64.err
timeout 900 python bench.py --config cfg4 --n 125000000 --steps 3 --warmup 3 --cpu-seconds 8 > $D/bench_cfg4.json 2> $D/bench_cfg4.err
RX='regex:^k_'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function --kernel-name "$RX" -c 100 --csv --log-file $D/launches_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tc$" -s 1 -c 1 -o $D/scan_tc_cfg1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $D/ncu_full.log 2>&1
tail -c 400 $D/*.json
ls -la $D
