# Developer script: GPU tests, bench lines, launch list and a full ncu capture
# of the scan kernel (run under gpurun; outputs in gpurun_out/$TAG).
TAG=${TAG:-r1b}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_cfg1.json 2> $O/ref_cfg1.err; echo "ref rc=$?"
RX='regex:^k_'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function --kernel-name "$RX" -c 100 --csv --log-file $O/launches_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tc2?$" -s 3 -c 1 -o $O/scan_tc_cfg1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 python bench.py --config cfg0 --steps 10 --warmup 3 > $O/bench_cfg0.json 2> $O/bench_cfg0.err; echo "cfg0 rc=$?"
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2 rc=$?"
tail -c 400 $O/*.json
ls -la $O
