O=gpurun_out/r3k; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 1500 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_short.json 2> $O/bench_short.err; echo "bench rc=$?"
timeout 1800 ncu --nvtx --nvtx-include "qadc_timed_region/" --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function -c 200 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?"; tail -2 $O/ncu_launch.log | cut -c1-200
wc -l $O/launches_cfg4.csv
