mkdir -p gpurun_out/s7
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s7/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s7/pytest_gpu.log
tail -30 gpurun_out/s7/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python tools/phase_times.py cfg1 10000000 1000 2>&1 | head -8
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s7/bench_cfg1.json 2> gpurun_out/s7/bench_cfg1.err; cat gpurun_out/s7/bench_cfg1.json; tail -3 gpurun_out/s7/bench_cfg1.err
