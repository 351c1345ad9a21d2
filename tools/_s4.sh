mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/pytest_gpu.log
tail -5 gpurun_out/s4/pytest_gpu.log
timeout 600 python tools/phase_times.py cfg2 100000000 10000 > gpurun_out/s4/phase_cfg2.txt 2>&1
head -6 gpurun_out/s4/phase_cfg2.txt
timeout 1200 python bench.py --config cfg4 --n 100000000 --steps 3 --warmup 3 --cpu-seconds 8 > gpurun_out/s4/bench_cfg4_n1e8.json 2> gpurun_out/s4/bench_cfg4_n1e8.err
cat gpurun_out/s4/bench_cfg4_n1e8.json; tail -5 gpurun_out/s4/bench_cfg4_n1e8.err
