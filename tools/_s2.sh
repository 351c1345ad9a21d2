mkdir -p gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s2/smoke.log
timeout 600 python bench.py > gpurun_out/s2/bench_cfg1.json 2> gpurun_out/s2/bench_cfg1.err
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2/bench_cfg2.json 2> gpurun_out/s2/bench_cfg2.err
tail -c 400 gpurun_out/s2/pytest_gpu.log gpurun_out/s2/smoke.log
cat gpurun_out/s2/bench_cfg1.json gpurun_out/s2/bench_cfg2.json
