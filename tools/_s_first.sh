set -x
mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/s3/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/s3/smoke.log
timeout 600 python bench.py > gpurun_out/s3/bench_cfg1.json 2> gpurun_out/s3/bench_cfg1.err; echo "bench rc=$?"
cat gpurun_out/s3/bench_cfg1.json; tail -5 gpurun_out/s3/bench_cfg1.err
