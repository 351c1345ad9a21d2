mkdir -p gpurun_out/s8
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s8/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s8/pytest_gpu.log
tail -30 gpurun_out/s8/pytest_gpu.log
timeout 600 python tools/phase_times.py cfg1 10000000 1000 2>&1 | grep -v Warn | head -6
timeout 600 python tools/phase_times.py cfg2 100000000 10000 2>&1 | grep -v Warn | head -6
timeout 600 python tools/phase_times.py cfg0 1000000 100 2>&1 | grep -v Warn | head -5
timeout 600 python tools/phase_times.py cfg3 1000000 1000 2>&1 | grep -v Warn | head -5
