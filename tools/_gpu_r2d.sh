# Round-2: fused tensor-core probe tests first (short timeout), then all GPU tests, bench cfg4 + reference arm, cfg2.
TAG=${TAG:-r2d}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "probe or assign" > $O/pytest_probe.log 2>&1; echo "probe tests rc=$?"; tail -5 $O/pytest_probe.log
nvidia-smi --query-gpu=name,utilization.gpu --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_gpu.log
QADC_BUILD_TIMING=1 timeout 1500 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench rc=$?"; tail -c 4000 $O/bench_cfg4.json; tail -5 $O/bench_cfg4.err
timeout 1500 python bench.py --impl reference --steps 5 --warmup 2 > $O/ref_cfg4.json 2> $O/ref_cfg4.err; echo "ref rc=$?"; tail -c 1500 $O/ref_cfg4.json; tail -5 $O/ref_cfg4.err
timeout 900 python bench.py --config cfg2 --steps 10 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2 rc=$?"; tail -c 2500 $O/bench_cfg2.json; tail -3 $O/bench_cfg2.err
