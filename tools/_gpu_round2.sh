# Round-2 measurement set (run under gpurun; outputs in gpurun_out/$TAG)
TAG=${TAG:-r2f}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log | cut -c1-200
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench cfg4 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_cfg4.json 2> $O/ref_cfg4.err; echo "ref rc=$?"
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config cfg2 --nprobe 64 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg2_np64.json 2> $O/bench_cfg2_np64.err; echo "cfg2 np64 rc=$?"
timeout 600 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "cfg1 rc=$?"
timeout 600 python bench.py --config cfg0 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg0.json 2> $O/bench_cfg0.err; echo "cfg0 rc=$?"
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3 rc=$?"
for f in $O/bench_*.json $O/ref_cfg4.json; do echo "== $f"; tail -c 300 $f; echo; done
