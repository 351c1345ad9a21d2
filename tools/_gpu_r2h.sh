O=gpurun_out/r2h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python bench.py --config cfg4 --steps 5 --warmup 2 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg4.json')); print(d['ms_per_step'], d['roofline']['scan_kernel_ms'], d['roofline']['frac'], d['phases_ms'], d['workload_notes'])"
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg2.json')); print(d['ms_per_step'], d['roofline']['scan_kernel_ms'], d['roofline']['frac'], d['phases_ms'])"
