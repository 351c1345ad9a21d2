O=gpurun_out/r3j; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "warpgroup or ivf_search_vs_oracle or cfg2 or opq" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config cfg2 --nprobe 64 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg2_np64.json 2> $O/bench_cfg2_np64.err; echo "cfg2 np64 rc=$?"
QADC_B200_TCW_WIDE_PAIRS=100000 timeout 900 python bench.py --config cfg2 --nprobe 64 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg2_np64_narrow.json 2> $O/bench_cfg2_np64_narrow.err; echo "cfg2 np64 narrow rc=$?"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r3j/bench_*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
    print(f.split('/')[-1], 'ms %.2f'%d['ms_per_step'], 'scan', r['scan_kernel_ms'], r.get('list_passes'), r.get('roof_ms'), d.get('parity',{}).get('vs_cpu_reference'))
PY
KNOB_COMPARE=1 timeout 1500 python tools/knob_sweep.py cfg4 "" > $O/sweep0.txt 2>&1; grep "^\[" $O/sweep0.txt | cut -c1-400
