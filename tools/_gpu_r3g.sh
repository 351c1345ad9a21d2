O=gpurun_out/r3g; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "warpgroup or ivf_search_vs_oracle or cfg2" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
KNOB_COMPARE=1 timeout 1500 python tools/knob_sweep.py cfg4 "" > $O/sweep0.txt 2>&1; grep "^\[" $O/sweep0.txt | cut -c1-400
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2 rc=$?"; python -c "
import json;d=json.loads(open('$O/bench_cfg2.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['phases_ms'],d.get('parity',{}).get('vs_cpu_reference'))"
