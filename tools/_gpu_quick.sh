# Developer script: GPU parity tests + one cfg1 bench line (gpurun_out/$TAG).
TAG=${TAG:-q}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); r=d['roofline']
print('value %.4g ms/step %.3f scan_ms %s frac %s e2e %.4g' % (d['value'], d['ms_per_step'], r['scan_kernel_ms'], r['frac'], d['e2e']['value']))"
tail -5 $O/bench_cfg1.err
