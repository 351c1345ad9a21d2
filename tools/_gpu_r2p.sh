O=gpurun_out/r2p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"k_residual_lut|k_quantize|k_prefix|k_select" -s 4 -c 4 -o $O/tables_cfg2 python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python bench.py --config cfg0 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_cfg0.json 2> $O/bench_cfg0.err; python -c "
import json; d=json.load(open('$O/bench_cfg0.json')); print(d['ms_per_step'], d['roofline']['scan_kernel_ms'], d['phases_ms'], d['e2e']['ms_per_step'])"
