# Record run: default bench (cfg4) with CPU baselines + parity, the reference arm, cfg1 and cfg2 lines.
O=gpurun_out/r2n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
QADC_BUILD_TIMING=1 timeout 1800 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench rc=$?"; tail -c 600 $O/bench_cfg4.err
timeout 1800 python bench.py --impl reference --steps 5 --warmup 2 > $O/ref_cfg4.json 2> $O/ref_cfg4.err; echo "ref rc=$?"; tail -c 400 $O/ref_cfg4.err
timeout 900 python bench.py --config cfg1 --steps 10 --warmup 3 --recall 200 > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "cfg1 rc=$?"; tail -c 400 $O/bench_cfg1.err
timeout 900 python bench.py --config cfg2 --steps 10 --warmup 3 --recall 200 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2 rc=$?"; tail -c 400 $O/bench_cfg2.err
