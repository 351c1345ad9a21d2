# Round-2: cfg4 coarse quantizer (GPU Lloyd, K=65536), encoder speed, k_scan QT experiments at cfg4.
TAG=${TAG:-r2b}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python tools/train_coarse.py --K 65536 --n 2097152 --iters 10 --out $O/cfg4_coarse_K65536.npy > $O/train_coarse.log 2>&1; echo "train rc=$?"; tail -3 $O/train_coarse.log
QADC_BUILD_TIMING=1 QADC_B200_VARIANT_STATS=1 timeout 900 python tools/phase_times.py cfg4 > $O/phase_cfg4.txt 2>&1; echo "phase rc=$?"; head -12 $O/phase_cfg4.txt
QADC_B200_QT=16 QADC_B200_VARIANT_STATS=1 timeout 900 python bench.py --config cfg4 --steps 5 --warmup 2 --no-cpu-baseline > $O/bench_cfg4_qt16.json 2> $O/bench_cfg4_qt16.err; echo "qt16 rc=$?"; tail -c 1500 $O/bench_cfg4_qt16.json; tail -3 $O/bench_cfg4_qt16.err
