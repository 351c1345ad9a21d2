# Round-2 baseline: GPU tests, cfg4/cfg2 phase times, ncu --set full of the PRMT scan at cfg4 + cfg2.
TAG=${TAG:-r2a}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
lscpu > $O/lscpu.txt 2>&1; python -c "import numpy; numpy.show_config()" > $O/numpy_config.txt 2>&1
QADC_BUILD_TIMING=1 timeout 1200 python tools/phase_times.py cfg4 > $O/phase_cfg4.txt 2>&1; echo "phase cfg4 rc=$?"; cat $O/phase_cfg4.txt | head -40
timeout 600 python tools/phase_times.py cfg2 > $O/phase_cfg2.txt 2>&1; echo "phase cfg2 rc=$?"; head -30 $O/phase_cfg2.txt
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan$" -s 2 -c 1 -o $O/scan_prmt_cfg4 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"; tail -3 $O/ncu_cfg4.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan$" -s 2 -c 1 -o $O/scan_prmt_cfg2 python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_cfg2.log 2>&1; echo "ncu cfg2 rc=$?"; tail -3 $O/ncu_cfg2.log
ls -la $O
