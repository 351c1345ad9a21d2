O=gpurun_out/r2l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python tools/phase_times.py cfg4 > $O/phase_cfg4.txt 2>&1; echo "rc=$?"; grep -v Warn $O/phase_cfg4.txt | head -12
