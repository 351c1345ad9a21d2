O=gpurun_out/r2m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "opq or cfg2 or ivf or shards" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 900 python tools/phase_times.py cfg2 > $O/phase_cfg2.txt 2>&1; echo "rc=$?"; grep -v Warn $O/phase_cfg2.txt | head -8
