O=gpurun_out/r2q; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "opq or cfg2 or ivf or tables or flat" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 600 python tools/phase_times.py cfg2 > $O/phase_cfg2.txt 2>&1; grep -v Warn $O/phase_cfg2.txt | sed -n 3,8p
timeout 1200 python tools/knob_sweep.py cfg4 "" 2>&1 | tail -2
