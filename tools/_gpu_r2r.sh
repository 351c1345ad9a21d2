python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python tools/knob_sweep.py cfg4 "" 2>&1 | tail -2
