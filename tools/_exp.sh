python -m pytest tests -x -q -m gpu 2>&1 | tail -2
P="python tools/phase_times.py"
$P cfg2 30000000 10000 2>&1 | grep -v Warn | head -9
