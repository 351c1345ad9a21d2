python -m pytest tests -x -q -m gpu 2>&1 | tail -2
P="python tools/phase_times.py"
$P cfg1 2>&1 | grep -E "k_scan<|total"
$P cfg0 2>&1 | grep -E "k_scan<|total"
$P cfg3 2>&1 | grep -E "k_scan<|total"
