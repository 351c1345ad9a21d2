python -m pytest tests -x -q -m gpu 2>&1 | tail -2
P="python tools/phase_times.py"
$P cfg2 30000000 10000 2>&1 | grep -E "k_scan<"
QADC_B200_LINEAR=1 $P cfg2 30000000 10000 2>&1 | grep -E "k_scan<"
$P cfg1 2>&1 | grep -E "k_scan<"
$P cfg3 2>&1 | grep -E "k_scan<"
$P cfg0 2>&1 | grep -E "k_scan<"
