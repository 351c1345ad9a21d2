P="python tools/phase_times.py"
for r in 17 23 29 35 47; do echo "cfg3 r=$r"; QADC_B200_RANGES=$r $P cfg3 2>&1 | grep -E "k_scan<"; done
for r in 41 65; do echo "cfg1 r=$r"; QADC_B200_RANGES=$r $P cfg1 2>&1 | grep -E "k_scan<"; done
