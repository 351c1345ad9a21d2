P="python tools/phase_times.py"
for rb in 1 2 4 16; do echo "rb=$rb"; QADC_B200_RANK_BUCKETS=$rb $P cfg2 30000000 10000 2>&1 | grep -E "k_scan<"; done
QADC_B200_VARIANT_STATS=1 QADC_B200_RANK_BUCKETS=1 python bench.py --config cfg2 --n 30000000 --queries 10000 --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep "qadc_b200" | tail -2
