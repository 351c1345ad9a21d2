# Developer script: scan-time experiments (QADC_B200_TC_DEBUG bits make results invalid when != 0).
# usage: RUNS="VAR=val,VAR2=val ..." bash tools/_gpu_dbg.sh   (one bench run per space-separated entry)
for r in ${RUNS:-QADC_B200_TC_DEBUG=0}; do
  env ${r//,/ } timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3 ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$r', 'scan_ms', d['roofline']['scan_kernel_ms'], 'step', round(d['ms_per_step'],3), 'cands', round(d['candidates_per_query'],1), 'launches', d['gpu_launches'])"
done
