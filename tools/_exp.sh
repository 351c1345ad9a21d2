P="python tools/phase_times.py"
for env in "X=1" "QADC_B200_NO_ORDER=1"; do
  echo "== $env"; env $env $P cfg2 30000000 10000 2>&1 | grep -E "k_scan<"
  env $env $P cfg1 2>&1 | grep -E "k_scan<"
  env $env $P cfg1 2>&1 | grep -E "k_scan<"
done
