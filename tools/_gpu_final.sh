TAG=${TAG:-r2g}
O=gpurun_out/$TAG
mkdir -p $O
TAG=$TAG bash tools/_gpu_round2.sh
RX='regex:^k_(scan|nn_|residual|prefix|quantize|qmax|select|slot|emit|scatter|count|item|init|tables)'
timeout 1800 ncu --nvtx --nvtx-include "qadc_timed_region/" --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function -c 200 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan_tcw$" -s 2 -c 1 -o $O/scan_tcw_cfg4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 python bench.py --config cfg2 --recall 200 --steps 3 --warmup 3 --no-cpu-baseline > $O/recall_cfg2.json 2> $O/recall_cfg2.err; echo "recall rc=$?"
ls -la $O | head -40
