mkdir -p gpurun_out/r1
RX='regex:^k_(scan|select|prefix|qmax|quantize|residual_lut|probe|probe_fast|tables|count_pairs|count_codes|scan_lists|scatter_pairs|emit_items|item_class|item_offsets|item_scatter|slot_offsets|init_bounds)$'
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function --kernel-name "$RX" -c 100 --csv --log-file gpurun_out/r1/launches_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function --kernel-name "$RX" -c 100 --csv --log-file gpurun_out/r1/launches_cfg2.csv python bench.py --config cfg2 --n 30000000 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_(scan|probe_fast|residual_lut)$" -c 3 -o gpurun_out/r1/cfg2_full python tools/phase_times.py cfg2 30000000 10000 > /dev/null 2>&1
ls -la gpurun_out/r1
