# k_scan at cfg4: ncu --set full of one launch (current code) + bench line
O=gpurun_out/r2g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
QADC_BUILD_TIMING=1 timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_scan$" -s 2 -c 1 -o $O/scan_prmt_cfg4 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"; tail -c 1500 $O/ncu_cfg4.log
