O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"k_nn_rerank" -s 1 -c 1 -o $O/nn_rr python tools/probe_tc_dbg.py 65536 10000 64 > $O/ncu.log 2>&1; echo rc=$?; tail -3 $O/ncu.log
