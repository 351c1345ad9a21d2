O=gpurun_out/r2e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/probe_tc_dbg.py 65536 10000 64 > $O/dbg6.txt 2>&1; echo rc=$?; cat $O/dbg6.txt
timeout 300 python tools/probe_tc_dbg.py 65536 100000 1 > $O/dbg7.txt 2>&1; echo rc=$?; tail -8 $O/dbg7.txt
