O=gpurun_out/r2k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_dist.py -m gpu -x -q > $O/p1.log 2>&1; echo "dist rc=$?"; tail -3 $O/p1.log
if grep -q failed $O/p1.log; then timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_dist.py -m gpu -x -q -k list_shards > $O/san.log 2>&1; grep -A12 "Invalid" $O/san.log | head -40; fi
