O=gpurun_out/r2o; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
df -h /dev/shm /tmp | tail -2
timeout 2400 python tools/knob_sweep.py cfg4 "" "QADC_B200_RANK_BUCKETS=1" "QADC_B200_RANK_BUCKETS=1;QADC_B200_NO_HALF=1" "QADC_B200_NO_ORDER=1" "QADC_B200_RANK_BUCKETS=4" 2>&1 | tee $O/sweep.txt
timeout 900 python tools/list_stats.py cfg4 > $O/list_stats.txt 2>&1; cat $O/list_stats.txt | tail -12
