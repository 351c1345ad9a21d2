for S in 16 8 5 3; do echo "slices<=$S"; QADC_B200_PROBE_SLICES=$S timeout 120 python tools/probe_tc_dbg.py 65536 10000 64 2>&1 | grep -E "k_nn_tc|rerank|mismatch|candidates"; done
