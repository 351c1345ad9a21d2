mkdir -p gpurun_out/s5
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tools/tc_proto tools/tc_proto.cu
timeout 120 tools/tc_proto check > gpurun_out/s5/tc_check.txt 2>&1; echo "rc=$?" >> gpurun_out/s5/tc_check.txt
cat gpurun_out/s5/tc_check.txt
timeout 120 tools/tc_proto bench 10000000 > gpurun_out/s5/tc_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/s5/tc_bench.txt
cat gpurun_out/s5/tc_bench.txt
timeout 900 python -X importtime -c "pass" 2>/dev/null
timeout 900 python tools/phase_times.py cfg4 100000000 10000 > gpurun_out/s5/phase_cfg4.txt 2>&1
head -14 gpurun_out/s5/phase_cfg4.txt
