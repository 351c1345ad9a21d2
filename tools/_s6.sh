mkdir -p gpurun_out/s6
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tools/tc_proto tools/tc_proto.cu
for nq in 32 64 128 256; do timeout 60 tools/tc_proto check 0 $nq; done > gpurun_out/s6/tc.txt 2>&1
for nq in 32 64 128 256; do timeout 60 tools/tc_proto bench 10000000 $nq; done >> gpurun_out/s6/tc.txt 2>&1
cat gpurun_out/s6/tc.txt
timeout 900 python tools/phase_times.py cfg4 100000000 10000 > gpurun_out/s6/phase_cfg4.txt 2>&1
head -8 gpurun_out/s6/phase_cfg4.txt
