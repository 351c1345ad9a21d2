# Round-end measurement set (developer script): bench lines + launch lists.
set -x
mkdir -p gpurun_out/r1
python bench.py > gpurun_out/r1/bench_cfg1.json 2> gpurun_out/r1/bench_cfg1.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1/ref_cfg1.json 2> gpurun_out/r1/ref_cfg1.err
python bench.py --config cfg0 --steps 10 --warmup 3 > gpurun_out/r1/bench_cfg0.json 2> gpurun_out/r1/bench_cfg0.err
python bench.py --config cfg3 --steps 10 --warmup 3 > gpurun_out/r1/bench_cfg3.json 2> gpurun_out/r1/bench_cfg3.err
python bench.py --config cfg2 --steps 5 --warmup 3 --recall 200 > gpurun_out/r1/bench_cfg2.json 2> gpurun_out/r1/bench_cfg2.err
python bench.py --config cfg2 --nprobe 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1/bench_cfg2_np64.json 2> gpurun_out/r1/bench_cfg2_np64.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r1/launches_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r1/launches_cfg2.csv python bench.py --config cfg2 --n 30000000 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
tail -c 300 gpurun_out/r1/*.json
