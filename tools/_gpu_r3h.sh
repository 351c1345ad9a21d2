O=gpurun_out/r3h; mkdir -p $O
timeout 600 python tools/phase_times.py cfg0 > $O/phase_cfg0.txt 2>&1; grep -v Warn $O/phase_cfg0.txt | tail -32 | cut -c1-150
timeout 600 python tools/host_overhead.py > $O/host.txt 2>&1; tail -5 $O/host.txt | cut -c1-200
