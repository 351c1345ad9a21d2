timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/phase_times.py cfg1 10000000 1000 2>&1 | grep -v Warn | head -5
timeout 600 python tools/phase_times.py cfg3 1000000 1000 2>&1 | grep -v Warn | head -4
timeout 600 python tools/phase_times.py cfg0 1000000 100 2>&1 | grep -v Warn | head -4
