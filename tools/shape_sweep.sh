export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/gpu_probe.py 2 3 52 2>&1 | cut -c1-24,170-460
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize_target.py 2>&1 | tail -3
