export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/gpu_probe.py 2 3 52 2>&1 | cut -c1-24,170-460
