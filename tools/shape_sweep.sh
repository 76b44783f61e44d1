export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[512] /" | cut -c1-24,170-460
RLX_THREADS=256 timeout 300 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[256] /" | cut -c1-24,170-460
RLX_THREADS=128 timeout 300 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[128] /" | cut -c1-24,170-460
