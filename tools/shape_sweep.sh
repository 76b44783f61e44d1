# first-decision probe at configs 2-3 (development aid)
export PYTHONDONTWRITEBYTECODE=1
timeout 200 python tools/gpu_probe.py 2 3 2>&1 | cut -c1-20,160-420
