# lane-group shape sweep of the first decision (development aid)
export PYTHONDONTWRITEBYTECODE=1
for sh in 2,8 4,4 8,4 4,8; do RLX_SHAPE=$sh timeout 120 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[$sh] /" | cut -c1-330; done
for sh in 8,4 4,8 16,4; do RLX_SHAPE=$sh timeout 120 python tools/gpu_probe.py 3 2>&1 | sed "s/^/[$sh] /" | cut -c1-330; done
