# lane-group shape sweep at configs 4/5 (cap 2) (development aid)
export PYTHONDONTWRITEBYTECODE=1
for sh in 16,4 32,2 8,8; do RLX_SHAPE=$sh timeout 200 python tools/gpu_probe.py 52 2>&1 | sed "s/^/[$sh] /" | cut -c1-24,170-460; done
for sh in 16,4 32,2; do RLX_SHAPE=$sh timeout 200 python tools/gpu_probe.py 42 2>&1 | sed "s/^/[$sh] /" | cut -c1-24,170-460; done
