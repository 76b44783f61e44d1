# lane-group shape sweep with the v5 kernel (development aid)
export PYTHONDONTWRITEBYTECODE=1
for sh in 8,4 16,2; do RLX_SHAPE=$sh timeout 200 python tools/gpu_probe.py 3 2>&1 | sed "s/^/[$sh] /" | cut -c1-24,170-460; done
for sh in 16,4 32,2; do RLX_SHAPE=$sh timeout 300 python tools/gpu_probe.py 52 2>&1 | sed "s/^/[$sh] /" | cut -c1-24,170-460; done
for sh in 8,2 16,1 4,4; do RLX_SHAPE=$sh timeout 200 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[$sh] /" | cut -c1-24,170-460; done
