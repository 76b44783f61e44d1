export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[all groups] /" | cut -c1-30,170-460
RLX_DIAG_ONE_GROUP=1 timeout 300 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[1 group\/warp] /" | cut -c1-30,170-460
RLX_SHAPE=16,1 timeout 300 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[16x1 all] /" | cut -c1-30,170-460
RLX_SHAPE=16,1 RLX_DIAG_ONE_GROUP=1 timeout 300 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[16x1 1 grp] /" | cut -c1-30,170-460
