# occupancy sweep (development aid)
export PYTHONDONTWRITEBYTECODE=1
D=$PWD/paper_2604_23838_b200
timeout 120 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[t512] /" | cut -c1-20,160-420
for t in 640 768; do RLX_LIB=$D/librlx_t$t.so timeout 120 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[t$t] /" | cut -c1-20,160-420; done
for t in 640 768; do RLX_LIB=$D/librlx_t$t.so RLX_SHAPE=16,2 timeout 120 python tools/gpu_probe.py 3 2>&1 | sed "s/^/[t$t 16,2] /" | cut -c1-24,160-420; done
