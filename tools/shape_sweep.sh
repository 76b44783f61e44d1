# lane-group shape sweep of the first decision (development aid)
export PYTHONDONTWRITEBYTECODE=1
MB=$PWD/paper_2604_23838_b200/librlx_mb2.so
for sh in 16,1 8,2; do RLX_LIB=$MB RLX_SHAPE=$sh timeout 120 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[mb2 $sh] /" | cut -c1-24,160-420; done
for sh in 32,1 16,2; do RLX_LIB=$MB RLX_SHAPE=$sh timeout 120 python tools/gpu_probe.py 3 2>&1 | sed "s/^/[mb2 $sh] /" | cut -c1-24,160-420; done
for sh in 32,2 16,4; do RLX_LIB=$MB RLX_SHAPE=$sh timeout 300 python tools/gpu_probe.py 4 2>&1 | sed "s/^/[mb2 $sh] /" | cut -c1-24,160-420; done
