# lane-shape sweep of config 2 on the current kernel (same box)
export PYTHONDONTWRITEBYTECODE=1
for r in 1 2; do for sh in 4,4 8,2 16,1 2,8; do RLX_SHAPE=$sh timeout 300 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[$sh r$r] /" >> gpurun_out/r02_sh2.log; done; done
