# round 2: lane-shape sweep with the per-warp pass queue (G lanes x WPL workers per lane)
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-sh}
for sh in 8,2 4,4 2,8 16,1; do RLX_SHAPE=$sh timeout 300 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[$sh] /" >> gpurun_out/r02_${TAG}_c2.log; done
for sh in 16,4 8,8; do RLX_SHAPE=$sh timeout 600 python tools/gpu_probe.py 52 42 2>&1 | sed "s/^/[$sh] /" >> gpurun_out/r02_${TAG}_c5.log; done
