# round 2: A/B of run-time knobs (pass-queue order, lane shape) on configs 2 / 5-cap2 / 4-cap2
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-ab}
timeout 600 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_${TAG}_base.log 2>&1
RLX_PASS_ORDER=1 timeout 600 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_${TAG}_order1.log 2>&1
RLX_SHAPE=32,2 timeout 600 python tools/gpu_probe.py 52 42 > gpurun_out/r02_${TAG}_shape32x2.log 2>&1
RLX_SHAPE=4,4 timeout 600 python tools/gpu_probe.py 2 > gpurun_out/r02_${TAG}_shape4x4.log 2>&1
RLX_SHAPE=16,1 timeout 600 python tools/gpu_probe.py 2 > gpurun_out/r02_${TAG}_shape16x1.log 2>&1
