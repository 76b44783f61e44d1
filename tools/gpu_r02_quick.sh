# round 2 iteration: probe configs 2 / 5-cap2 / 4-cap2 and the GPU parity suite
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-q}
timeout 900 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_${TAG}_probe.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_probe.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02_${TAG}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_pytest_gpu.log
