# lockstep check: a short guarded probe of the product library first, then A/B and the GPU suite
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-s3ls}
timeout 120 python tools/gpu_probe.py 42 > gpurun_out/r02_${TAG}_probe.log 2>&1; rc=$?; echo rc=$rc >> gpurun_out/r02_${TAG}_probe.log
[ $rc -ne 0 ] && exit 1
VARIANTS="${VARIANTS}" ROUNDS=${ROUNDS:-2} CFGS="${CFGS:-52 42 2}" TAG=${TAG}_ab bash tools/gpu_ab.sh
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02_${TAG}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_pytest_gpu.log
