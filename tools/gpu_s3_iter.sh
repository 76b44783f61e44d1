# one kernel iteration: same-box A/B of side-built variants, then the GPU parity suite on the product library
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-s3}
VARIANTS="${VARIANTS}" ROUNDS=${ROUNDS:-2} CFGS="${CFGS:-52 42 2}" TAG=${TAG}_ab bash tools/gpu_ab.sh
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02_${TAG}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_pytest_gpu.log
