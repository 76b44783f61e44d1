set -x
export PYTHONDONTWRITEBYTECODE=1
bash tools/shape_sweep.sh > gpurun_out/sweep.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
