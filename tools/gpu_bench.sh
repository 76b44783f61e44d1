# bench + reference arm + smoke only
set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 15 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 --cpu-seconds 20 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
timeout 900 python -m pytest tests/test_bench_multirank.py -m gpu -q > gpurun_out/pytest_multirank.log 2>&1; echo rc=$? >> gpurun_out/pytest_multirank.log
