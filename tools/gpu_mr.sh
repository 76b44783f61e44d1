export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests/test_bench_multirank.py -m gpu -q > gpurun_out/pytest_multirank.log 2>&1; echo rc=$? >> gpurun_out/pytest_multirank.log
