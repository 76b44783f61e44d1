export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "golden_candidate_keys" > gpurun_out/pytest_keys.log 2>&1; echo rc=$? >> gpurun_out/pytest_keys.log
