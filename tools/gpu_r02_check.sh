# round-2 check of HEAD: GPU parity suite, smoke, probe of configs 2 / 5-cap2 / 4-cap2
set -x
export PYTHONDONTWRITEBYTECODE=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r02_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02_smoke.log
timeout 600 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_probe_base.log 2>&1; echo rc=$? >> gpurun_out/r02_probe_base.log
