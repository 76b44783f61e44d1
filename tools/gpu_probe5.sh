export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python tools/gpu_probe.py 52 42 > gpurun_out/probe5.log 2>&1; echo rc=$? >> gpurun_out/probe5.log
