# one GPU session: probe, parity tests, bench, smoke, ncu (outputs under gpurun_out/)
set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/gpu_probe.py 1 2 3 > gpurun_out/probe.log 2>&1; echo rc=$? >> gpurun_out/probe.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 400 python tools/gpu_probe.py 5 >> gpurun_out/probe.log 2>&1; echo rc=$? >> gpurun_out/probe.log
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/prof_cfg2 -f \
    python tools/ncu_target.py config2 2 none 60000 > gpurun_out/ncu_full.log 2>&1
