# one GPU session: parity tests, probe, bench, smoke, ncu launch list + full capture of the bench workload
set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/gpu_probe.py 1 2 3 > gpurun_out/probe.log 2>&1; echo rc=$? >> gpurun_out/probe.log
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 15 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 --cpu-seconds 20 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/prof_bench -f \
    python tools/ncu_target.py config2 2 none > gpurun_out/ncu_full.log 2>&1
