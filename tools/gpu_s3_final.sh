# round 2 measurement session of the current kernel: GPU suite, smoke, bench (both arms), p50 over the first
# 16 decisions, ncu launch list of the bench, ncu metrics of one full config-5 cap-2 decision
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-s3fin}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_${TAG}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r02_${TAG}_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_${TAG}_bench.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_${TAG}_bench_ref.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_bench_ref.log
timeout 900 python tools/p50_first16.py 16 config2 config3 config4_cap2 config5_cap2 > gpurun_out/r02_${TAG}_p50.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_p50.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-schedule --e2e-steps 1 > gpurun_out/r02_${TAG}_bench_under_ncu.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__registers_per_thread,smsp__warps_eligible.avg.per_cycle_active \
    --clock-control none -k regex:rlx_score -s 1 -c 1 --csv --log-file gpurun_out/r02_${TAG}_c5full_metrics.csv \
    python tools/ncu_target.py config5 4 2 > gpurun_out/r02_${TAG}_ncu_c5full.log 2>&1
# (compute-sanitizer is closed on the GPU pool since this session: runs under it left GPUs needing a reset;
#  the last sanitizer logs are profiles/r02_sanitize_*.txt)
