# ncu of the bench workload: launch list of a short bench + full capture of one config-2 decision
set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-schedule > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/prof_bench -f \
    python tools/ncu_target.py config2 2 none > gpurun_out/ncu_full.log 2>&1
