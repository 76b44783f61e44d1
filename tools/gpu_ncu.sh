# ncu capture of the scoring kernel (one GPU): launch list of a short bench + full set on config2 cap 3
set -x
export PYTHONDONTWRITEBYTECODE=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/prof_cfg2cap3 -f \
    python tools/ncu_target.py config2 2 3 > gpurun_out/ncu_full.log 2>&1
