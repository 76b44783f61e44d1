# round 2: graph construction tests on the device + metrics-only ncu of one full config-5 cap-2 decision
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-g}
timeout 900 python -m pytest tests/test_graphgen.py -m gpu -q -s > gpurun_out/r02_${TAG}_graphgen.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_graphgen.log
timeout 1500 ncu --metrics gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__registers_per_thread,smsp__warps_eligible.avg.per_cycle_active,launch__grid_size,launch__block_size \
    --clock-control none -k regex:rlx_score -s 1 -c 1 --csv --log-file gpurun_out/r02_${TAG}_c5full_metrics.csv \
    python tools/ncu_target.py config5 4 2 > gpurun_out/r02_${TAG}_ncu_c5full.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_ncu_c5full.log
