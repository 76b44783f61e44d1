set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_bench_multirank.py -m gpu -q -x > gpurun_out/pytest_multirank.log 2>&1; echo rc=$? >> gpurun_out/pytest_multirank.log
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active \
   --clock-control none -k regex:rlx_score -s 1 -c 1 --csv --log-file gpurun_out/ncu_traffic_cfg2.csv python tools/ncu_target.py config2 2 none > gpurun_out/ncu_traffic.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
