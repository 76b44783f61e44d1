# p50 decision latency over the first 16 decisions (configs 2, 3) and a full config-1 schedule
set -x
export PYTHONDONTWRITEBYTECODE=1
for c in config2 config3; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --schedule-config $c --schedule-decisions 16 > gpurun_out/sched_$c.log 2>&1; echo rc=$? >> gpurun_out/sched_$c.log
done
