# parity at configs 4/5 (cap 2) and their bench lines
set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "first_decision" > gpurun_out/pytest_big.log 2>&1; echo rc=$? >> gpurun_out/pytest_big.log
for c in config5_cap2 config4_cap2; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --cpu-seconds 20 --no-schedule > gpurun_out/bench_$c.log 2>&1; echo rc=$? >> gpurun_out/bench_$c.log
done
