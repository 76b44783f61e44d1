# round 2: threads-per-CTA variants (register budget 65536/threads) on configs 2 / 5-cap2 / 4-cap2
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-sw}
for v in "" _t384 _t256; do
  RLX_LIB=$PWD/paper_2604_23838_b200/librlx$v.so timeout 900 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_${TAG}_probe$v.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_probe$v.log
done
for c in "config2 2 none" "config3 3 3" "config4 3 2" "config5 4 2"; do
  set -- $c
  timeout 600 python tools/shard_balance.py $1 $2 $3 2 4 8 > gpurun_out/r02_shard_balance_$1.json 2> gpurun_out/r02_shard_balance_$1.log; echo rc=$? >> gpurun_out/r02_shard_balance_$1.log
done
