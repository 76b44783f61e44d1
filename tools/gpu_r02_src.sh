# round 2: graphgen tests + source-level ncu of a config-5 cap-2 merge shard (1000 merges)
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-s}
timeout 900 python -m pytest tests/test_graphgen.py -m gpu -q -s > gpurun_out/r02_${TAG}_graphgen.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_graphgen.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c5m -f \
    python tools/ncu_target.py config5 4 2 32046:33046 > gpurun_out/r02_${TAG}_ncu_c5m.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_ncu_c5m.log
