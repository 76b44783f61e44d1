# source-level ncu of the current kernel: config 2 (first 60k serials), config 5 cap 2 (1,000 merges)
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-s2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c2 -f \
    python tools/ncu_target.py config2 2 none 60000 > gpurun_out/r02_${TAG}_ncu_c2.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c5m -f \
    python tools/ncu_target.py config5 4 2 32046:33046 > gpurun_out/r02_${TAG}_ncu_c5m.log 2>&1
