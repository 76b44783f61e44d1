set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/prof_cfg2_v6 -f \
    python tools/ncu_target.py config2 2 none 60000 > gpurun_out/ncu_full.log 2>&1
