# lane-group shape sweep of the first decision (development aid)
export PYTHONDONTWRITEBYTECODE=1
for sh in 4,4 8,4; do RLX_SHAPE=$sh timeout 120 python tools/gpu_probe.py 2 2>&1 | sed "s/^/[$sh] /" | cut -c1-20,160-420; done
for sh in 8,4 16,4; do RLX_SHAPE=$sh timeout 120 python tools/gpu_probe.py 3 2>&1 | sed "s/^/[$sh] /" | cut -c1-20,160-420; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/prof_cfg2_v5 -f \
    python tools/ncu_target.py config2 2 none 60000 > gpurun_out/ncu_full.log 2>&1
