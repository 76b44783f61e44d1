# round-2 baseline on one B200: probe configs 2 / 5-cap2 / 4-cap2, full ncu capture of the config-5 cap-2 kernel
set -x
export PYTHONDONTWRITEBYTECODE=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt 2>&1
timeout 600 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_probe_base.log 2>&1; echo rc=$? >> gpurun_out/r02_probe_base.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_base_config5cap2 -f \
    python tools/ncu_target.py config5 4 2 > gpurun_out/r02_ncu_c5.log 2>&1; echo rc=$? >> gpurun_out/r02_ncu_c5.log
