# round 2: source-level ncu captures of the scoring kernel (config 2 first 60k serials; config 5 cap 2 serials 30000-36000)
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-base}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c2 -f \
    python tools/ncu_target.py config2 2 none 60000 > gpurun_out/r02_${TAG}_ncu_c2.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_ncu_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c5 -f \
    python tools/ncu_target.py config5 4 2 30000:36000 > gpurun_out/r02_${TAG}_ncu_c5.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_ncu_c5.log
