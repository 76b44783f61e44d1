# round 2: source-level ncu captures (config 2 first 60k serials; config 5 cap 2 serials 31500-32300), racecheck, short bench
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-v6}
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_target.py > gpurun_out/r02_${TAG}_sanitize_racecheck.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_sanitize_racecheck.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c2 -f \
    python tools/ncu_target.py config2 2 none 60000 > gpurun_out/r02_${TAG}_ncu_c2.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_ncu_c2.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c5 -f \
    python tools/ncu_target.py config5 4 2 31500:32300 > gpurun_out/r02_${TAG}_ncu_c5.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_ncu_c5.log
timeout 1500 python bench.py --steps 3 --warmup 3 --cpu-seconds 30 > gpurun_out/r02_${TAG}_bench.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_bench.log
