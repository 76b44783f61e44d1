# source-level ncu capture of the product kernel on config 2 (first 60k serials)
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-s3p}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c2 -f \
    python tools/ncu_target.py config2 2 none 60000 > gpurun_out/r02_${TAG}_ncu_c2.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_ncu_c2.log
