# A/B of side-built variants, then a source-level ncu capture of the product kernel on 1,000 config-5 cap-2 merges
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-s3p}
if [ -n "$VARIANTS" ]; then VARIANTS="${VARIANTS}" ROUNDS=${ROUNDS:-2} CFGS="${CFGS:-52 42 2}" TAG=${TAG}_ab bash tools/gpu_ab.sh; fi
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c5m -f \
    python tools/ncu_target.py config5 4 2 32046:33046 > gpurun_out/r02_${TAG}_ncu_c5m.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_ncu_c5m.log
