# ncu --set full of one whole config-5 cap-2 decision. NOTE: with source counters this exceeded 40 min on a 5 s launch
# (timed out, round 2); the committed evidence is the --metrics capture of the whole decision (gpu_s3_final.sh) and
# --set full of 1,000 merges (gpu_s3_prof.sh).
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-s3nf}
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:rlx_score -s 1 -c 1 -o gpurun_out/r02_${TAG}_c5full -f \
    python tools/ncu_target.py config5 4 2 > gpurun_out/r02_${TAG}_ncu.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_ncu.log
