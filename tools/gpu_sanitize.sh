# NOTE: compute-sanitizer is closed on the GPU pool (round 2): runs under it left GPUs needing a reset. Kept for the record.
# compute-sanitizer memcheck / racecheck / synccheck on small decisions (outputs under gpurun_out/)
set -x
export PYTHONDONTWRITEBYTECODE=1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py > gpurun_out/sanitize_$tool.log 2>&1; echo rc=$? >> gpurun_out/sanitize_$tool.log
done
