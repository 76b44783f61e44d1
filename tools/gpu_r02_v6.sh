# round 2 kernel check: probe, GPU parity suite, config-5 cap-2 key dump, racecheck + memcheck on small decisions
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-v6}
timeout 900 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_${TAG}_probe.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_probe.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_${TAG}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_pytest_gpu.log
timeout 600 python tools/dump_keys.py config5 4 2 gpurun_out/keys_config5_cap2.npz > gpurun_out/r02_${TAG}_dump.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_dump.log
for tool in racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py > gpurun_out/r02_${TAG}_sanitize_$tool.log 2>&1; echo rc=$? >> gpurun_out/r02_${TAG}_sanitize_$tool.log
done
