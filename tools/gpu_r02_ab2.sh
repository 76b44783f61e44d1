# round 2: A/B of the member-rate placement (registers vs shared memory) on configs 2 / 5-cap2 / 4-cap2
set -x
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-ab2}
timeout 600 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_${TAG}_base.log 2>&1
RLX_LIB=$PWD/paper_2604_23838_b200/librlx_rrs32.so timeout 600 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_${TAG}_rrs32.log 2>&1
timeout 600 python tools/gpu_probe.py 2 52 42 > gpurun_out/r02_${TAG}_base2.log 2>&1
