set -x
export PYTHONDONTWRITEBYTECODE=1
RLX_LIB=$PWD/paper_2604_23838_b200/librlx_dbg.so timeout 300 python tools/dbg_shapes.py config3 > gpurun_out/dbg_shapes.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
