export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/gpu_probe.py 2 3 2>&1 | sed "s/^/[shfl] /" | cut -c1-24,170-460
RLX_LIB=$PWD/paper_2604_23838_b200/librlx_smin.so timeout 300 python tools/gpu_probe.py 2 3 2>&1 | sed "s/^/[smem] /" | cut -c1-24,170-460
