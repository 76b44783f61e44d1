# A/B of side-built kernel variants (paper_2604_23838_b200/librlx_<v>.so) on one box, alternating rounds.
# A variant "v@G,WPL" runs librlx_<v>.so with RLX_SHAPE=G,WPL (lane-group shape override).
# usage: VARIANTS="p0t0 p1t1 p1t1@32,2" ROUNDS=2 CFGS="2 52 42" bash tools/gpu_ab.sh
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-ab}
for r in $(seq ${ROUNDS:-2}); do
  for v in $VARIANTS; do
    lib=${v%%@*}
    shape=""
    [ "$lib" != "$v" ] && shape=${v#*@}
    RLX_SHAPE=$shape RLX_LIB=$PWD/paper_2604_23838_b200/librlx_$lib.so timeout 900 python tools/gpu_probe.py ${CFGS:-2 52 42} 2>&1 | sed "s/^/[$v r$r] /" >> gpurun_out/r02_${TAG}.log
  done
done
