"""p50 decision latency over the first K decisions from t=0 (SURVEY §8(d):
16 at configs 3-5), host state in -> action out through the public chooser,
one JSON line per config (bench.schedule_latency).

    python tools/p50_first16.py [K] config2 config3 config4_cap2 config5_cap2
"""
import json
import sys

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402

k = int(sys.argv[1])
for cfg in sys.argv[2:]:
    print(json.dumps(bench.schedule_latency(cfg, 0, max_decisions=k)), flush=True)
