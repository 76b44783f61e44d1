"""Best-of-rounds kernel time per (config, variant) of a tools/gpu_ab.sh log, and whether all
variants agree on the winning key.   python tools/ab_summary.py gpurun_out/<log>"""
import collections
import re
import sys

d = collections.defaultdict(list)
best = collections.defaultdict(set)
order = []
for line in open(sys.argv[1]):
    m = re.match(r'\[(\S+) r(\d+)\] (config\d+) .*best=(\(.*?\)) .*kernel=([\d.]+)ms', line)
    if m:
        v, _, c, b, k = m.groups()
        d[(c, v)].append(float(k))
        best[c].add(b)
        if v not in order:
            order.append(v)
for c in sorted(best, key=lambda x: -len(x)):
    row = "  ".join(f"{v}:{min(d[(c, v)]):.0f}" for v in order if d[(c, v)])
    print(f"{c:9s} {row}  winners_agree={len(best[c]) == 1}")
