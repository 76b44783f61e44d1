"""Per-function instruction / stall breakdown of an ncu source page (development aid).

    ncu -i rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [--lines]
"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
data = []
hdr = None
fname = None
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        ix = hdr.index('Instructions Executed')
        ws = hdr.index('Warp Stall Sampling (All Samples)')
        th = hdr.index('Thread Instructions Executed')
        continue
    if r[0] == 'Function Name' or hdr is None:
        continue
    try:
        data.append((int(r[ix] or 0), int(r[ws] or 0), int(r[th] or 0), fname, int(r[0]), r[1][:100]))
    except ValueError:
        pass
src = open(next((a.split('=',1)[1] for a in sys.argv if a.startswith('--src=')), 'paper_2604_23838_b200/csrc/rlx_kernels.cu')).read().split('\n')
ranges = []
for i, l in enumerate(src, 1):
    m = re.match(r'\s*RLX_HD .*?(\w+)\(', l)
    if m:
        ranges.append((i, m.group(1)))


def fn_of(line):
    name = '?'
    for st, n in ranges:
        if st <= line:
            name = n
        else:
            break
    return name


agg = {}
for ins, ws, th, f, ln, s in data:
    key = fn_of(ln) if f == 'rlx_kernels.cu' else f
    a = agg.setdefault(key, [0, 0, 0])
    a[0] += ins
    a[1] += ws
    a[2] += th
tot = sum(v[0] for v in agg.values())
tots = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{k:22s} inst {v[0] / tot * 100:5.1f}%  stall {v[1] / tots * 100:5.1f}%  thr/inst {v[2] / max(v[0], 1):5.1f}")
if '--lines' in sys.argv:
    print('--- top lines')
    for d in sorted(data, reverse=True)[:40]:
        print(f"{d[0] / tot * 100:5.1f}% {d[1] / tots * 100:5.1f}% thr {d[2] / max(d[0], 1):4.1f} {d[3]}:{d[4]} {d[5]}")
