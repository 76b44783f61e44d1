"""Static SASS size per source function of one kernel (development aid).

    nvdisasm -g -c <cubin> > all.sass; python tools/sass_size.py all.sass <kernel-substring>
"""
import collections
import re
import sys

txt = open(sys.argv[1]).read()
key = sys.argv[2]
i = txt.index(key + ':')
j = txt.find('.section', i)
body = txt[i:j if j > 0 else None].split('\n')
cur = None
cnt = collections.Counter()
for l in body:
    m = re.search(r'//## File ".*?/([\w.]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/', l) and cur:
        cnt[cur] += 1
src = open('paper_2604_23838_b200/csrc/rlx_kernels.cu').read().split('\n')
ranges = []
for i2, l in enumerate(src, 1):
    m = re.match(r'\s*(?:RLX_HD|RLX_NI|__device__|__global__).*?(\w+)\(', l)
    if m:
        ranges.append((i2, m.group(1)))


def fn(f, ln):
    if f != 'rlx_kernels.cu':
        return f
    name = '?'
    for st, n in ranges:
        if st <= ln:
            name = n
        else:
            break
    return name


agg = collections.Counter()
for (f, ln), c in cnt.items():
    agg[fn(f, ln)] += c
print('total', sum(cnt.values()))
for k, v in agg.most_common(30):
    print(f"{v:6d} {k}")
