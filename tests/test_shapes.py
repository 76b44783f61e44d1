"""Every worker count the planner accepts (1..128) maps to a compiled
kernel shape (G lanes x WPL workers per lane, G*WPL >= W)."""

import re

from helpers import ROOT


def test_every_worker_count_has_a_kernel_shape():
    src = open(f"{ROOT}/paper_2604_23838_b200/csrc/rlx_kernels.cu").read()
    inst = set()
    for wpl_block in re.finditer(r"WPL == (\d+)\) \{\s*switch \(G\) \{(.*?)\}", src, re.S):
        wpl = int(wpl_block.group(1))
        for g in re.findall(r"case (\d+): return rlx_score_kernel<(\d+), (\d+)>", wpl_block.group(2)):
            assert int(g[0]) == int(g[1]) and int(g[2]) == wpl
            inst.add((int(g[0]), wpl))
    body = re.search(r"void choose_shape\(int W, int& G, int& WPL\) \{(.*?)\n\}", src, re.S).group(1)
    m = re.search(r"WPL = W <= (\d+) \? (\d+) : (\d+);", body)
    cut, small, big = (int(x) for x in m.groups())
    for W in range(1, 129):
        wpl = small if W <= cut else big
        g = 1
        while g * wpl < W:
            g *= 2
        assert (g, wpl) in inst, (W, g, wpl)
