"""Quick GPU probe: first-decision timing per config (development aid)."""
import sys
import time

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from helpers import instance  # noqa: E402
from paper_2604_23838_b200.state import State as HostState  # noqa: E402
from paper_2604_23838_b200.native import Evaluator  # noqa: E402

CFG = {1: (1, None), 2: (2, None), 3: (3, 3), 4: (3, 3), 5: (4, 3), 52: (4, 2), 42: (3, 2)}
which = [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5]
for k in which:
    w, cap = CFG[k]
    inst = instance(f"config{str(k)[0]}")
    ev = Evaluator(inst)
    st = HostState(inst)
    t = time.time()
    d = ev.decide(st, w, cap)
    t1 = time.time() - t
    t = time.time()
    d = ev.decide(st, w, cap)
    t2 = time.time() - t
    print(f"config{k} W={w} cap={cap}: n={d.n_candidates} (mux {d.n_multiplex} merge {d.n_merge} excl {d.n_exclusive})"
          f" best=({d.cost!r}, {d.finish!r}, {d.priority}, {d.serial}) passes={d.passes} bytes={d.alg_bytes:.3e}"
          f" kernel={d.kernel_ms:.2f}ms plan={d.plan_ms:.2f}ms wall1={t1*1e3:.1f}ms wall2={t2*1e3:.1f}ms"
          f" cand/s={d.n_candidates/(d.kernel_ms/1e3):.3e} GB/s={d.alg_bytes/(d.kernel_ms/1e3)/1e9:.1f}"
          f" events={d.events} ev/pass={d.events/max(d.passes,1):.1f} ev/s={d.events/(d.kernel_ms/1e3):.3e}", flush=True)
