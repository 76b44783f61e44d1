"""Benchmark of the B200 look-ahead chooser (the north-star hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config config5_cap2] [--impl ours|reference]

A *step* is one look-ahead decision: every candidate of the decision state
(enumerate_actions, rlmux/scheduler.py:648-703) is scored by the W-round
list-scheduling simulation (candidate_cost + action_finish_estimate,
:773-918) and the (cost, finish, priority, serial) argmin is taken
(:963-972). The workload is the FIRST decision of the named config
(tests/golden/instances/<config>.json.gz, built with the reference's own
generator). Default: config 5 (BASELINE.json configs[4]:
8 pipelines, 64 simulated GPUs, 64k rollouts, depth 4) with merge sets
capped at 2 members — the largest decision that completes in the
reference: at cap 3 the reference itself raises SchedulingError on serial
819010 (a livelocking merge follow-up; tests/golden/livelock.json), which
the device reproduces. 64,814 candidates (32,046 multiplex, 32,256 merges,
512 exclusive), ~10.3M list-scheduling passes, ~1.2e10 simulated events.

Reported (one JSON line on rank 0):
  value      candidates evaluated / s, whole job, plan resident in HBM
             (RLX_F_REUSE_PLAN: scoring kernel + argmin + cross-GPU min-loc),
             CUDA events on the launching stream, max over ranks
  e2e        the same metric through the public chooser (the `_drive` seam):
             host state -> plan -> H2D -> kernel -> D2H -> action
  roofline   SURVEY §8(d) algorithmic bytes of the scoring kernel per launch
             / its CUDA-event duration, against the measured HBM copy peak
  cpu_baseline  the CPU port of the reference chooser (oracle/rlx_oracle.c,
             all host threads), class-stratified sample of the same decision
             with a fixed budget (--cpu-seconds), extrapolated to the decision

With N>1 (torchrun, NCCL) the serial range is split into N cost-balanced
shards and the shard winners meet in ONE all-reduce per decision
(paper_2604_23838_b200/dist.py): strong scaling (the decision is fixed).

`--impl reference` times the reference algorithm on the host cores (rank 0
only): the C restatement in oracle/ (the reference is pure Python with no
native build; the port is ~100x faster per candidate than the Python, so
it is the stricter baseline), plus the unmodified Python reference itself
(rlmux installed into baseline/_ref) on a non-merge sample, forked over all
cores, reported as `python_reference` with its keys checked against the port.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (window, max_merge, description)
    "config1": (1, None, "sync GRPO, 1 Qwen3-8B-shaped pipeline, 8 simulated GPUs, 256 rollouts, depth 1"),
    "config2": (2, None, "2 multiplexed sync pipelines (8B+14B), 16 simulated GPUs, 1024 rollouts, depth 2, "
                         "long-tail migration, uncapped merges"),
    "config3": (3, 3, "async RL 4 pipelines, 32 simulated GPUs, 4096 heavy-tailed rollouts, depth 3, merge cap 3"),
    "config5": (4, 3, "8 pipelines, 64 simulated GPUs, 64k rollouts, depth 4, merge cap 3"),
    # the reference itself raises SchedulingError at the cap-3 first decision
    # of configs 4 and 5 (a livelocking merge follow-up, tests/golden/livelock.json);
    # cap 2 removes those merges and gives the largest decisions that complete
    "config4_cap2": (3, 2, "4 agentic pipelines (tool waits), 64 simulated GPUs, 16k rollouts, depth 3, merge cap 2"),
    "config5_cap2": (4, 2, "8 pipelines, 64 simulated GPUs, 64k rollouts, depth 4, merge cap 2"),
}
METRIC = "look-ahead candidates evaluated/sec & p50 decision latency at 1/2/4/8 B200"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def load_instance(name):
    from paper_2604_23838_b200 import load_instance as li

    return li(os.path.join(ROOT, "tests", "golden", "instances", f"{name.split('_')[0]}.json.gz"))


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_record(config):
    """(dram read+write bytes per scoring launch, issue summary) from the
    committed ncu capture of this workload (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(config), d.get("issue", {}).get(config)
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def class_ranges(n_mux, n_merge, n_excl):
    """Serial ranges of the three candidate classes (enumerate_actions order:
    multiplex, merges, exclusive; scheduler.py:648-703)."""
    return {"multiplex": (0, n_mux), "merge": (n_mux, n_mux + n_merge),
            "exclusive": (n_mux + n_merge, n_mux + n_merge + n_excl)}


# share of the CPU budget per class (merges cost 3(1+F) passes, the others 3)
_CLASS_SHARE = {"merge": 0.75, "multiplex": 0.2, "exclusive": 0.05}


def cpu_stratified(inst, state, window, cap, counts, seconds, seed=0):
    """Class-stratified timing of the CPU port (oracle/rlx_oracle.c) on every
    host thread, with a fixed budget of `seconds` that does not depend on
    --steps. Per class: batches of uniformly drawn candidates (a multiple of
    the thread count, doubling while the budget allows); the class's wall
    time per candidate t_c includes batch stragglers, as a real parallel CPU
    chooser pays them. The decision estimate is sum_c n_c * t_c, so
    rate = n_total / that (extrapolated from the sample)."""
    import numpy as np

    from oracle.oracle import Oracle

    threads = os.cpu_count() or 1
    o = Oracle(inst, nthreads=threads)
    rng = np.random.default_rng(seed)
    ranges = class_ranges(*counts)
    live = {c: r for c, r in ranges.items() if r[1] > r[0]}
    share = sum(_CLASS_SHARE[c] for c in live)
    per_class = {}
    est = 0.0
    for c, (lo, hi) in live.items():
        budget = seconds * _CLASS_SHARE[c] / share
        n_c = hi - lo
        pool = rng.permutation(n_c)[: 1 << 20] + lo if n_c <= 8 << 20 else rng.choice(n_c, 1 << 20) + lo
        used, wall, batch, last = 0, 0.0, threads, 0.0
        while used < len(pool) and (used == 0 or wall + 2 * last <= budget):
            part = np.sort(pool[used:used + batch])
            t = time.perf_counter()
            o.score(state, window, cap, serials=part, want_keys=True)
            last = time.perf_counter() - t
            wall += last
            used += len(part)
            batch = min(batch * 2, 64 * threads)
        t_c = wall / used
        per_class[c] = {"candidates": n_c, "sampled": used, "wall_s": wall, "wall_s_per_candidate": t_c}
        est += n_c * t_c
    n_total = sum(counts)
    return {"rate": n_total / est, "decision_s": est, "threads": threads, "classes": per_class,
            "sampled": sum(v["sampled"] for v in per_class.values()),
            "wall_s": sum(v["wall_s"] for v in per_class.values())}


def cpu_baseline_record(r, n_total, kind="port"):
    parts = ", ".join(f"{c} {v['sampled']}/{v['candidates']} ({v['wall_s_per_candidate'] * 1e3:.3g} ms/cand wall)"
                      for c, v in r["classes"].items())
    return {"value": r["rate"], "unit": "candidates/s", "cores": r["threads"], "kind": kind,
            "sample": f"class-stratified sample of the {n_total}-candidate decision ({parts}), scored by "
                      f"oracle/rlx_oracle.c on {r['threads']} host threads in {r['wall_s']:.1f} s ({cpu_model()}); "
                      f"value = n_total / sum_c n_c * t_c (extrapolated decision time {r['decision_s']:.1f} s)"}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


_PYREF = {}


def _pyref_init(inst, window):
    import rlmux.scheduler as rsch

    from paper_2604_23838_b200.instance_io import to_reference

    ri = to_reference(inst)
    _PYREF.update(inst=ri, state=rsch.ExecState(ri), window=window, mod=rsch)


def _pyref_score(action_json):
    """The reference chooser's work for one non-merge candidate
    (scheduler.py:963-972: candidate_cost + action_finish_estimate)."""
    from paper_2604_23838_b200.instance_io import action_as, action_from_json

    rsch = _PYREF["mod"]
    a = action_as(action_from_json(action_json), rsch)
    t = time.perf_counter()
    cost = rsch.candidate_cost(_PYREF["state"], a, _PYREF["window"])
    fin = rsch.action_finish_estimate(_PYREF["state"], a)
    return time.perf_counter() - t, cost, fin


def python_reference_sample(inst, state, window, cap, counts, seconds, seed=1):
    """The UNMODIFIED reference (rlmux installed in baseline/_ref from
    /root/reference) scoring a uniform sample of the decision's non-merge
    candidates, forked over every host core, next to the C port on the same
    candidates (one thread). Merges are not sampled: one config-5 merge
    costs ~20 min of single-core Python. Returns per-candidate thread
    seconds of both, the key agreement, and the port/Python ratio."""
    import multiprocessing as mp

    import numpy as np

    if not os.path.isdir(os.path.join(REF_DIR, "rlmux")):
        return {"unavailable": "baseline/_ref/rlmux not installed"}
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from oracle.oracle import Oracle
    from paper_2604_23838_b200.instance_io import action_to_json

    procs = os.cpu_count() or 1
    n_mux, n_merge, n_excl = counts
    rng = np.random.default_rng(seed)
    pool_serials = np.concatenate([rng.permutation(n_mux), n_mux + n_merge + rng.permutation(n_excl)])
    pool_serials = rng.permutation(pool_serials)[:4096]
    o1 = Oracle(inst, nthreads=1)
    ctx = mp.get_context("fork")
    done, wall, times, keys = 0, 0.0, [], []
    with ctx.Pool(procs, initializer=_pyref_init, initargs=(inst, window)) as pool:
        last = 0.0
        while done < len(pool_serials) and (done == 0 or wall + last <= seconds):
            part = [int(x) for x in pool_serials[done:done + procs]]
            acts = [action_to_json(o1.candidate(state, s, cap)) for s in part]
            t = time.perf_counter()
            res = pool.map(_pyref_score, acts, chunksize=1)
            last = time.perf_counter() - t
            wall += last
            times += [r[0] for r in res]
            keys += [(s, r[1], r[2]) for s, r in zip(part, res)]
            done += len(part)
    sample = sorted(k[0] for k in keys)
    t = time.perf_counter()
    r = o1.score(state, window, cap, serials=sample, want_keys=True)
    port_s = time.perf_counter() - t
    port = {s: tuple(k) for s, k in zip(sample, r["keys"])}
    agree = all(port[s] == (c, f) for s, c, f in keys)
    py_t = sum(times) / len(times)
    port_t = port_s / len(sample)
    return {"kind": "reference (rlmux, unmodified, baseline/_ref)", "procs": procs,
            "sample": f"{len(sample)} uniformly drawn multiplex/exclusive candidates, forked over {procs} processes "
                      f"in {wall:.1f} s",
            "python_thread_s_per_candidate": py_t, "port_thread_s_per_candidate": port_t,
            "port_speedup_over_python": py_t / port_t, "keys_match_port": agree,
            "candidates_per_s_nonmerge": procs / py_t}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class _Enough(Exception):
    pass


def schedule_latency(name, device, cpu=False, max_decisions=None):
    """p50 decision latency over a whole look-ahead schedule (SURVEY §8(d):
    config 1 has 18 decisions, mostly 1-8 candidates, so this measures the
    fixed per-decision overhead). GPU: the public chooser; cpu=True: the
    oracle port's chooser (reference arm)."""
    from paper_2604_23838_b200 import drive

    window, cap, _ = CONFIGS[name]
    inst = load_instance(name)
    if cpu:
        from oracle.oracle import Oracle

        choose = Oracle(inst, nthreads=os.cpu_count() or 1).chooser(window, cap)
    else:
        from paper_2604_23838_b200.native import Evaluator

        choose = Evaluator(inst, device=device).chooser(window, cap)
    lat = []

    def timed(state):
        if max_decisions is not None and len(lat) >= max_decisions:
            raise _Enough()
        t = time.perf_counter()
        a = choose(state)
        lat.append((time.perf_counter() - t) * 1e3)
        return a

    def run():
        try:
            return len(drive(inst, timed, "lookahead", {}).actions)
        except _Enough:
            return None

    if max_decisions is None:
        run()  # warm-up: a whole schedule
    else:
        from paper_2604_23838_b200.state import State as HostState

        choose(HostState(inst))  # warm-up: the first decision
    lat.clear()
    t = time.perf_counter()
    n_actions = run()
    total = time.perf_counter() - t
    what = "full lookahead_schedule" if max_decisions is None else f"first {len(lat)} decisions from t=0"
    out = {"workload": f"{name} {what} (W={window}, max_merge={cap})", "decisions": len(lat),
           "p50_decision_ms": statistics.median(lat), "max_decision_ms": max(lat), "schedule_s": total}
    if n_actions is not None:
        out["actions"] = n_actions
    return out


def run_reference(args):
    """The reference arm: the CPU port of the reference chooser on every host
    thread (class-stratified, fixed budget --cpu-seconds independent of
    --steps), plus the unmodified Python reference (baseline/_ref) on a
    non-merge sample next to the port. Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle import Oracle
    from paper_2604_23838_b200.state import State as HostState

    window, cap, desc = CONFIGS[args.config]
    inst = load_instance(args.config)
    st = HostState(inst)
    counts = Oracle(inst, nthreads=1).counts(st, window, cap)
    n_total = sum(counts)
    r = cpu_stratified(inst, st, window, cap, counts, args.cpu_seconds)
    value = r["rate"]
    sched = (schedule_latency(args.schedule_config, 0, cpu=True, max_decisions=args.schedule_decisions)
             if args.schedule_p50 else None)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "candidates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * r["decision_s"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, golden instance)",
        "config": {"workload": f"{args.config} first decision: {desc}", "window": window, "max_merge": cap,
                   "candidates_per_decision": n_total},
        "cpu_baseline": cpu_baseline_record(r, n_total),
        "e2e": {"value": value, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.python_seconds > 0:
        line["python_reference"] = python_reference_sample(inst, st, window, cap, counts, args.python_seconds)
    if sched is not None:
        line["schedule"] = sched
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    # RLX_DIST_BACKEND=gloo runs several ranks on one device (test of the
    # multi-rank path on a 1-GPU box); the product path is NCCL, one GPU per rank
    backend = os.environ.get("RLX_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2604_23838_b200.dist import WORDS, best_row, unpack
    from paper_2604_23838_b200.state import State as HostState
    from paper_2604_23838_b200.native import Evaluator

    window, cap, desc = CONFIGS[args.config]
    inst = load_instance(args.config)
    st = HostState(inst)
    ev = Evaluator(inst, device=local)
    # one explicit stream for torch ops, NCCL, CUDA events and the library
    # (torch's default current stream is the legacy NULL stream, which the
    # library cannot be pointed at: NULL means "the handle's own stream")
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ev.set_stream(stream.cuda_stream)
    part = (rank, world)
    table = torch.zeros((world, WORDS), dtype=torch.int64, device=dev)
    row_ptr = table.data_ptr() + rank * WORDS * 8
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def minloc():
        if world > 1:
            dist.all_reduce(table, op=dist.ReduceOp.SUM)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- plan + upload once (also the first warm-up), then the resident loop
    d0 = ev.decide(st, window, cap, part=part, dev_key_ptr=row_ptr)
    n_total = d0.n_candidates
    ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kern_ms, bytes_l, passes_l, events_l = [], [], [], []
    winners = set()
    for i in range(args.warmup):
        table.zero_()
        ev.rescore(window, part=part, dev_key_ptr=row_ptr)
        minloc()
    torch.cuda.synchronize(dev)
    barrier()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        barrier()
        for i in range(args.steps):
            flush.fill_(i)  # L2 flush between timed steps (outside the step events)
            table.zero_()
            ev_a[i].record(stream)
            d = ev.rescore(window, part=part, dev_key_ptr=row_ptr)
            minloc()
            ev_b[i].record(stream)
            kern_ms.append(d.kernel_ms)
            bytes_l.append(d.alg_bytes)
            passes_l.append(d.passes)
            events_l.append(d.events)
            rows = table.cpu().numpy().view(np.uint64)
            winners.add(unpack(rows[best_row(rows)]))
        torch.cuda.synchronize(dev)
        barrier()
        step_ms = [a.elapsed_time(bb) for a, bb in zip(ev_a, ev_b)]
        # ---- e2e through the public chooser (host state in, action out)
        choose = ev.chooser(window, cap, group=dist.group.WORLD if world > 1 else None)
        e2e_ms, wall_ms = [], []
        e2e_steps = min(max(args.steps, 3), args.e2e_steps)
        for i in range(1 + e2e_steps):  # one warm-up (the plan is the same decision)
            flush.fill_(i)
            torch.cuda.synchronize(dev)
            barrier()
            t = time.perf_counter()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            action = choose(st)
            a1.record(stream)
            torch.cuda.synchronize(dev)
            w = (time.perf_counter() - t) * 1e3
            if i >= 1:
                e2e_ms.append(a0.elapsed_time(a1))
                wall_ms.append(w)
        last_e2e = ev.last
        from paper_2604_23838_b200.instance_io import action_to_json

        e2e_action = action_to_json(action)
    clocks = clk.summary()
    sum_ms = max_over_ranks(sum(step_ms))
    ms_per_step = sum_ms / args.steps
    e2e_sum = max_over_ranks(sum(e2e_ms))
    p50_wall = max_over_ranks(statistics.median(wall_ms))
    kernel_avg = max_over_ranks(sum(kern_ms) / len(kern_ms))
    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return 0
    value = n_total * args.steps / (sum_ms / 1e3)
    e2e_value = n_total * len(e2e_ms) / (e2e_sum / 1e3)
    peak, peak_src = measured_peak()
    alg_bytes = statistics.mean(bytes_l)  # rank 0's shard bytes per launch
    achieved = alg_bytes / (statistics.mean(kern_ms) / 1e3) / 1e9
    traffic, issue = ncu_record(args.config)
    sched = None
    if world == 1 and args.schedule_p50:
        sched = schedule_latency(args.schedule_config, local, max_decisions=args.schedule_decisions)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        counts = (d0.n_multiplex, d0.n_merge, d0.n_exclusive)
        cpu = cpu_baseline_record(cpu_stratified(inst, st, window, cap, counts, args.cpu_seconds), n_total)
    winner = sorted(winners)
    line = {
        "metric": METRIC, "value": value, "unit": "candidates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, golden instance)",
        "config": {"workload": f"{args.config} first decision: {desc}", "window": window, "max_merge": cap,
                   "candidates_per_decision": n_total, "parallelism": f"candidate shards x{world}",
                   "l2": "flushed between timed steps (256 MiB write outside the step events)"},
        "decisions_per_s": 1e3 / ms_per_step,
        "p50_decision_ms": p50_wall,
        "e2e": {"value": e2e_value, "unit": "candidates/s", "h2d_bytes_per_step": int(last_e2e.h2d_bytes),
                "d2h_bytes_per_step": int(last_e2e.d2h_bytes) + (8 * WORDS * world if world > 1 else 0),
                "p50_decision_ms": p50_wall, "decisions_per_s": 1e3 * len(e2e_ms) / e2e_sum},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "kernel": "rlx_score_kernel",
                     "kernel_ms": statistics.mean(kern_ms), "alg_bytes_per_launch": alg_bytes,
                     "passes_per_launch": statistics.mean(passes_l),
                     "kernel_share_of_step": kernel_avg / ms_per_step},
        # the kernel's actual bound: SM instruction issue (SURVEY's HBM byte
        # model counts window re-reads that shared-memory staging removes)
        "issue_roofline": None if issue is None else {
            "bound": "sm_issue", "achieved": issue["sm_inst_issued_pct"], "peak": 100.0, "unit": "% of peak issue",
            "frac": issue["sm_inst_issued_pct"] / 100.0, "source": issue["source"]},
        "passes_per_decision": int(passes_l[-1]), "events_per_decision": int(events_l[-1]),
        "events_per_s": events_l[-1] / (statistics.mean(kern_ms) / 1e3),
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
        "winner": {"cost": winner[0][0], "finish": winner[0][1], "priority": winner[0][2],
                   "serial": winner[0][3]} if len(winner) == 1 else [list(w) for w in winner],
        "first_decide_plan_ms": d0.plan_ms,
        "action": e2e_action,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if sched is not None:
        line["schedule"] = sched
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("RLX_BENCH_CONFIG", "config5_cap2"), choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=60.0,
                    help="fixed CPU-port budget (class-stratified), independent of --steps")
    ap.add_argument("--python-seconds", type=float, default=40.0,
                    help="budget of the unmodified Python reference sample (reference arm; 0 = skip)")
    ap.add_argument("--e2e-steps", type=int, default=5, help="decisions timed through the public chooser")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--schedule-config", default="config1", choices=sorted(CONFIGS))
    ap.add_argument("--no-schedule", dest="schedule_p50", action="store_false")
    ap.add_argument("--schedule-decisions", type=int, default=None,
                    help="time only the first K decisions (SURVEY §8(d): 16 at configs 3-5)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
