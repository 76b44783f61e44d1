"""Generate the golden fixtures under tests/golden/ from the live reference.

TEST INFRASTRUCTURE ONLY. Needs /root/reference (build container); the
GPU box only reads the committed outputs.

    python tests/golden/make_golden.py instances      # config + fixture instances
    python tests/golden/make_golden.py schedules      # full recorded schedules (small instances)
    python tests/golden/make_golden.py schedules_knobs  # the same with non-default Instance knobs
    python tests/golden/make_golden.py keys [cfg...]  # sampled per-candidate keys at decision 0
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import time
import zlib
from multiprocessing import Pool

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import refharness as H  # noqa: E402

INST_DIR = os.path.join(HERE, "instances")


def _dump(obj, name):
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt", encoding="utf-8", compresslevel=9) as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path))


def fixture_instances():
    out = {"trap": H.rf.lookahead_trap_instance(), "async_small": H.build_async_small()}
    for s in range(100):
        out[f"rand{s:03d}"] = H.rf.random_small_instance(s)
    for s in range(20):
        out[f"mig{s:02d}"] = H.rf.random_migration_case(s)[3]
    return out


def cmd_instances(which):
    os.makedirs(INST_DIR, exist_ok=True)
    if not which or "fixtures" in which:
        fx = fixture_instances()
        blob = {k: H.instance_to_json(v) for k, v in fx.items()}
        _dump(blob, "instances/fixtures.json.gz")
    for k in (1, 2, 3, 4, 5):
        if which and str(k) not in which:
            continue
        t = time.time()
        inst = H.build_config(k)
        H.save_instance_json(inst, os.path.join(INST_DIR, f"config{k}.json.gz"))
        st = H.ExecState(inst)
        n = sum(len(g.nodes) for g in inst.graphs)
        e = sum(len(g.edges) for g in inst.graphs)
        print(f"config{k}: nodes={n} edges={e} ready={len(st.ready_compute())} "
              f"cands(cap3)={len(H.capped_enumerate(st, 3))} build={time.time()-t:.1f}s", flush=True)


def _sched_job(args):
    name, inst_json_name, window, max_merge, policy = args
    inst = _load_fixture(inst_json_name)
    t = time.time()
    if policy == "greedy_ref":
        sched = H.rs.greedy_schedule(inst)
        dec = None
    else:
        sched, dec = H.recorded_lookahead(inst, window, max_merge)
    from rlmux.sim import simulate
    rep = simulate(sched, inst)
    return name, {"instance": inst_json_name, "window": window, "max_merge": max_merge,
                  "policy": policy, "actions": H.schedule_to_json(sched), "decisions": dec,
                  "makespan": rep.makespan, "throughput": rep.aggregate_throughput,
                  "per_pipeline_latency": rep.per_pipeline_latency,
                  "per_pipeline_tokens": rep.per_pipeline_tokens, "secs": time.time() - t}


_FX_CACHE = {}


def _load_fixture(name):
    if name.startswith("config"):
        base = name.split("|")[0]
        if base not in _FX_CACHE:
            _FX_CACHE[base] = H.build_config(int(base[6:]))
        inst = _FX_CACHE[base]
        if name.endswith("|knobs"):
            inst = H.Instance(graphs=inst.graphs, model=inst.model, headroom=KNOBS["headroom"],
                              realloc_penalty=KNOBS["realloc_penalty"],
                              default_migration_cost=KNOBS["default_migration_cost"])
        return inst
    if not _FX_CACHE.get("_fx"):
        _FX_CACHE["_fx"] = fixture_instances()
    inst = _FX_CACHE["_fx"][name.split("|")[0]]
    if name.endswith("|nomerge"):
        inst = H.Instance(graphs=inst.graphs, model=inst.model, merge_enabled=False)
    if name.endswith("|knobs"):  # non-default Instance knobs (scheduler.py:117-122)
        inst = H.Instance(graphs=inst.graphs, model=inst.model, headroom=KNOBS["headroom"],
                          realloc_penalty=KNOBS["realloc_penalty"],
                          default_migration_cost=KNOBS["default_migration_cost"])
    return inst


# realloc penalty on (:463-470), a default migration cost for spec-less
# pipelines (:539-542), and a wider memory headroom (feasible, complements)
KNOBS = {"headroom": 0.1, "realloc_penalty": 0.5, "default_migration_cost": 0.25}


def cmd_schedules_knobs():
    jobs = []
    for w in (1, 3):
        jobs.append((f"trap_knobs_w{w}", "trap|knobs", w, None, "lookahead"))
        jobs.append((f"async_small_knobs_w{w}_cap3", "async_small|knobs", w, 3, "lookahead"))
    for s in range(0, 100, 3):
        for w in (1, 3):
            jobs.append((f"rand{s:03d}_knobs_w{w}", f"rand{s:03d}|knobs", w, None, "lookahead"))
    for s in range(20):
        jobs.append((f"mig{s:02d}_knobs_w2", f"mig{s:02d}|knobs", 2, None, "lookahead"))
    jobs.append(("config1_knobs_w1_cap3", "config1|knobs", 1, 3, "lookahead"))
    with Pool(8) as pool:
        res = dict(pool.map(_sched_job, jobs, chunksize=1))
    _dump(res, "schedules_knobs.json.gz")


def cmd_schedules():
    jobs = []
    for w in (1, 2, 3):
        jobs.append((f"trap_w{w}", "trap", w, None, "lookahead"))
        jobs.append((f"async_small_w{w}_cap3", "async_small", w, 3, "lookahead"))
    for s in range(100):
        for w in (1, 3):
            jobs.append((f"rand{s:03d}_w{w}", f"rand{s:03d}", w, None, "lookahead"))
        jobs.append((f"rand{s:03d}_w3_nomerge", f"rand{s:03d}|nomerge", 3, None, "lookahead"))
    for s in range(20):
        jobs.append((f"mig{s:02d}_w2", f"mig{s:02d}", 2, None, "lookahead"))
    for w in (1, 3):
        jobs.append((f"config1_w{w}", "config1", w, None, "lookahead"))
        jobs.append((f"config1_w{w}_cap3", "config1", w, 3, "lookahead"))
    with Pool(8) as pool:
        res = dict(pool.map(_sched_job, jobs, chunksize=1))
    _dump(res, "schedules.json.gz")


def _keys_job(args):
    cfg, window, max_merge, idx = args
    inst = _load_fixture(cfg)
    st = H.ExecState(inst)
    with H.capped(max_merge):
        cands = H.capped_enumerate(st, max_merge)
        t = time.time()
        keys = H.candidate_keys(st, cands, window, idx)
    return cfg, keys, time.time() - t


def cmd_keys(which):
    # (instance, W, cap, n_nonmerge_sample, n_merge_sample)
    plan = {
        "trap": ("trap", 3, None, None, None),
        "async_small": ("async_small", 3, 3, None, None),
        "config1": ("config1", 1, None, None, None),
        "config2": ("config2", 2, 3, 48, 16),
        "config3": ("config3", 3, 3, 24, 4),
        "config4": ("config4", 3, 3, 16, 4),
        "config5": ("config5", 4, 3, 8, 2),
        # every candidate of the config-2 cap-3 first decision (about 6 min on 8 cores)
        "config2_full": ("config2", 2, 3, None, None),
        # larger samples at the big configs (a different seed per name)
        "config3_more": ("config3", 3, 3, 64, 8),
        "config4_more": ("config4", 3, 3, 48, 8),
        "config5_cap2": ("config5", 4, 2, 32, 8),
    }
    out = {}
    path = os.path.join(HERE, "keys.json.gz")
    if os.path.exists(path):
        with gzip.open(path, "rt") as fh:
            out = json.load(fh)
    for name, (inst_name, window, cap, n_nm, n_m) in plan.items():
        if (which and name not in which) or (not which and "_" in name):
            continue
        inst = _load_fixture(inst_name)
        st = H.ExecState(inst)
        cands = H.capped_enumerate(st, cap)
        rng = random.Random(1234 if "_" not in name else zlib.crc32(name.encode()))
        if n_nm is None:
            idx = list(range(len(cands)))
        else:
            nm = [i for i, c in enumerate(cands) if not isinstance(c.action, H.Merge)]
            mg = [i for i, c in enumerate(cands) if isinstance(c.action, H.Merge)]
            idx = sorted(rng.sample(nm, min(n_nm, len(nm))) + rng.sample(mg, min(n_m, len(mg))))
        chunks = [idx[i::8] for i in range(8)]
        t = time.time()
        with Pool(8) as pool:
            res = pool.map(_keys_job, [(inst_name, window, cap, ch) for ch in chunks if ch])
        keys = sorted(k for _, ks, _ in res for k in keys_fix(ks))
        out[name] = {"instance": inst_name, "window": window, "max_merge": cap,
                     "n_candidates": len(cands), "keys": keys,
                     "cpu_secs": sum(s for _, _, s in res), "wall_secs": time.time() - t}
        print(name, len(keys), "keys", f"{time.time()-t:.1f}s", flush=True)
        _dump(out, "keys.json.gz")


def keys_fix(ks):
    return [list(k) for k in ks]


if __name__ == "__main__":
    cmd = sys.argv[1]
    rest = sys.argv[2:]
    if cmd == "instances":
        cmd_instances(rest)
    elif cmd == "schedules":
        cmd_schedules()
    elif cmd == "schedules_knobs":
        cmd_schedules_knobs()
    elif cmd == "keys":
        cmd_keys(rest)
    else:
        raise SystemExit(__doc__)
