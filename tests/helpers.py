"""Shared test helpers: golden data and instances."""
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_gz(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt", encoding="utf-8") as fh:
        return json.load(fh)


_cache = {}


def fixtures():
    from paper_2604_23838_b200 import load_instances

    if "fx" not in _cache:
        _cache["fx"] = load_instances(os.path.join(GOLDEN, "instances", "fixtures.json.gz"))
    return _cache["fx"]


def instance(name):
    """Golden instance by name: fixtures, `name|nomerge`, or config1..5."""
    from paper_2604_23838_b200 import load_instance
    from paper_2604_23838_b200.model import Instance

    base = name.split("|")[0]
    if base.startswith("config"):
        if base not in _cache:
            _cache[base] = load_instance(os.path.join(GOLDEN, "instances", f"{base}.json.gz"))
        inst = _cache[base]
    else:
        inst = fixtures()[base]
    if name.endswith("|nomerge"):
        inst = Instance(graphs=inst.graphs, model=inst.model, merge_enabled=False)
    if name.endswith("|knobs"):  # tests/golden/make_golden.py KNOBS
        inst = Instance(graphs=inst.graphs, model=inst.model, headroom=0.1, realloc_penalty=0.5,
                        default_migration_cost=0.25)
    return inst


