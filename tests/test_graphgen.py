"""Sub-Stage Graph construction on the GPU (
rlmux/workload.py:275-392 cohort replay, rlmux/graph.py:206-403
segmentation + construct_graph).

CPU: the batch generator draws exactly the reference generator's numbers
(live reference in the build container; skipped elsewhere), and the
pipeline tables of a reference PipelineSpec convert losslessly.
GPU: the five BASELINE.json config instances built by
`graphgen.build_config` on the device are JSON-identical to the committed
golden instances, which the live reference's own generator and
`construct_graph` produced (tests/golden/make_golden.py).
"""
import gzip
import json
import os
import sys

import numpy as np
import pytest

from helpers import GOLDEN

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def rlmux_workload():
    if not os.path.isdir(REF):
        pytest.skip("reference not present")
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import rlmux.workload

    return rlmux.workload


def _ref_tables(spec):
    from paper_2604_23838_b200.graphgen import batch_from_spec

    return batch_from_spec(spec)


@pytest.mark.parametrize("kw,seed", [
    (dict(batch=256, workers=8, model_params=8e9, pipeline_id="qwen8b"), 0),
    (dict(batch=1024, workers=32, model_params=32e9, decode_sigma=1.5, pipeline_id="p3"), 13),
    (dict(batch=4096, workers=64, model_params=0.6e9, tool_prob=0.5, tool_latency_mean=2.0, pipeline_id="a0"), 30),
    (dict(batch=64, workers=4, prompt_sigma=0.0, decode_sigma=0.0, pipeline_id="flat"), 7),
])
def test_generator_matches_reference(rlmux_workload, kw, seed):
    from paper_2604_23838_b200 import graphgen

    ours = graphgen.generate_synthetic(graphgen.GeneratorConfig(**kw), seed)
    spec = rlmux_workload.generate_synthetic(rlmux_workload.GeneratorConfig(**kw), seed)
    theirs = _ref_tables(spec)
    for f in ("prompt", "turn_off", "turn_prefill", "turn_decode", "turn_tool"):
        a, b = getattr(ours, f), getattr(theirs, f)
        assert a.dtype == b.dtype and np.array_equal(a, b), f
    assert (ours.pipeline_id, ours.model_params, ours.dp_workers, ours.stages) == (
        spec.pipeline_id, spec.model_params, spec.dp_workers, tuple(spec.stages))


def _golden(k):
    with gzip.open(os.path.join(GOLDEN, "instances", f"config{k}.json.gz"), "rt", encoding="utf-8") as fh:
        return json.load(fh)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_config_instances_built_on_device_equal_golden(k):
    import time

    from paper_2604_23838_b200 import graphgen
    from paper_2604_23838_b200.instance_io import instance_to_json

    batches = graphgen.config_batches(k)
    st = graphgen.BuildStats()
    t = time.perf_counter()
    inst = graphgen.build_config(k, batches=batches, stats=st)
    secs = time.perf_counter() - t
    got = instance_to_json(inst)
    want = _golden(k)
    assert got["graphs"] == want["graphs"]
    # the golden files spell the reference's default slowdown table "default"
    from paper_2604_23838_b200.instance_io import instance_from_json

    want["table"] = instance_to_json(instance_from_json(want))["table"]
    assert got == want
    print(f"config{k}: {st.records} step records, {st.segments} rollout sub-stages, kernels {st.kernel_ms:.1f} ms, "
          f"tables -> instance {secs * 1e3:.0f} ms")
