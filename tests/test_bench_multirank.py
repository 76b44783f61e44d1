"""The multi-rank bench path (torchrun, candidate shards, one all-reduce per
decision) on a 1-GPU box: two ranks share cuda:0 over gloo. Every rank must
agree on the single-GPU winner of the decision."""

import json
import os
import socket
import subprocess
import sys

import pytest

from helpers import ROOT

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(cmd, env):
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_two_ranks_match_one():
    env = dict(os.environ, RLX_DIST_BACKEND="gloo")
    args = ["bench.py", "--config", "config2", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-schedule"]
    one = _run([sys.executable] + args, env)
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args + ["--gpus", "2"], env)
    assert two["n_gpus"] == 2
    assert two["winner"] == one["winner"]
    assert two["config"]["candidates_per_decision"] == one["config"]["candidates_per_decision"]
