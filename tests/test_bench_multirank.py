"""The multi-rank bench path (torchrun, candidate shards, one all-reduce per
decision) on a 1-GPU box: 2 or 3 ranks (uneven shards) share cuda:0 over
gloo. The ranks must agree on the single-GPU winner of the decision, for the
resident-plan steps and for the public-chooser (e2e) decisions."""

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


@pytest.mark.parametrize("ranks", [2, 3])
def test_ranks_match_one(ranks):
    env = dict(os.environ, RLX_DIST_BACKEND="gloo")
    args = ["bench.py", "--config", "config2", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-schedule"]
    one = _run([sys.executable] + args, env)
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
                "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args + ["--gpus", str(ranks)], env)
    assert two["n_gpus"] == ranks
    assert two["winner"] == one["winner"]
    assert two["action"] == one["action"]
    assert two["config"]["candidates_per_decision"] == one["config"]["candidates_per_decision"]
