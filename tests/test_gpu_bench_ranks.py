"""bench.py --gpus N on ONE GPU (ranks wrap onto device 0; gloo instead of NCCL, which rejects two
ranks on one device): the multi-rank step runs, prints n_gpus = N, and -- the shards holding
exactly the single-GPU inputs and drawing the same Philox words -- emits exactly the tokens of
the single-GPU run (KV-head TP x batch DP)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(gpus):
    env = dict(os.environ, MD_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    args = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--config", "tiny", "--steps", "4",
            "--warmup", "3", "--skip-cpu", "--skip-e2e"]
    r = subprocess.run(args, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])


def test_ranks_emit_the_single_gpu_tokens():
    one = _bench(1)
    two = _bench(2)       # tp2 x dp1
    eight = _bench(8)     # tp4 x dp2 (tiny: 4 KV heads, batch 2)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2 and eight["n_gpus"] == 8
    assert two["config"]["parallelism"] == "tp2xdp1" and eight["config"]["parallelism"] == "tp4xdp2"
    assert two["tokens_per_step"] == one["tokens_per_step"] == eight["tokens_per_step"]
    assert two["scaling_efficiency"]["E_verify"] > 0
