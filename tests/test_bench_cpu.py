"""bench.py's host plumbing on CPU: `--gpus N` re-launches itself under torch.distributed.run
(gloo, 127.0.0.1) and every rank derives its shard of the tp x dp grid (P:460,
P:727); the reference arm (the oracle) prints the contract line for the same
workload; the Eq.1 helpers match their closed forms."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(args, timeout=300):
    env = dict(os.environ, MD_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])


def test_gpus_2_spawns_two_ranks():
    j = _run(["--gpus", "2", "--config", "tiny", "--plan-only"])
    assert j["n_gpus"] == 2 and j["tp"] == 2 and j["dp"] == 1
    assert j["covers_once"] and j["tp_gather_rank_major"] and j["max_over_ranks"]


def test_qwen_at_8_ranks_is_tp4_dp2():
    """Qwen2.5-7B (28 q / 4 KV heads) over 8 ranks: 4-way KV-head TP x 2-way batch DP."""
    j = _run(["--gpus", "8", "--config", "qwen_100k", "--plan-only"])
    assert (j["tp"], j["dp"]) == (4, 2) and j["config"]["parallelism"] == "tp4xdp2"
    assert j["covers_once"] and j["tp_gather_rank_major"]
    shards = np.array(j["shards"])
    assert sorted(set(map(tuple, shards[:, 6:8].tolist()))) == [(0, 32), (32, 64)]   # batch halves
    assert sorted(set(map(tuple, shards[:, 2:4].tolist()))) == [(0, 7), (7, 14), (14, 21), (21, 28)]


def test_grid_choice():
    from paper_2408_11049_b200.tp import rank_plan, tp_dp_grid
    assert tp_dp_grid(8, 32, 8, 256) == (8, 1)
    assert tp_dp_grid(8, 28, 4, 64) == (4, 2)
    assert tp_dp_grid(4, 32, 32, 64) == (4, 1)
    assert tp_dp_grid(1, 28, 4, 64) == (1, 1)
    with pytest.raises(ValueError):
        tp_dp_grid(8, 28, 4, 63)                  # the batch must split over dp
    p = rank_plan(5, 8, 64, 28, 4)
    assert (p["tp_rank"], p["dp_rank"]) == (1, 1) and p["q_heads"] == slice(7, 14) and p["batch"] == slice(32, 64)


def test_reference_arm_line_for_the_same_workload():
    j = _run(["--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1"])
    assert j["impl"] == "reference" and j["unit"] == "tokens/s" and j["higher_is_better"]
    assert j["config"] == bench.workload_config("tiny", 0.8)
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["value"] > 0
    # the tokens per step are the oracle acceptance's on the GPU arm's Philox steps 1..2
    p, q = bench.accept_inputs("tiny", 0.8)
    toks = [bench.oracle_accept_seconds("tiny", p, q, i)[1] for i in (1, 2)]
    assert j["tokens_per_step"] == pytest.approx(np.mean(toks))


def test_eq1_helpers():
    assert bench.omega_eq1(4, 0.8) == pytest.approx(3.3616)
    assert bench.omega_eq1(3, 0.8) == pytest.approx(2.952)
    assert bench.alpha_from_omega(4, 3.3616) == pytest.approx(0.8, abs=1e-9)
    beta = np.full((3, 4), 0.8)
    # overlap_stats' expected tokens with beta = alpha everywhere is Eq.1
    p = np.zeros((1, 5, 2), np.float32)
    q = np.zeros((1, 4, 2), np.float32)
    p[..., 0], p[..., 1] = 0.9, 0.1
    q[..., 0], q[..., 1] = 0.7, 0.3                   # beta = 0.7 + 0.1 = 0.8 per position
    b, om = bench.overlap_stats(p, q)
    assert np.allclose(b, 0.8) and om == pytest.approx(bench.omega_eq1(4, 0.8))
    assert beta.shape == (3, 4)
