"""The multi-GPU bench path (torchrun, one process per rank, replicas sharded by global
index, statistics all-reduced) run with 2 ranks on ONE GPU over gloo -- the round's GPU
allocation has a single device, NCCL refuses two ranks per device.  The merged statistics
must equal the oracle's for the global batch (weak scaling: 2 x C1 replicas)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle as O
import wsinputs as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_bench_matches_oracle():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    steps, warmup = 2, 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", str(steps), "--warmup", str(warmup), "--workload", "C1", "--dist-backend", "gloo",
           "--same-device", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 prints exactly one JSON line
    d = json.loads(lines[0])
    w = W.CONFIGS["C1"]
    assert d["n_gpus"] == 2 and d["config"]["n_envs_global"] == 2 * w.n_envs and d["scaling"] == "weak"
    assert d["value"] > 0 and d["gpu_launches"] >= 2 * steps
    # oracle: the global batch, same number of chained roll-outs
    o = O.Batch("cartpole", 2 * w.n_envs, 1, W.SEED, t_capacity=w.T)
    probs = W.uniform_probs(2 * w.n_envs, 1, 2)
    for _ in range(warmup + steps):
        assert o.rollout(w.T, probs) == 0
    st = np.array(o.array("stats")).sum(0)
    got = d["episode_stats_last_step"]
    assert got["episodes"] == st[0]
    assert abs(got["mean_return"] - st[1] / st[0]) < 1e-9
    assert abs(got["mean_length"] - st[2] / st[0]) < 1e-9
