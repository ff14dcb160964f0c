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


@pytest.mark.parametrize("reduce", ["p2p", "nccl"])
def test_two_rank_bench_matches_oracle(reduce):
    """reduce = p2p: libws's peer-memory all-reduce kernel (CUDA IPC); nccl: the
    torch.distributed all_reduce path (gloo here)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    steps, warmup = 2, 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", str(steps), "--warmup", str(warmup), "--workload", "C1", "--dist-backend", "gloo",
           "--same-device", "--no-cpu-baseline", "--stats-reduce", reduce]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 prints exactly one JSON line
    d = json.loads(lines[0])
    w = W.CONFIGS["C1"]
    assert d["n_gpus"] == 2 and d["config"]["n_envs_global"] == 2 * w.n_envs and d["scaling"] == "weak"
    assert d["value"] > 0 and d["gpu_launches"] >= 2 * steps
    assert ("peer-memory" in d["config"]["parallelism"]) == (reduce == "p2p"), d["config"]["parallelism"]
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


@pytest.mark.parametrize("env,E_g,T", [("cartpole", 1000, 300), ("acrobot", 333, 120)])
def test_peer_memory_stats_allreduce(tmp_path, env, E_g, T):
    """Every rank's merged per-slot statistics (libws peer-memory kernel) equal, slot for slot
    and bit for bit, the oracle's statistics of the whole global batch, for several chained
    roll-outs (both gather-buffer parities)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n_roll = 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "tests/peer_worker.py", str(tmp_path),
           env, str(E_g), str(T), str(n_roll)]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    n_act = {"cartpole": 2, "acrobot": 3}[env]
    probs = W.random_probs(E_g, 1, n_act, seed=41, zero_frac=0.2)
    o = O.Batch(env, E_g, 1, W.SEED, t_capacity=T)
    ref = []
    for _ in range(n_roll):
        assert o.rollout(T, probs, n_threads=8) == 0
        ref.append(np.array(o.array("stats")).copy())
    for rank in (0, 1):
        got = np.load(os.path.join(tmp_path, f"stats_rank{rank}.npy")).astype(np.float64)
        got[..., 1] *= 2.0 ** -32
        got[..., 3] *= 2.0 ** -32
        for k in range(n_roll):
            assert np.array_equal(got[k][:, [0, 2]], ref[k][:, [0, 2]]), (rank, k)
            np.testing.assert_allclose(got[k][:, [1, 3]], ref[k][:, [1, 3]], rtol=1e-12, atol=E_g * 2.0 ** -32)
