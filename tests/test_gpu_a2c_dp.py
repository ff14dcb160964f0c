"""NEXT-N2 data parallelism: A2C with the global batch sharded over 2 ranks (torchrun, gloo,
one GPU -- the round's allocation has a single device) equals the single-process run on
the whole batch: the normalisation moments and the first gradient agree to fp32
accumulation order, and both ranks hold bitwise-identical parameters after every update
(they apply the same all-reduced gradient)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import wsinputs as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("E_g", [1000, 1001])
def test_two_rank_a2c_equals_single_process(tmp_path, E_g):
    """E_g = 1001: shards of 500 and 501 replicas -- the loss mean and the advantage
    normalisation must still use the global batch (not rows x world)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    T, iters = 64, 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "a2c_worker.py"), str(tmp_path), str(E_g), str(T), str(iters)]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    r0, r1 = np.load(tmp_path / "rank0.npz"), np.load(tmp_path / "rank1.npz")
    assert np.array_equal(r0["params"], r1["params"])          # replicas stay in sync
    assert np.array_equal(r0["grad0"], r1["grad0"]) and np.array_equal(r0["mom"], r1["mom"])
    # single process, whole batch
    from paper_2408_00930_b200 import Env
    from paper_2408_00930_b200.a2c import A2C
    env = Env(E_g, 1, "cartpole", W.SEED, t_capacity=T)
    tr = A2C(env, 64, params=torch.from_numpy(W.a2c_params(4, 64, 2, seed=71)), lr=1e-3)
    tr.iteration(T)
    torch.cuda.synchronize()
    g = tr.grad.cpu().numpy()
    scale = np.abs(g).max()
    assert np.all(np.abs(r0["grad0"] - g) <= 1e-4 * scale), np.abs(r0["grad0"] - g).max() / scale


def test_peer_memory_fused_allreduce_adam_equals_nccl_path(tmp_path):
    """peer=True: the moments and the gradient are reduced over CUDA-IPC peer memory and the
    gradient all-reduce is fused with clip + Adam (ws_pgroup_allreduce_adam, no NCCL / gloo
    call on the training path).  With 2 ranks the fp64 rank-order sum rounded to fp32 equals
    the fp32 two-term sum, so parameters must equal the torch.distributed path bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    E_g, T, iters = 1000, 64, 3
    dirs = {}
    for mode in ("dist", "peer"):
        d = tmp_path / mode
        d.mkdir()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()),
               os.path.join(ROOT, "tests", "a2c_worker.py"), str(d), str(E_g), str(T), str(iters)] + \
              (["peer"] if mode == "peer" else [])
        out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-3000:]
        dirs[mode] = d
    p0, p1 = np.load(dirs["peer"] / "rank0.npz"), np.load(dirs["peer"] / "rank1.npz")
    assert int(p0["peer_status"]) == 0 and int(p1["peer_status"]) == 0
    assert np.array_equal(p0["params"], p1["params"])
    q0 = np.load(dirs["dist"] / "rank0.npz")
    assert np.array_equal(p0["mom"], q0["mom"])
    assert np.array_equal(p0["grad0"], q0["grad0"])
    assert np.array_equal(p0["params"], q0["params"])
