"""NEXT-N3 on the GPU: the copy-based baseline pipeline (ws_rollout_staged, SPEC
baseline_copy_pipeline S:484-492) computes exactly the in-place roll-out -- its host-side
trajectories are bitwise identical to the fused in-place store ("results must be
bitwise identical to the in-place pipeline under the same seed") and to the oracle -- and
pays a measured, non-zero transfer time every step (P:106 / P:122)."""
import numpy as np
import pytest
import torch

import oracle as O
import wsinputs as W

pytestmark = pytest.mark.gpu
SEED = W.SEED


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2408_00930_b200 as P
    return P


CASES = [("cartpole", 300, 1, 200, {}), ("acrobot", 100, 1, 60, {}), ("pendulum", 200, 1, 80, {}),
         ("tag", 4, 100, 40, {"param0": 20, "param1": 10}), ("surface", 40, 1, 30, {"param0": 20}),
         ("dummy", 256, 1, 120, {})]


def probs_for(env, E, A):
    w = {"cartpole": 2, "acrobot": 3, "tag": 5, "dummy": 2}
    if env in w:
        return W.random_probs(E, A, w[env], seed=5, zero_frac=0.2)
    if env == "pendulum":
        return W.gaussian_params(E, A, 1, 0.0, 0.0)
    return W.gaussian_params(E, A, 20, 0.0, float(np.log(0.025)))


@pytest.mark.parametrize("env,E,A,T,kw", CASES)
def test_staged_equals_in_place(P, env, E, A, T, kw):
    probs = probs_for(env, E, A)
    ref = P.Env(E, A, env, SEED, t_capacity=T, **kw)
    ref.rollout(T, torch.from_numpy(probs).cuda())
    ref.synchronize()
    g = P.Env(E, A, env, SEED, t_capacity=T, **kw)
    dst = g.host_store(T)
    hp = torch.from_numpy(probs).pin_memory()
    rep = g.rollout_staged(T, hp, dst)
    a = {k: v.cpu().numpy() for k, v in ref.buffers().items() if v is not None}
    for k, v in dst.items():
        assert np.array_equal(v.numpy(), a[k][:T], equal_nan=True), k
    b = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    for k in ("obs", "act", "rew", "done", "state", "obs_live", "reset_count", "ep_step", "stats"):
        if k in a:
            assert np.array_equal(b[k], a[k], equal_nan=True), k
    assert rep["transfer_ms"] > 0 and rep["total_ms"] >= rep["transfer_ms"]
    assert rep["h2d_bytes"] == T * probs.size * 4
    assert rep["d2h_bytes"] == sum(v.numel() * v.element_size() for v in dst.values())


def test_staged_matches_oracle(P):
    E, T = 200, 150
    probs = W.random_probs(E, 1, 2, seed=9)
    g = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    dst = g.host_store(T)
    g.rollout_staged(T, torch.from_numpy(probs).pin_memory(), dst)
    o = O.Batch("cartpole", E, 1, SEED, t_capacity=T)
    assert o.rollout(T, probs) == 0
    for k in ("obs", "act", "rew", "done", "logp"):
        assert np.array_equal(dst[k].numpy(), o.array(k)[:T]), k


def test_staged_per_step_probabilities(P):
    """step_stride > 0: the trainer sends a different probability block every step."""
    E, T, n = 128, 40, 3
    probs = np.stack([W.random_probs(E, 1, n, seed=100 + t) for t in range(T)])
    g = P.Env(E, 1, "acrobot", SEED, t_capacity=T)
    dst = g.host_store(T)
    g.rollout_staged(T, torch.from_numpy(probs).pin_memory(), dst, row_stride=n, step_stride=E * n)
    ref = P.Env(E, 1, "acrobot", SEED, t_capacity=T)
    ref.rollout(T, torch.from_numpy(probs).cuda(), row_stride=n, step_stride=E * n)
    assert np.array_equal(dst["act"].numpy(), ref.buffers()["act"].cpu().numpy()[:T])
    assert np.array_equal(dst["obs"].numpy(), ref.buffers()["obs"].cpu().numpy()[:T])


def test_staged_is_slower_than_in_place(P):
    """dummy env E = 256 -> transfer > 0 and steps/s strictly below in-place."""
    E, T = 256, 200
    probs = torch.full((E, 1, 2), 0.5)
    g = P.Env(E, 1, "dummy", SEED, t_capacity=T)
    d = torch.full((E, 1, 2), 0.5, device="cuda")
    g.rollout(T, d)
    g.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(g.stream)
    g.rollout(T, d)
    ev[1].record(g.stream)
    torch.cuda.synchronize()
    in_place_ms = ev[0].elapsed_time(ev[1])
    dst = g.host_store(T)
    rep = g.rollout_staged(T, probs.pin_memory(), dst)
    assert rep["transfer_ms"] > 0 and rep["total_ms"] > in_place_ms
