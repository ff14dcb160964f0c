"""NEXT-N1 on the GPU: the fused roll-out with in-kernel MLP inference (ws_rollout_policy)
against the oracle's policy roll-out (oracle/wso.cpp policy_probs, DESIGN R29), element by
element; the all-zero policy against the uniform-probability fused roll-out."""
import numpy as np
import pytest
import torch

import oracle as O
import wsinputs as W
from test_gpu_parity import compare

pytestmark = pytest.mark.gpu
SEED = W.SEED
OBS = {"cartpole": 4, "acrobot": 6, "dummy": 4}
NACT = {"cartpole": 2, "acrobot": 3, "dummy": 2}


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2408_00930_b200 as P
    return P


@pytest.mark.parametrize("env,H,E,T,scale", [("cartpole", 32, 300, 200, 2.0), ("cartpole", 64, 257, 300, 3.0),
                                             ("acrobot", 32, 200, 120, 2.0), ("acrobot", 64, 96, 150, 1.0),
                                             ("dummy", 32, 100, 50, 1.0)])
def test_policy_rollout_parity(P, env, H, E, T, scale):
    D, n = OBS[env], NACT[env]
    w = W.policy_weights(D, H, n, seed=61, scale=scale)
    g = P.Env(E, 1, env, SEED, t_capacity=T)
    g.rollout_policy(T, torch.from_numpy(w).cuda(), H)
    assert g.status() == 0
    o = O.Batch(env, E, 1, SEED, t_capacity=T)
    assert o.rollout_policy(T, w, H, n_threads=8) == 0
    buf = {k: (v.cpu().numpy() if v is not None else None) for k, v in g.buffers().items()}
    amb = np.zeros((T, E, 1), np.uint8)
    compare(buf, o, amb, env, T)
    # the policy really varies the action distribution
    if env != "dummy":
        assert 0.02 < (buf["act"][:T] == 0).mean() < 0.98


def test_zero_policy_equals_uniform_rollout(P):
    E, T, H = 500, 200, 32
    g = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    g.rollout_policy(T, torch.zeros(4 * H + H + H * 2 + 2, device="cuda"), H)
    u = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    u.rollout(T, torch.full((E, 1, 2), 0.5, device="cuda"))
    a = {k: v.cpu().numpy() for k, v in g.buffers().items()}
    b = {k: v.cpu().numpy() for k, v in u.buffers().items()}
    for k in ("act", "logp", "obs", "rew", "done", "state", "reset_count", "stats"):
        assert np.array_equal(a[k], b[k]), k


def test_policy_c2_size_sampled_windows(P):
    """C2 shape (10K replicas x 1000 steps, H = 64) on the GPU; the oracle recomputes sampled
    replica windows (streams keyed by the global index, R15)."""
    E, T, H = 10_000, 1000, 64
    w = W.policy_weights(4, H, 2, seed=62, scale=2.0)
    g = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    g.rollout_policy(T, torch.from_numpy(w).cuda(), H)
    assert g.status() == 0
    buf = g.buffers()
    for off, n in ((0, 64), (5_000, 64), (9_936, 64)):
        o = O.Batch("cartpole", n, 1, SEED, env_offset=off, n_envs_global=E, t_capacity=T)
        assert o.rollout_policy(T, w, H, n_threads=8) == 0
        sub = {k: (v[:, off:off + n].cpu().numpy() if k in ("obs", "act", "logp", "rew", "done") else
                   v[off:off + n].cpu().numpy()) for k, v in buf.items() if v is not None and k != "stats"}
        sub["stats"] = np.array(o.array("stats"))
        compare(sub, o, np.zeros((T, n, 1), np.uint8), "cartpole", T)


def test_policy_invalid_weights_are_sticky(P):
    E, T, H = 64, 20, 32
    w = W.policy_weights(4, H, 2, seed=63)
    w[-1] = np.nan  # b2[1] = NaN -> every probability row is NaN
    g = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    g.rollout_policy(T, torch.from_numpy(w).cuda(), H)
    assert g.status() == P._abi.INVALID_PROBS
    buf = g.buffers()
    assert (buf["act"][:T] == -1).all() and (buf["done"][:T] == 0).all() and (buf["rew"][:T] == 0).all()


def test_policy_argument_validation(P):
    g = P.Env(8, 1, "cartpole", SEED, t_capacity=4)
    w = torch.zeros(4 * 32 + 32 + 32 * 2 + 2, device="cuda")
    with pytest.raises(P.WSError):
        g.rollout_policy(4, w, 48)  # hidden must be 32 or 64
    with pytest.raises(P.WSError):
        g.rollout_policy(5, w, 32)  # T beyond the store capacity
    t = P.Env(2, 10, "tag", SEED, t_capacity=4)
    with pytest.raises(P.WSError):
        t.rollout_policy(4, w, 32)  # multi-agent env: not supported by the policy roll-out
    p = P.Env(4, 1, "pendulum", SEED, t_capacity=4)
    with pytest.raises(P.WSError):
        p.rollout_policy(4, w, 32)  # continuous actions
