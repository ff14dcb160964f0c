"""Pins of the oracle's batch semantics: make_batch / step_all / auto_reset / run_rollout
(S:131-175), the in-place store and the statistics (row A8)."""
import numpy as np
import pytest
from scipy import stats

import oracle as O

SEED = 0x24080930


def _probs(E, A, n):
    return np.full((E, A, n), 1.0 / n, np.float32)


def test_reset_is_deterministic_and_in_distribution():
    """S:137-139 same seed -> bitwise-identical initial states, distinct per env;
    S:156 / Q11 initial distribution U(-0.05, 0.05)^4 (KS test over 4e5 draws)."""
    a = O.Batch("cartpole", 100000, seed=7)
    b = O.Batch("cartpole", 100000, seed=7)
    sa, sb = a.array("state"), b.array("state")
    assert np.array_equal(sa, sb)
    assert len(np.unique(sa[:, 0])) > 90000
    assert sa.min() >= -0.05 and sa.max() < 0.05
    for i in range(4):
        assert stats.kstest(sa[:, i], stats.uniform(loc=-0.05, scale=0.1).cdf).pvalue > 1e-4
    c = O.Batch("cartpole", 1000, seed=8)
    assert not np.array_equal(c.array("state"), sa[:1000])
    ba = O.Batch("acrobot", 50000, seed=1)
    ac = ba.array("state")
    assert ac.min() >= -0.1 and ac.max() < 0.1
    bp = O.Batch("pendulum", 50000, seed=1)
    pe = bp.array("state")
    assert stats.kstest(pe[:, 0], stats.uniform(loc=-np.pi, scale=2 * np.pi).cdf).pvalue > 1e-4
    assert stats.kstest(pe[:, 1], stats.uniform(loc=-1, scale=2).cdf).pvalue > 1e-4


def test_invalid_arguments():
    with pytest.raises(ValueError):
        O.Batch("cartpole", 0)            # S:138 E = 0 -> InvalidParams
    with pytest.raises(ValueError):
        O.Batch("nosuchenv", 4)           # S:135 UnknownEnvironment
    with pytest.raises(ValueError):
        O.Batch("cartpole", 4, n_agents=2)  # single-agent env
    b = O.Batch("cartpole", 4, t_capacity=2)
    assert b.rollout(3, _probs(4, 1, 2)) == O.OUT_OF_RANGE  # S:79 SlotOutOfRange
    assert b.rollout(0, _probs(4, 1, 2)) == O.INVALID_ARGUMENT  # S:166 T >= 1
    assert b.step(None) == O.BAD_STATE


def _rollout(env, E, T, n_threads=1, offset=0, E_global=0, A=1, probs=None, **kw):
    b = O.Batch(env, E, A, seed=SEED, env_offset=offset, n_envs_global=E_global, t_capacity=T, **kw)
    inf = b.info()
    if probs is None:
        probs = _probs(E, A, inf["n_actions"]) if inf["n_actions"] else np.zeros((E, A, 2 * inf["act_dim"]), np.float32)
    assert b.rollout(T, probs, n_threads=n_threads) == 0
    return b


NAMES = ["obs", "act", "logp", "rew", "done", "obs_live", "ep_step", "reset_count", "ep_ret"]


@pytest.mark.parametrize("env", ["cartpole", "acrobot", "pendulum", "surface", "tag", "dummy"])
def test_worker_count_invariance(env):
    """S:178 / S:583: bitwise-identical store for W in {1, 2, 4, 8}."""
    A = 12 if env == "tag" else 1
    kw = {"p0": 4} if env == "surface" else {}
    ref = _rollout(env, 16, 40, 1, A=A, **kw)
    for w in (2, 4, 8):
        b = _rollout(env, 16, 40, w, A=A, **kw)
        for n in NAMES:
            assert np.array_equal(ref.array(n), b.array(n), equal_nan=True), (env, n, w)
        np.testing.assert_allclose(ref.array("stats"), b.array("stats"), rtol=1e-12)


def test_sharding_invariance():
    """Reading Q15: streams keyed by the GLOBAL env index -> two shards with env_offset
    reproduce the unsharded batch env for env."""
    E, T = 40, 120
    full = _rollout("cartpole", E, T)
    lo = _rollout("cartpole", 25, T, offset=0, E_global=E)
    hi = _rollout("cartpole", 15, T, offset=25, E_global=E)
    for n in ["obs", "act", "logp", "rew"]:
        assert np.array_equal(full.array(n), np.concatenate([lo.array(n), hi.array(n)], axis=1))
    assert np.array_equal(full.array("done"), np.concatenate([lo.array("done"), hi.array("done")], axis=1))
    np.testing.assert_allclose(full.array("stats"), lo.array("stats") + hi.array("stats"), rtol=1e-12)


def test_rollout_equals_sample_step_loop():
    """run_rollout == T x (sample, log_step + step_all + auto_reset)."""
    E, T = 30, 60
    a = _rollout("acrobot", E, T)
    b = O.Batch("acrobot", E, seed=SEED, t_capacity=T)
    p = _probs(E, 1, 3)
    for _ in range(T):
        assert b.sample(p) == 0
        assert b.step() == 0
    for n in NAMES + ["stats"]:
        assert np.array_equal(a.array(n), b.array(n)), n


def test_rollout_invariants_cartpole():
    E, T = 64, 500
    b = _rollout("cartpole", E, T)
    obs, act, done, rew = b.array("obs"), b.array("act"), b.array("done"), b.array("rew")
    st, rc = b.array("stats"), b.array("reset_count")
    # reset_count == number of done flags (BJ:5 "reset counters")
    assert np.array_equal(rc, (done != 0).sum(axis=0))
    # reward 1 every step; actions in range; logp = ln 0.5
    assert np.all(rew == 1.0) and set(np.unique(act)) <= {0, 1}
    assert np.all(b.array("logp") == np.float32(np.log(0.5)))
    # continuity: obs[t+1] = step(obs[t], act[t]) when not done; reset state otherwise
    for t in range(T - 1):
        for e in range(0, E, 7):
            _, nxt, _, term = O.cartpole_step(obs[t, e, 0], act[t, e, 0])
            if done[t, e] == 0:
                assert np.array_equal(obs[t + 1, e, 0], nxt)
                assert not term
            else:
                assert bool(done[t, e] & 1) == term
                assert np.all(np.abs(obs[t + 1, e, 0]) < 0.05)  # fresh initial state
    # statistics (A8): counts and lengths exact
    assert st[:, 0].sum() == (done != 0).sum()
    # uniform-random CartPole mean episodic reward in [15, 35]
    mean_ret = st[:, 1].sum() / st[:, 0].sum()
    assert 15 <= mean_ret <= 35
    assert st[:, 2].sum() == st[:, 1].sum()  # reward 1 per step -> return == length


def test_selective_reset_and_isolation():
    """envs without done are untouched; S:179 isolation: changing env j's
    inputs never changes another env's trajectory."""
    E, T = 8, 50
    p = _probs(E, 1, 2)
    a = _rollout("cartpole", E, T, probs=p)
    p2 = p.copy(); p2[3, 0] = [0.9, 0.1]
    b = _rollout("cartpole", E, T, probs=p2)
    for e in range(E):
        same = np.array_equal(a.array("obs")[:, e], b.array("obs")[:, e])
        assert same == (e != 3)


def test_dummy_spec_example():
    """T=3, E=2, constant-reward dummy env (reward 1, done at step 3) -> mean
    episodic reward 3.0, mean length 3."""
    b = _rollout("dummy", 2, 3, max_steps=3)
    st = b.array("stats")
    assert st[:, 0].sum() == 2
    assert st[:, 1].sum() / st[:, 0].sum() == 3.0
    assert st[:, 2].sum() / st[:, 0].sum() == 3.0
    assert list(b.array("done")[:, 0]) == [0, 0, 2]  # bit1 = truncated


def test_truncation_flags():
    """Pendulum never terminates and truncates at 200 (Q10); CartPole with T_max=10."""
    b = _rollout("pendulum", 4, 450)
    d = b.array("done")
    assert set(np.nonzero(d[:, 0])[0]) == {199, 399} and np.all(d[199] == 2)
    c = _rollout("cartpole", 64, 60, max_steps=10)
    d = c.array("done")
    for e in range(64):
        length = 0
        for t in range(60):
            length += 1
            if d[t, e]:
                assert length <= 10
                assert bool(d[t, e] & 2) == (length == 10)  # truncated exactly at T_max
                length = 0
        assert length < 10


def test_invalid_action_is_sticky_and_not_advanced():
    """S:144 InvalidAction; reading Q19: env not advanced, rew = 0, done = 0, sticky."""
    b = O.Batch("cartpole", 3, seed=1, t_capacity=4)
    s0 = b.array("state").copy()
    assert b.step(np.array([[1], [5], [0]], np.int32)) == 0
    assert b.synchronize() == O.INVALID_ACTION
    s1 = b.array("state")
    assert np.array_equal(s1[1], s0[1]) and not np.array_equal(s1[0], s0[0])
    assert b.array("rew")[0, 1, 0] == 0.0 and b.array("done")[0, 1] == 0
    assert np.isnan(b.array("logp")[0, 0, 0])  # Q27 fixed actions -> logp NaN
    assert b.step(np.array([[1], [1], [0]], np.int32)) == 0
    assert b.synchronize() == O.INVALID_ACTION  # sticky until reset
    b.reset()
    assert b.synchronize() == O.OK
    # invalid probabilities
    b.set_capacity(2)
    assert b.sample(np.array([[[0.5, 0.5]], [[-1.0, 2.0]], [[0.0, 0.0]]], np.float32)) == 0
    assert b.synchronize() == O.INVALID_PROBS
    assert list(b.array("act")[0, :, 0]) == [b.array("act")[0, 0, 0], -1, -1]


def test_tag_rollout_structure():
    E, A, T = 6, 100, 200
    b = _rollout("tag", E, T, A=A)
    obs, rew, done = b.array("obs"), b.array("rew"), b.array("done")
    nt = 10
    assert np.all(obs[0, :, :nt, 2] == 1.0) and np.all(obs[0, :, nt:, 2] == 0.0)  # roles (Q22)
    assert np.all(obs[:, :, :, 0] >= 0) and np.all(obs[:, :, :, 0] <= 1)
    # runners: reward in {-1, 0.01, 0}; once -1, stays 0 until reset
    r = rew[:, :, nt:]
    assert set(np.unique(r)) <= {np.float32(-1), np.float32(0.01), np.float32(0)}
    assert np.all(done[-1] != 0)  # T_max = 200 -> everything ended by the last slot
