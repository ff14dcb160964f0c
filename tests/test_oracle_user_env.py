"""Pins of the oracle's NEXT-N4 registered-env path (oracle/wso.cpp K_USER, DESIGN R32):
CartPole rewritten as a user env must reproduce the already-pinned built-in CartPole
roll-out bit for bit (same engine semantics around a different step function), MountainCar
obeys gym's rules (velocity and position bounds, inelastic left wall, goal, reward -1,
truncation at 200), and the point mass reads its per-replica parameters and the shared map."""
import numpy as np
import pytest

import oracle as O
import wsinputs as W
import wsinputs.user_envs as U

SEED = W.SEED


@pytest.fixture(scope="module", autouse=True)
def registered():
    for name, (src, dims) in U.ENVS.items():
        O.register_user_env(name, src, **dims)


def test_user_cartpole_equals_builtin():
    E, T = 64, 600
    probs = W.random_probs(E, 1, 2, seed=3)
    a = O.Batch("cartpole", E, 1, SEED, t_capacity=T, max_steps=30)
    b = O.Batch("u_cartpole", E, 1, SEED, t_capacity=T, max_steps=30)
    assert a.rollout(T, probs) == 0 and b.rollout(T, probs) == 0
    for k in ("obs", "act", "logp", "rew", "done", "stats", "state", "obs_live", "reset_count", "ep_step"):
        assert np.array_equal(a.array(k), b.array(k), equal_nan=True), k
    assert (a.array("done")[:T] & 2).any() and (a.array("done")[:T] & 1).any()  # both done kinds


def test_mountaincar_rules():
    E, T = 200, 400
    o = O.Batch("u_mountaincar", E, 1, SEED, t_capacity=T)
    assert o.rollout(T, W.random_probs(E, 1, 3, seed=4)) == 0
    obs, rew, done = o.array("obs")[:T], o.array("rew")[:T], o.array("done")[:T]
    x, v = obs[..., 0, 0], obs[..., 0, 1]
    assert np.all(rew == -1.0)
    assert np.all((x >= -1.2) & (x <= 0.6)) and np.all(np.abs(v) <= 0.07)
    # initial distribution U(-0.6, -0.4), v = 0 (every slot right after a reset)
    first = np.concatenate([obs[0, :, 0]] + [obs[t + 1, done[t] != 0, 0] for t in range(T - 1)])
    assert np.all((first[:, 0] >= -0.6) & (first[:, 0] < -0.4)) and np.all(first[:, 1] == 0)
    # random actions essentially never reach the goal: truncation at exactly 200 steps
    assert (done == 2).sum() >= E and np.all(o.array("stats")[:T][:, 2][o.array("stats")[:T][:, 0] > 0] % 200 == 0)
    # inelastic left wall: a state at x = -1.2 never carries negative velocity
    assert np.all(v[x == -1.2] >= 0)


def test_mountaincar_step_from_rest_closed_form():
    """From x = -pi/6 (the valley floor, cos(3x) = 0 up to rounding), v = 0, a push right
    adds exactly the force 0.001 (gravity term vanishes to fp32 precision): one step."""
    E = 1
    o = O.Batch("u_mountaincar", E, 1, SEED, t_capacity=1)
    st = o.array("state")
    st[0, 0] = np.float32(-np.pi / 6)
    st[0, 1] = 0.0
    assert o.step(np.array([2], np.int32)) == 0
    s = o.array("state")[0]
    assert abs(s[1] - 0.001) < 1e-9 and abs(s[0] - (np.float32(-np.pi / 6) + s[1])) < 1e-7


def test_pointmass_parameters_and_shared_map():
    E, T = 32, 150
    prm, grid = U.pointmass_data(E)
    o = O.Batch("u_pointmass", E, 1, SEED, t_capacity=T, env_prm=prm, env_shared=grid)
    assert o.rollout(T, W.random_probs(E, 1, 3, seed=6)) == 0
    rew = o.array("rew")[:T, :, 0]
    obs = o.array("obs")[:T, :, 0]
    assert np.all(np.isin(rew, grid))                          # rewards come from the shared map
    assert np.array_equal(obs[:, :, 2], np.broadcast_to(prm[:, 0], (T, E)))  # obs carries prm[0]
    # parameter jitter: the same actions with another force gain give other trajectories
    prm2 = prm.copy()
    prm2[:, 0] *= 2
    o2 = O.Batch("u_pointmass", E, 1, SEED, t_capacity=T, env_prm=prm2, env_shared=grid)
    assert o2.rollout(T, W.random_probs(E, 1, 3, seed=6)) == 0
    assert np.array_equal(o.array("act")[:1], o2.array("act")[:1])
    assert not np.array_equal(o.array("obs")[2:, :, :, :2], o2.array("obs")[2:, :, :, :2])


def test_noisy_mueller_brown_surface():
    """u_mbgrid (noisy PES): with a zero noise grid the observed energy is the Mueller-Brown
    energy of the pinned oracle function (fp32 terms, within fp32 rounding), the start lies
    near minimum B (E ~ -108, tests/golden/mueller_brown_stationary.txt); with noise the
    energy moves by exactly the grid cell's value; steps move by the replica's step size."""
    E, T = 64, 60
    prm, grid0 = U.mbgrid_data(E, noise=0.0)
    o = O.Batch("u_mbgrid", E, 1, SEED, t_capacity=T, env_prm=prm, env_shared=grid0)
    assert o.rollout(T, W.random_probs(E, 1, 5, seed=9)) == 0
    obs = o.array("obs")[:T, :, 0]
    ref = np.array([[O.mb_energy(float(x), float(y))[0] for x, y in row[:, :2]] for row in obs])
    np.testing.assert_allclose(obs[..., 2], ref, rtol=2e-5, atol=2e-4)
    assert np.all(np.abs(obs[0, :, 2] + 108.17) < 6.0)  # near minimum B at the start
    step = np.abs(np.diff(obs[:, :, :2], axis=0)).sum(-1)
    nxt = obs[1:, :, :2]
    inside = (nxt[..., 0] > -1.5) & (nxt[..., 0] < 1.2) & (nxt[..., 1] > -0.5) & (nxt[..., 1] < 2.0)
    moved = (step > 0) & (o.array("done")[:T - 1] == 0) & inside  # box clipping excluded
    np.testing.assert_allclose(step[moved], np.broadcast_to(prm[:, 0], step.shape)[moved], rtol=1e-5, atol=1e-6)
    _, grid = U.mbgrid_data(E)
    o2 = O.Batch("u_mbgrid", E, 1, SEED, t_capacity=T, env_prm=prm, env_shared=grid)
    assert o2.rollout(T, W.random_probs(E, 1, 5, seed=9)) == 0
    x, y = o2.array("obs")[0, :, 0, 0], o2.array("obs")[0, :, 0, 1]
    ix = np.clip(np.floor((x + np.float32(1.5)) * np.float32(32 / 2.7)).astype(int), 0, 31)
    iy = np.clip(np.floor((y + np.float32(0.5)) * np.float32(32 / 2.5)).astype(int), 0, 31)
    np.testing.assert_allclose(o2.array("obs")[0, :, 0, 2] - o.array("obs")[0, :, 0, 2], grid[iy * 32 + ix],
                               rtol=1e-5, atol=1e-4)


def test_user_pendulum_continuous_equals_builtin():
    """A continuous-action registered env (act_dim 1, R14 Gaussian head): Pendulum written as
    user C source reproduces the pinned built-in oracle Pendulum roll-out bit for bit."""
    E, T = 48, 250
    rows = W.gaussian_params(E, 1, 1, 0.3, -0.2)
    a = O.Batch("pendulum", E, 1, SEED, t_capacity=T)
    b = O.Batch("u_pendulum", E, 1, SEED, t_capacity=T)
    assert a.rollout(T, rows) == 0 and b.rollout(T, rows) == 0
    for k in ("obs", "act", "logp", "rew", "done", "stats", "state", "obs_live", "reset_count"):
        assert np.array_equal(a.array(k), b.array(k), equal_nan=True), k
