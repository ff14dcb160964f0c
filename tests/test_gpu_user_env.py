"""NEXT-N4 on the GPU: environments registered as C source (ws_register_env, NVRTC ->
sm_100a fused roll-out template) against the oracle's registered-env path (pinned in
tests/test_oracle_user_env.py), element by element; CartPole written as a user env against
the hand-written built-in CartPole kernel; per-replica parameters and shared data; sharding
invariance; the single-step path is refused."""
import numpy as np
import pytest
import torch

import oracle as O
import wsinputs as W
import wsinputs.user_envs as U

pytestmark = pytest.mark.gpu
SEED = W.SEED


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2408_00930_b200 as P
    for name, (src, dims) in U.ENVS.items():
        P.register_env(name, src, **dims)
        O.register_user_env(name, src, **dims)
    return P


KEYS = ("obs", "act", "logp", "rew", "done", "stats", "state", "obs_live", "reset_count", "ep_step")


def same(buf, o, T):
    for k in KEYS:
        ref = o.array(k)
        got = buf[k]
        if k in ("obs", "act", "logp", "rew", "done"):
            got, ref = got[:T], ref[:T]
        if k == "stats":
            continue
        assert np.array_equal(got, ref, equal_nan=True), k


@pytest.mark.parametrize("name,E,T,max_steps", [("u_cartpole", 1000, 300, 0), ("u_cartpole", 77, 120, 25),
                                                ("u_mountaincar", 513, 450, 0), ("u_mountaincar", 1, 10, 3)])
def test_registered_env_matches_oracle(P, name, E, T, max_steps):
    n = U.ENVS[name][1]["n_actions"]
    probs = W.random_probs(E, 1, n, seed=21, zero_frac=0.2)
    g = P.Env(E, 1, name, SEED, t_capacity=T, max_steps=max_steps)
    g.rollout(T, torch.from_numpy(probs).cuda())
    assert g.status() == 0
    o = O.Batch(name, E, 1, SEED, t_capacity=T, max_steps=max_steps)
    assert o.rollout(T, probs) == 0
    buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    same(buf, o, T)
    assert np.array_equal(g.stats_f64(T).cpu().numpy(), o.array("stats")[:T])


def test_user_cartpole_equals_builtin_kernel(P):
    """The NVRTC-compiled user CartPole and the hand-written k_rollout_discrete<CartPole>
    produce the same store bit for bit (both follow R3-R6 and the engine readings)."""
    E, T = 4096, 400
    probs = torch.from_numpy(W.random_probs(E, 1, 2, seed=22)).cuda()
    a = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    b = P.Env(E, 1, "u_cartpole", SEED, t_capacity=T)
    a.rollout(T, probs)
    b.rollout(T, probs)
    A = {k: v.cpu().numpy() for k, v in a.buffers().items() if v is not None}
    B = {k: v.cpu().numpy() for k, v in b.buffers().items() if v is not None}
    for k in ("obs", "act", "logp", "rew", "done", "stats", "state", "obs_live", "reset_count", "ep_step"):
        assert np.array_equal(A[k], B[k], equal_nan=True), k


def test_pointmass_parameters_and_shared_grid(P):
    E, T = 700, 200
    prm, grid = U.pointmass_data(E)
    probs = W.random_probs(E, 1, 3, seed=23)
    tp, tg = torch.from_numpy(prm).cuda(), torch.from_numpy(grid).cuda()
    g = P.Env(E, 1, "u_pointmass", SEED, t_capacity=T, env_prm=tp, env_shared=tg)
    g.rollout(T, torch.from_numpy(probs).cuda())
    o = O.Batch("u_pointmass", E, 1, SEED, t_capacity=T, env_prm=prm, env_shared=grid)
    assert o.rollout(T, probs) == 0
    buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    same(buf, o, T)
    # a parameter change through ws_set_env_data + ws_reset takes effect
    prm2 = prm.copy()
    prm2[:, 1] = 0.0
    g.set_env_data(torch.from_numpy(prm2).cuda(), tg)
    g.reset()
    g.rollout(T, torch.from_numpy(probs).cuda())
    o2 = O.Batch("u_pointmass", E, 1, SEED, t_capacity=T, env_prm=prm2, env_shared=grid)
    assert o2.rollout(T, probs) == 0
    same({k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}, o2, T)


def test_sharded_registered_env(P):
    """Two shards of a registered env equal the corresponding replicas of one unsharded run
    (streams keyed by the global replica index, R15)."""
    E, T = 300, 100
    probs = torch.from_numpy(W.random_probs(E, 1, 3, seed=24)).cuda()
    full = P.Env(E, 1, "u_mountaincar", SEED, t_capacity=T)
    full.rollout(T, probs)
    F = full.buffers()["obs"].cpu().numpy()
    h = 128
    s1 = P.Env(E - h, 1, "u_mountaincar", SEED, env_offset=h, n_envs_global=E, t_capacity=T)
    s1.rollout(T, probs[h:].contiguous())
    assert np.array_equal(s1.buffers()["obs"].cpu().numpy(), F[:, h:])


def test_single_step_path_refused(P):
    g = P.Env(8, 1, "u_mountaincar", SEED, t_capacity=4)
    with pytest.raises(P.WSError):
        g.sample(torch.full((8, 1, 3), 1 / 3, device="cuda"))


@pytest.mark.parametrize("H", [32, 64])
def test_registered_env_policy_rollout(P, H):
    """The R29 policy inside the registered env's loop (ws_rollout_policy on a C-source env)
    equals the oracle's policy roll-out, and the user CartPole with the critic equals the
    hand-written policy kernel on the built-in CartPole bit for bit (values included)."""
    E, T = 300, 150
    w = W.policy_weights(4, H, 2, seed=91, scale=2.0)
    g = P.Env(E, 1, "u_cartpole", SEED, t_capacity=T)
    g.rollout_policy(T, torch.from_numpy(w).cuda(), H)
    assert g.status() == 0
    o = O.Batch("u_cartpole", E, 1, SEED, t_capacity=T)
    assert o.rollout_policy(T, w, H, n_threads=4) == 0
    buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    for k in ("obs", "act", "rew", "done", "obs_live", "reset_count"):
        ref = o.array(k)[:T] if k in ("obs", "act", "rew", "done") else o.array(k)
        got = buf[k][:T] if k in ("obs", "act", "rew", "done") else buf[k]
        assert np.array_equal(got, ref), k
    lg, lo = buf["logp"][:T], o.array("logp")[:T]
    assert np.all(np.abs(lg.view(np.int32).astype(np.int64) - lo.view(np.int32).astype(np.int64)) <= 2)
    # critic variant against the built-in kernel
    params = torch.from_numpy(W.a2c_params(4, H, 2, seed=92)).cuda()
    a = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    b = P.Env(E, 1, "u_cartpole", SEED, t_capacity=T)
    va, ba = torch.empty(T * E, device="cuda"), torch.empty(E, device="cuda")
    vb, bb = torch.empty(T * E, device="cuda"), torch.empty(E, device="cuda")
    a.rollout_actor_critic(T, params, H, va, ba)
    b.rollout_actor_critic(T, params, H, vb, bb)
    A = {k: v.cpu().numpy() for k, v in a.buffers().items() if v is not None}
    B = {k: v.cpu().numpy() for k, v in b.buffers().items() if v is not None}
    for k in ("obs", "act", "rew", "done", "state", "obs_live", "stats"):
        assert np.array_equal(A[k], B[k]), k
    assert torch.equal(va, vb) and torch.equal(ba, bb)


def test_registered_env_trains(P):
    """The training loop on an environment supplied as C source (CartPole through the
    composer) solves it like the built-in env."""
    from paper_2408_00930_b200.train import train
    curve = train("u_cartpole", 10000, 32, 3000, lr=3e-3, target=475.0, log_every=50)
    print(f"u_cartpole solved: mean return {curve[-1][2]:.1f} after {curve[-1][1]:.3g} env steps, "
          f"{curve[-1][0]:.2f} s")
    assert curve[-1][2] >= 475.0


def test_noisy_pes_env_matches_oracle(P):
    """u_mbgrid: a discrete walker on a noisy Mueller-Brown PES (fp32 terms with ws_exp, a
    shared 32 x 32 noise grid, per-replica step sizes) -- GPU store vs the oracle."""
    E, T = 1000, 200
    prm, grid = U.mbgrid_data(E)
    probs = W.random_probs(E, 1, 5, seed=151)
    g = P.Env(E, 1, "u_mbgrid", SEED, t_capacity=T, env_prm=torch.from_numpy(prm).cuda(),
              env_shared=torch.from_numpy(grid).cuda())
    g.rollout(T, torch.from_numpy(probs).cuda())
    assert g.status() == 0
    o = O.Batch("u_mbgrid", E, 1, SEED, t_capacity=T, env_prm=prm, env_shared=grid)
    assert o.rollout(T, probs) == 0
    buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    same(buf, o, T)
    st_g, st_o = g.stats_f64(T).cpu().numpy(), np.array(o.array("stats"))[:T]
    assert np.array_equal(st_g[:, [0, 2]], st_o[:, [0, 2]])
    np.testing.assert_allclose(st_g[:, [1, 3]], st_o[:, [1, 3]], rtol=1e-12, atol=E * 2.0 ** -32)


def test_continuous_registered_env_equals_builtin(P):
    """A continuous-action C-source env (act_dim 1): the NVRTC template's R14 Gaussian head and
    the user's Pendulum reproduce the hand-written Pendulum kernels bit for bit (given rows and
    per-step rows), and match the oracle's registered-env path."""
    E, T = 700, 220
    rows = W.gaussian_params(E, 1, 1, 0.3, -0.2)
    for stride_rows in (rows, np.stack([W.gaussian_params(E, 1, 1, 0.1 * t, -0.3) for t in range(T)])):
        step_stride = 0 if stride_rows.ndim == 3 else E * 2
        tr = torch.from_numpy(np.ascontiguousarray(stride_rows)).cuda()
        a = P.Env(E, 1, "pendulum", SEED, t_capacity=T)
        b = P.Env(E, 1, "u_pendulum", SEED, t_capacity=T)
        a.rollout(T, tr, row_stride=2, step_stride=step_stride)
        b.rollout(T, tr, row_stride=2, step_stride=step_stride)
        assert a.status() == 0 and b.status() == 0
        A = {k: v.cpu().numpy() for k, v in a.buffers().items() if v is not None}
        B = {k: v.cpu().numpy() for k, v in b.buffers().items() if v is not None}
        for k in ("obs", "act", "rew", "done", "state", "obs_live", "reset_count"):
            assert np.array_equal(A[k], B[k]), k
        la, lb = A["logp"].ravel(), B["logp"].ravel()
        assert np.all(np.abs(la.view(np.int32).astype(np.int64) - lb.view(np.int32).astype(np.int64)) <= 2)
    o = O.Batch("u_pendulum", E, 1, SEED, t_capacity=T)
    assert o.rollout(T, rows) == 0
    g = P.Env(E, 1, "u_pendulum", SEED, t_capacity=T)
    g.rollout(T, torch.from_numpy(rows).cuda())
    buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    for k in ("obs", "act", "rew", "done"):
        assert np.array_equal(buf[k][:T], o.array(k)[:T]), k
