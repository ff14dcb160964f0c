"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
on the same seeded inputs.  Bars (BJ:5, DESIGN R16/R17):
  - action indices, done flags, reset counters: bit-exact (a mismatch is only allowed on a
    draw the oracle flags as within 1e-6 of a CDF boundary);
  - fp32 observations / states / rewards: |g - o| <= 1e-5 max(|o|, s_dim) (R17); the
    expected and reported outcome is bitwise equality;
  - log-probabilities: <= 2 ulp; statistics: counts exact, sums rel. 1e-6.
"""
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


def _probs_for(env, E, A, kind="uniform", T=None, seed=1):
    n = {"cartpole": 2, "acrobot": 3, "tag": 5, "dummy": 2}.get(env, 0)
    if n:
        if kind == "uniform":
            return W.uniform_probs(E, A, n) if T is None else np.broadcast_to(W.uniform_probs(E, A, n), (T, E, A, n)).copy()
        return W.random_probs(E, A, n, seed=seed, zero_frac=0.25, T=T)
    d = {"pendulum": 1}.get(env, 0)
    return None, d


def _params(env):
    return {"surface": dict(p0=20)}.get(env, {})


SCALE = {"cartpole": [2.4, 1.0, 0.21, 1.0], "acrobot": [1, 1, 1, 1, 1, 1], "pendulum": [1, 1, 1], "dummy": [1] * 4}


def assert_close_q17(got, ref, scale=1.0, what=""):
    """R17: |g - o| <= 1e-5 * max(|o|, s_dim); returns the number of bitwise mismatches."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    both_nan = np.isnan(got) & np.isnan(ref)
    tol = 1e-5 * np.maximum(np.abs(ref), scale)
    ok = (np.abs(got - ref) <= tol) | both_nan
    if not ok.all():
        idx = np.argwhere(~ok)[:5]
        raise AssertionError(f"{what}: {int((~ok).sum())} elements beyond R17 tolerance, first {idx.tolist()}: "
                             f"gpu={got[tuple(idx[0])]} oracle={ref[tuple(idx[0])]}")
    return int(((got != ref) & ~both_nan).sum())


def ulp_diff(a, b):
    a = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    a = np.where(a < 0, -(a & 0x7FFFFFFF), a)
    b = np.where(b < 0, -(b & 0x7FFFFFFF), b)
    return np.abs(a - b)


def decode(st):
    """libws stats slab (fixed-point int64, DESIGN R20) -> float64."""
    st = np.asarray(st)
    if st.dtype == np.int64:
        st = st.astype(np.float64)
        st[:, 1] *= 2.0 ** -32
        st[:, 3] *= 2.0 ** -32
    return st


def run_pair(P, env, E, T, A=1, probs=None, step_stride=0, offset=0, E_global=0, block=0, params=None,
             max_steps=0):
    params = params or {}
    g = P.Env(E, A, env, SEED, env_offset=offset, n_envs_global=E_global, t_capacity=T, block_size=block,
              param0=params.get("p0", 0), param1=params.get("p1", 0), max_steps=max_steps)
    o = O.Batch(env, E, A, SEED, env_offset=offset, n_envs_global=E_global, t_capacity=T,
                p0=params.get("p0", 0), p1=params.get("p1", 0), max_steps=max_steps)
    g.rollout(T, torch.from_numpy(np.ascontiguousarray(probs)).cuda(), row_stride=probs.shape[-1],
              step_stride=step_stride)
    assert g.status() == 0
    amb = np.zeros((T, E, A), np.uint8)
    assert o.rollout(T, probs, row_stride=probs.shape[-1], step_stride=step_stride, ambiguous=amb, n_threads=8) == 0
    buf = {k: (v.cpu().numpy() if v is not None else None) for k, v in g.buffers().items()}
    return g, o, buf, amb


def compare(buf, o, amb, env, T, exact_float=True):
    """Full comparison; returns a dict of mismatch counts (bitwise) for reporting."""
    act_g, act_o = buf["act"][:T], np.array(o.array("act"))
    if act_g.dtype == np.int32:
        diff = act_g != act_o
        assert not (diff & (amb == 0)).any(), f"{env}: {int(diff.sum())} action mismatches outside the R16 band"
        assert not diff.any(), f"{env}: ambiguous-draw mismatches present ({int(diff.sum())}); adoption needed"
    else:
        assert_close_q17(act_g, act_o, 1.0, f"{env} act")
    assert np.array_equal(buf["done"][:T], np.array(o.array("done"))), f"{env}: done flags differ"
    assert np.array_equal(buf["reset_count"], np.array(o.array("reset_count"))), f"{env}: reset counters differ"
    assert np.array_equal(buf["ep_step"], np.array(o.array("ep_step")))
    scale = np.array(SCALE.get(env, [1.0]), np.float64)
    obs_o = np.array(o.array("obs"))
    sc = scale if scale.size == obs_o.shape[-1] else 1.0
    n_obs = assert_close_q17(buf["obs"][:T], obs_o, sc, f"{env} obs")
    n_rew = assert_close_q17(buf["rew"][:T], np.array(o.array("rew")), 1.0, f"{env} rew")
    lp_g, lp_o = buf["logp"][:T], np.array(o.array("logp"))
    assert np.array_equal(np.isnan(lp_g), np.isnan(lp_o))
    fin = ~np.isnan(lp_o)
    assert ulp_diff(lp_g[fin], lp_o[fin]).max(initial=0) <= 2, f"{env}: logp beyond 2 ulp"
    st_g, st_o = decode(buf["stats"][:T]), np.array(o.array("stats"))
    assert np.array_equal(st_g[:, [0, 2]], st_o[:, [0, 2]]), f"{env}: episode counts / lengths differ"
    # R20: each per-replica value is rounded to a multiple of 2^-32 at most (exact for
    # |r| >= 2^-8); the oracle's fp64 sums are exact at these magnitudes
    n_terms = float(buf["rew"].shape[1] * buf["rew"].shape[2])
    np.testing.assert_allclose(st_g[:, [1, 3]], st_o[:, [1, 3]], rtol=1e-12, atol=n_terms * 2.0 ** -32)
    if exact_float:
        assert n_obs == 0 and n_rew == 0, f"{env}: {n_obs} obs / {n_rew} rew not bitwise equal (within R17)"
    return {"obs_bitwise_mismatch": n_obs, "rew_bitwise_mismatch": n_rew, "ambiguous": int(amb.sum())}


# ------------------------------------------------------------------------------ primitives
def test_philox_device_known_answers(P):
    rows = torch.tensor([[0, 0, 0, 0, 0, 0],
                         [0xFFFFFFFF] * 6,
                         [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0]],
                        dtype=torch.int64).to(torch.int32).cuda()
    out = P.ws_test_philox(rows).cpu().numpy().view(np.uint32)
    for r in range(3):
        ref = O.philox(rows[r, :4].cpu().numpy().view(np.uint32), rows[r, 4:].cpu().numpy().view(np.uint32))
        assert list(out[r]) == list(ref)
    # random counters against the oracle
    rng = np.random.default_rng(0)
    rr = rng.integers(0, 2**32, (4096, 6), dtype=np.uint64).astype(np.uint32)
    out = P.ws_test_philox(torch.from_numpy(rr.view(np.int32)).cuda()).cpu().numpy().view(np.uint32)
    for i in range(0, 4096, 97):
        assert list(out[i]) == list(O.philox(rr[i, :4], rr[i, 4:]))


@pytest.mark.parametrize("p", [[0.5, 0.5], [0.1, 0.2, 0.7], [1 / 3, 1 / 3, 1 / 3], [0.0, 0.3, 0.0, 0.7],
                               [1.0, 0.0], [0.2] * 5, [3.0, 1.0], [1e-7, 1.0, 0.0, 2.5, 1e-3, 0.4, 0.0, 9.0]])
def test_sampler_exhaustive_grid_matches_oracle(P, p):
    counts = P.ws_test_sample_grid(torch.tensor(p, dtype=torch.float32).cuda()).cpu().numpy()
    ref, n_amb = O.sample_grid(p)
    assert counts[-1] == 0, "hoisted threshold search disagrees with the direct search"
    assert int(np.abs(counts[:-1] - ref).sum()) <= 2 * n_amb
    assert np.array_equal(counts[:-1], ref), f"grid counts differ: {counts[:-1]} vs {ref} ({n_amb} ambiguous)"


# ------------------------------------------------------------------------------ C1 / C2 CartPole
def test_c1_cartpole_parity(P):
    w = W.CONFIGS["C1"]
    probs = W.workload_probs(w)
    g, o, buf, amb = run_pair(P, "cartpole", w.n_envs, w.T, probs=probs)
    compare(buf, o, amb, "cartpole", w.T)


def test_c2_cartpole_full_size_parity(P):
    """BASELINE config C2 at full size (10K x 1000) in bench.py's launch configuration."""
    w = W.CONFIGS["C2"]
    probs = W.workload_probs(w)
    g, o, buf, amb = run_pair(P, "cartpole", w.n_envs, w.T, probs=probs)
    compare(buf, o, amb, "cartpole", w.T)


def test_cartpole_random_probs_per_step(P):
    """Per-step probability stream (step_stride != 0) with zeros and unnormalised rows."""
    E, T = 300, 120
    probs = W.random_probs(E, 1, 2, seed=3, zero_frac=0.2, T=T)
    g, o, buf, amb = run_pair(P, "cartpole", E, T, probs=probs, step_stride=E * 2)
    compare(buf, o, amb, "cartpole", T)


@pytest.mark.parametrize("env,A,n,params", [("acrobot", 1, 3, {}), ("dummy", 1, 2, {}), ("tag", 37, 5, {"p0": 9, "p1": 6})])
def test_discrete_per_step_probs(P, env, A, n, params):
    """Per-step probability rows (step_stride != 0) for the other discrete envs: the plan
    kernel's strided path (lane envs) and the tag kernel's per-step CDF variant."""
    E, T = 80, 96
    probs = W.random_probs(E, A, n, seed=21, zero_frac=0.25, T=T)
    g, o, buf, amb = run_pair(P, env, E, T, A=A, probs=probs, step_stride=E * A * n, params=params)
    compare(buf, o, amb, env, T)


@pytest.mark.parametrize("env,d,params", [("pendulum", 1, {}), ("surface", 20, {"p0": 20}), ("surface", 3, {"p0": 3})])
def test_gaussian_per_step_params(P, env, d, params):
    """Per-step Gaussian heads (step_stride != 0): both Gaussian plan kernels' strided paths."""
    E, T = 64, 70
    ls = float(np.log(0.025)) if env == "surface" else 0.0
    probs = np.stack([W.gaussian_params(E, 1, d, 0.0, ls, jitter=0.3, seed=100 + t) for t in range(T)])
    g, o, buf, amb = run_pair(P, env, E, T, probs=probs, step_stride=E * 2 * d, params=params)
    compare(buf, o, amb, env, T)


@pytest.mark.parametrize("env,A,n,step_stride", [("cartpole", 1, 2, False), ("acrobot", 1, 3, False),
                                                 ("tag", 20, 5, False), ("cartpole", 1, 2, True),
                                                 ("tag", 20, 5, True)])
def test_invalid_probability_rows_in_rollout(P, env, A, n, step_stride):
    """R13/R19 inside a fused roll-out: rows with p < 0, NaN or zero sum give act -1 and NaN
    logp, the replica (tag: the whole replica step) does not advance, rew = done = 0, and the
    status is WS_ERR_INVALID_PROBS -- element for element as the oracle."""
    E, T = 96, 60
    probs = W.random_probs(E, A, n, seed=13, zero_frac=0.2, T=T if step_stride else None)
    bad = probs[7] if step_stride else probs
    bad[5, 0, 0] = -1.0
    bad[40, A - 1, 1] = np.nan
    bad[77, 0, :] = 0.0
    ss = E * A * n if step_stride else 0
    g = P.Env(E, A, env, SEED, t_capacity=T)
    g.rollout(T, torch.from_numpy(np.ascontiguousarray(probs)).cuda(), row_stride=n, step_stride=ss)
    assert g.status() == P._abi.INVALID_PROBS
    o = O.Batch(env, E, A, SEED, t_capacity=T)
    amb = np.zeros((T, E, A), np.uint8)
    assert o.rollout(T, probs, row_stride=n, step_stride=ss, ambiguous=amb, n_threads=4) == 0
    assert o.synchronize() == P._abi.INVALID_PROBS
    buf = {k: (v.cpu().numpy() if v is not None else None) for k, v in g.buffers().items()}
    act = buf["act"][:T]
    assert (act[:, [5, 40, 77]] == -1).any()
    compare(buf, o, amb, env, T)


def test_fixed_actions_64_steps(P):
    """BJ:5: fp32 states and rewards within 1e-5 relative per step for fixed action
    sequences over 64 steps (ws_step with given actions), E = 1024."""
    for env, n in (("cartpole", 2), ("acrobot", 3)):
        E, T = 1024, 64
        acts = W.action_table(T, E, 1, n, seed=11)
        g = P.Env(E, 1, env, SEED, t_capacity=T)
        o = O.Batch(env, E, 1, SEED, t_capacity=T)
        for t in range(T):
            g.step(torch.from_numpy(acts[t]).cuda())
            assert o.step(acts[t]) == 0
            st_g = g.buffers()["state"].cpu().numpy()
            assert_close_q17(st_g, np.array(o.array("state")), np.array(SCALE[env][:4] if env == "cartpole" else 1.0),
                             f"{env} state t={t}")
        assert g.status() == 0
        buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
        assert np.array_equal(buf["done"], np.array(o.array("done")))
        n_obs = assert_close_q17(buf["obs"], np.array(o.array("obs")), 1.0, f"{env} obs")
        n_rew = assert_close_q17(buf["rew"], np.array(o.array("rew")), 1.0, f"{env} rew")
        assert n_obs == 0 and n_rew == 0
        assert np.isnan(buf["logp"]).all()  # R27 given actions


# ------------------------------------------------------------------------------ other envs
@pytest.mark.parametrize("env,E,A,T,params", [
    ("acrobot", 512, 1, 500, {}),
    ("pendulum", 512, 1, 400, {}),
    ("dummy", 333, 1, 250, {}),
    ("tag", 24, 100, 200, {}),
    ("tag", 16, 37, 120, {"p0": 7, "p1": 5}),
    ("surface", 256, 1, 200, {"p0": 20}),
    ("surface", 200, 1, 150, {"p0": 2}),
])
def test_env_parity(P, env, E, A, T, params):
    if env in ("pendulum", "surface"):
        d = params.get("p0", 1) if env == "surface" else 1
        probs = W.gaussian_params(E, A, d, 0.0, float(np.log(0.025)) if env == "surface" else 0.0, jitter=0.3, seed=4)
    else:
        n = {"acrobot": 3, "dummy": 2, "tag": 5}[env]
        probs = W.random_probs(E, A, n, seed=5, zero_frac=0.2)
    g, o, buf, amb = run_pair(P, env, E, T, A=A, probs=probs, params=params)
    compare(buf, o, amb, env, T)


@pytest.mark.parametrize("D", [20, 16, 8, 3])
def test_surface_goal_reached(P, D):
    """Per-step Gaussian heads that steer replicas into the goal ball: step 0 cancels each
    replica's reset offsets in q_2.. (read from the oracle's initial state), then q0 / q1 drift
    from minimum B toward minimum A (the goal) with tiny noise, so first episodes end at the goal
    (bonus reward, done bit 0), restart and later truncate; every third replica only diffuses and
    one replica's head is non-finite.  The segmented kernel's fast 4-step trips must hand every
    trip that may touch the goal ball (or a truncation / invalid action) to the exact per-step
    path -- element for element as the oracle."""
    E, T, ms = 300, {20: 203, 8: 197, 3: 200, 16: 196}[D], 150  # T % 8 = 3, 5, 0, 4: every tail path of the trip loops
    o = O.Batch("surface", E, 1, SEED, t_capacity=T, p0=D, max_steps=ms)
    q0 = np.array(o.array("state")).reshape(E, D)
    probs = np.zeros((T, E, 1, 2 * D), np.float32)
    probs[..., D:] = np.log(1e-6)
    probs[:, :, 0, 0] = -0.05 * 1.181 / 1.414
    probs[:, :, 0, 1] = 0.05
    if D > 2:
        probs[0, :, 0, 2:D] = -q0[:, 2:]
    probs[:, ::3, 0, :2] = 0.0  # every third replica only diffuses: truncated at max_steps
    probs[:, 7, 0, 0] = np.nan  # an invalid head: replica 7 never advances (sticky error)
    g = P.Env(E, 1, "surface", SEED, t_capacity=T, param0=D, max_steps=ms)
    g.rollout(T, torch.from_numpy(probs).cuda(), row_stride=2 * D, step_stride=E * 2 * D)
    amb = np.zeros((T, E, 1), np.uint8)
    assert o.rollout(T, probs, row_stride=2 * D, step_stride=E * 2 * D, ambiguous=amb, n_threads=8) == 0
    assert g.status() == o.synchronize() != 0
    buf = {k: (v.cpu().numpy() if v is not None else None) for k, v in g.buffers().items()}
    compare(buf, o, amb, "surface", T)
    assert int((buf["done"][:T] & 1).sum()) > E // 2  # goal terminations happened
    assert int((buf["done"][:T] & 2).sum()) > E // 4  # and truncations


@pytest.mark.parametrize("cfg,windows", [("C3a", [(0, 128), (49_936, 128), (99_872, 128)]),
                                         ("C3b", [(0, 128), (77_000, 128)]),
                                         ("C4", [(0, 8), (992, 8)]),
                                         ("C5", [(0, 64), (1936, 64)])])
def test_full_size_configs_sampled(P, cfg, windows):
    """BASELINE configs C3-C5 at full size on one GPU; the oracle recomputes sampled replica
    windows exactly (replicas are independent; streams are keyed by the global index)."""
    w = W.CONFIGS[cfg]
    probs = W.workload_probs(w)
    params = {"C4": {"p0": 20, "p1": 10}, "C5": {"p0": 20}}.get(cfg, {})
    g = P.Env(w.n_envs, w.n_agents, w.env, SEED, t_capacity=w.T, param0=params.get("p0", 0),
              param1=params.get("p1", 0))
    g.rollout(w.T, torch.from_numpy(probs).cuda())
    assert g.status() == 0
    buf = g.buffers()
    for off, n in windows:
        o = O.Batch(w.env, n, w.n_agents, SEED, env_offset=off, n_envs_global=w.n_envs, t_capacity=w.T,
                    p0=params.get("p0", 0), p1=params.get("p1", 0))
        amb = np.zeros((w.T, n, w.n_agents), np.uint8)
        assert o.rollout(w.T, probs[off:off + n], ambiguous=amb, n_threads=8) == 0
        sub = {k: (v[:, off:off + n].cpu().numpy() if k in ("obs", "act", "logp", "rew", "done") else
                   v[off:off + n].cpu().numpy()) for k, v in buf.items() if v is not None and k != "stats"}
        sub["stats"] = np.array(o.array("stats"))  # stats cover all replicas: checked separately
        compare(sub, o, amb, w.env, w.T)


@pytest.mark.parametrize("env,n", [("cartpole", 2), ("acrobot", 3), ("dummy", 2)])
def test_throughput_build_parity(P, env, n):
    """Above 148*4*32 replicas the fused discrete roll-out switches to its throughput build
    (other register budget and statistics window depth): full element-wise parity there too."""
    E, T = 20_000, 72
    probs = W.random_probs(E, 1, n, seed=31, zero_frac=0.1)
    g, o, buf, amb = run_pair(P, env, E, T, probs=probs)
    compare(buf, o, amb, env, T)


@pytest.mark.parametrize("env,n", [("cartpole", 2), ("acrobot", 3), ("dummy", 2)])
@pytest.mark.parametrize("max_steps", [1, 3, 7, 8, 9])
def test_short_truncation_limits(P, env, n, max_steps):
    """Truncation every few steps (R10): below 8 the fused CartPole loop leaves its 8-step
    refill window (fast path) for the per-step reset check; done bits, reset counters and
    statistics as the oracle."""
    E, T = 70, 45
    probs = W.random_probs(E, 1, n, seed=51, zero_frac=0.1)
    g, o, buf, amb = run_pair(P, env, E, T, probs=probs, max_steps=max_steps)
    compare(buf, o, amb, env, T)


@pytest.mark.parametrize("E,T", [(1, 1), (1, 37), (33, 1), (33, 9), (31, 64)])
def test_tiny_shapes(P, E, T):
    """Degenerate sizes: one replica, one step, a warp plus one replica, a partial warp."""
    probs = W.random_probs(E, 1, 2, seed=52, zero_frac=0.1)
    g, o, buf, amb = run_pair(P, "cartpole", E, T, probs=probs)
    compare(buf, o, amb, "cartpole", T)


def test_write_logp_off(P):
    """write_logp = 0: the log-prob slab is never written; everything else is unchanged."""
    E, T = 200, 50
    probs = W.random_probs(E, 1, 2, seed=53, zero_frac=0.1)
    g = P.Env(E, 1, "cartpole", SEED, t_capacity=T, write_logp=False)
    lp = g.buffers()["logp"]
    if lp is not None:
        lp.fill_(7.0)
    g.rollout(T, torch.from_numpy(probs).cuda())
    assert g.status() == 0
    o = O.Batch("cartpole", E, 1, SEED, t_capacity=T)
    assert o.rollout(T, probs) == 0
    buf = {k: (v.cpu().numpy() if v is not None else None) for k, v in g.buffers().items()}
    for k in ("act", "obs", "rew", "done", "reset_count", "ep_step"):
        assert np.array_equal(buf[k][:T] if buf[k].ndim > 1 else buf[k], np.array(o.array(k))[:T]
                              if np.array(o.array(k)).ndim > 1 else np.array(o.array(k))), k
    if buf["logp"] is not None:
        assert (buf["logp"] == 7.0).all()


# ------------------------------------------------------------------------------ invariants
def test_launch_shape_and_sharding_invariance(P):
    """S:148 / S:178 analog: per-replica outputs identical for every CTA size and for any
    split of the replicas into shards (global-index-keyed streams, R15)."""
    E, T = 1000, 300
    probs = W.uniform_probs(E, 1, 2)
    ref = None
    for block in (32, 64, 128, 256):
        g = P.Env(E, 1, "cartpole", SEED, t_capacity=T, block_size=block)
        g.rollout(T, torch.from_numpy(probs).cuda())
        b = {k: v.cpu().numpy() for k, v in g.buffers().items()}
        if ref is None:
            ref = b
        for k in ("obs", "act", "logp", "rew", "done", "state", "reset_count", "stats"):
            assert np.array_equal(b[k], ref[k]), (block, k)  # stats: exact integers (R20)
    parts = []
    for off, n in ((0, 333), (333, 334), (667, 333)):
        g = P.Env(n, 1, "cartpole", SEED, env_offset=off, n_envs_global=E, t_capacity=T)
        g.rollout(T, torch.from_numpy(probs[off:off + n]).cuda())
        parts.append({k: v.cpu().numpy() for k, v in g.buffers().items()})
    for k in ("obs", "act", "logp", "rew", "done"):
        assert np.array_equal(np.concatenate([p[k] for p in parts], axis=1), ref[k]), k
    st = sum(p["stats"] for p in parts)
    assert np.array_equal(st, ref["stats"])  # bit-identical merged statistics (R20)


def test_single_step_path_equals_fused_rollout(P):
    """ws_sample + ws_step (one launch each per step) == ws_rollout (one fused kernel)."""
    for env, A, n in (("cartpole", 1, 2), ("acrobot", 1, 3), ("tag", 50, 5), ("pendulum", 1, 0)):
        E, T = 96, 80
        probs = (W.random_probs(E, A, n, seed=9, zero_frac=0.2) if n else W.gaussian_params(E, A, 1, 0.0, 0.0, 0.3))
        pt = torch.from_numpy(probs).cuda()
        a = P.Env(E, A, env, SEED, t_capacity=T)
        a.rollout(T, pt)
        b = P.Env(E, A, env, SEED, t_capacity=T)
        for _ in range(T):
            b.sample(pt)
            b.step()
        ba = {k: v.cpu().numpy() for k, v in a.buffers().items()}
        bb = {k: v.cpu().numpy() for k, v in b.buffers().items()}
        for k in ("obs", "act", "logp", "rew", "done", "state", "reset_count", "ep_step", "obs_live", "stats"):
            assert np.array_equal(ba[k], bb[k], equal_nan=True), (env, k)


def test_zero_steady_state_allocation_and_stable_addresses(P):
    """S:86 / S:585: after the first roll-out no allocation; buffer addresses stable."""
    E, T = 2048, 100
    probs = torch.full((E, 1, 2), 0.5, device="cuda")
    g = P.Env(E, 1, "cartpole", SEED)
    g.rollout(T, probs)
    n0 = g.allocator.n_alloc
    ptrs = {k: v.data_ptr() for k, v in g.buffers().items()}
    for _ in range(20):
        g.rollout(T, probs)
    g.synchronize()
    assert g.allocator.n_alloc == n0
    assert {k: v.data_ptr() for k, v in g.buffers().items()} == ptrs
    # reset_count == number of done flags across the whole history of this handle
    g2 = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    total = torch.zeros(E, dtype=torch.int64, device="cuda")
    for _ in range(5):
        g2.rollout(T, probs)
        total += (g2.buffers()["done"] != 0).sum(0)
    assert torch.equal(total.to(torch.int64), g2.buffers()["reset_count"].to(torch.int64))


def test_invalid_inputs_are_sticky_errors(P):
    E = 8
    g = P.Env(E, 1, "cartpole", SEED, t_capacity=4)
    acts = torch.zeros((E, 1), dtype=torch.int32, device="cuda")
    acts[3] = 7
    s0 = g.buffers()["state"].clone()
    g.step(acts)
    assert g.status() == P._abi.INVALID_ACTION
    st = g.buffers()["state"]
    assert torch.equal(st[3], s0[3]) and not torch.equal(st[0], s0[0])
    assert g.buffers()["rew"][0, 3, 0].item() == 0.0
    g.step(torch.zeros((E, 1), dtype=torch.int32, device="cuda"))
    assert g.status() == P._abi.INVALID_ACTION  # sticky
    g.reset()
    assert g.status() == 0
    bad = torch.full((E, 1, 2), 0.5, device="cuda")
    bad[5, 0, 0] = -1.0
    g.rollout(4, bad)
    assert g.status() == P._abi.INVALID_PROBS
    b = g.buffers()
    assert (b["act"][:, 5] == -1).all() and (b["rew"][:, 5] == 0).all()
    with pytest.raises(P.WSError):
        g.rollout(5, bad)  # T beyond the store capacity
    with pytest.raises(P.WSError):
        g2 = P.Env(E, 1, "cartpole", SEED)
        g2.step(None)  # ws_step(NULL) without ws_sample


def test_rollout_host_e2e(P):
    E, T = 512, 200
    probs = torch.full((E, 1, 2), 0.5).pin_memory()
    g = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    st = g.rollout_host(T, probs)
    o = O.Batch("cartpole", E, 1, SEED, t_capacity=T)
    o.rollout(T, probs.numpy())
    ref = np.array(o.array("stats")).sum(0)
    assert st.episodes == ref[0] and st.sum_length == ref[2]
    assert abs(st.sum_return - ref[1]) <= 1e-9 * max(1, ref[1])


def test_rollout_host_pipelined_equals_synchronous(P):
    """ws_rollout_host_submit / _wait (two deep): a chain of six roll-outs with per-step host
    probabilities (the next submitted before the previous is awaited) returns, roll-out by
    roll-out, the statistics of ws_rollout_host on an identical handle, and leaves the same live
    state; waiting on an empty slot or resubmitting a pending one is WS_ERR_BAD_STATE."""
    E, T, n = 700, 150, 6
    hp = [torch.from_numpy(W.random_probs(E, 1, 2, seed=300 + k, zero_frac=0.1)).pin_memory() for k in range(n)]
    a = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    b = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    got = []
    a.rollout_host_submit(T, hp[0], 0)
    for k in range(n):
        if k + 1 < n:
            a.rollout_host_submit(T, hp[k + 1], (k + 1) & 1)
        got.append(a.rollout_host_wait(k & 1))
    for k in range(n):
        ref = b.rollout_host(T, hp[k])
        assert (got[k].episodes, got[k].sum_length, got[k].sum_return) == (ref.episodes, ref.sum_length, ref.sum_return), k
    for key in ("state", "reset_count", "ep_step", "obs_live"):
        assert torch.equal(a.buffers()[key], b.buffers()[key]), key
    with pytest.raises(P.WSError):
        a.rollout_host_wait(0)
    a.rollout_host_submit(T, hp[0], 1)
    with pytest.raises(P.WSError):
        a.rollout_host_submit(T, hp[0], 1)
    a.rollout_host_wait(1)


def test_unaligned_rollouts_and_chunks(P):
    """Roll-outs whose start step t0 is not a multiple of 4 (prologue / epilogue paths) and
    whose length is not a multiple of 32 (partial statistics windows), chained across calls
    (episodes span chunks), against the same chain on the oracle."""
    E = 200
    probs = W.uniform_probs(E, 1, 2)
    g = P.Env(E, 1, "cartpole", SEED, t_capacity=64)
    o = O.Batch("cartpole", E, 1, SEED, t_capacity=64)
    for T in (37, 50, 3, 64, 29):
        g.rollout(T, torch.from_numpy(probs).cuda())
        assert o.rollout(T, probs) == 0
        buf = {k: v.cpu().numpy() for k, v in g.buffers().items()}
        for k in ("obs", "act", "logp", "rew", "done"):
            assert np.array_equal(buf[k][:T], np.array(o.array(k))[:T]), (T, k)
        for k in ("state", "reset_count", "ep_step", "ep_ret", "obs_live"):
            assert np.array_equal(buf[k], np.array(o.array(k))), (T, k)
        st_o = np.array(o.array("stats"))[:T]
        st_g = decode(buf["stats"][:T])
        assert np.array_equal(st_g, st_o)  # integer rewards: exact


@pytest.mark.parametrize("E,block", [(10000, 128), (10000, 256), (130, 256), (33, 64)])
def test_statistics_exact_with_partial_ctas(P, E, block):
    """Exact fixed-point statistics (R20) equal the oracle's for grids whose last CTA has
    dead warps and a partial warp (shadow lanes)."""
    T = 200
    probs = W.uniform_probs(E, 1, 2)
    g = P.Env(E, 1, "cartpole", SEED, t_capacity=T, block_size=block)
    g.rollout(T, torch.from_numpy(probs).cuda())
    o = O.Batch("cartpole", E, 1, SEED, t_capacity=T)
    assert o.rollout(T, probs, n_threads=8) == 0
    assert np.array_equal(g.stats_f64(T).cpu().numpy(), np.array(o.array("stats")))
