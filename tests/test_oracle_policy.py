"""Pins of the oracle's NEXT-N1 MLP policy (oracle/wso.cpp policy_probs, DESIGN R29) against
things other than itself: exact arithmetic on dyadic inputs, an fp64 numpy evaluation of the
same network, closed-form softmax values, and the already-pinned uniform-probability roll-out."""
import numpy as np
import pytest

import oracle as O
import wsinputs as W


def unpack(w, D, H, N):
    W1 = w[:D * H].reshape(D, H)
    b1 = w[D * H:D * H + H]
    W2 = w[D * H + H:D * H + H + H * N].reshape(H, N)
    b2 = w[D * H + H + H * N:]
    return W1, b1, W2, b2


def mlp64(w, D, H, N, obs):
    W1, b1, W2, b2 = (x.astype(np.float64) for x in unpack(w, D, H, N))
    h = np.maximum(obs.astype(np.float64) @ W1 + b1, 0.0)
    l = h @ W2 + b2
    e = np.exp(l - l.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


@pytest.mark.parametrize("D,H,N", [(4, 32, 2), (6, 64, 3), (4, 8, 5)])
def test_policy_matches_fp64_network(D, H, N):
    """fp32 FMA evaluation within fp32 rounding of the fp64 network; a transposed or dropped
    weight block would be off by O(1)."""
    w = W.policy_weights(D, H, N, seed=7, scale=1.5)
    obs = np.random.default_rng(8).standard_normal((500, D)).astype(np.float32)
    p = O.policy_probs(w, D, H, N, obs)
    ref = mlp64(w, D, H, N, obs)
    np.testing.assert_allclose(p, ref, rtol=2e-5, atol=2e-6)
    assert np.allclose(p.sum(axis=1), 1.0, atol=1e-6)


def test_policy_exact_on_dyadic_inputs():
    """Weights, biases and observations that are small multiples of 1/16: every product and
    partial sum is exact in fp32, so the logits equal the exact rational values and the
    probabilities follow from the softmax reading alone."""
    D, H, N = 4, 4, 2  # (R29': H a multiple of 4 -- the fourth hidden unit is a zero column)
    W1 = np.array([[1, -2, 0.5, 0], [0.25, 1, -1, 0], [0, 0.5, 2, 0], [-1, 0.75, 1, 0]], np.float32)
    b1 = np.array([0.5, -0.25, 0, 0], np.float32)
    W2 = np.array([[1, -1], [0.5, 0.5], [-0.25, 1], [0, 0]], np.float32)
    b2 = np.array([0, 0], np.float32)
    w = np.concatenate([W1.ravel(), b1, W2.ravel(), b2]).astype(np.float32)
    obs = np.array([[0.5, -1, 0.25, 2]], np.float32)
    h = np.maximum(obs[0].astype(np.float64) @ W1 + b1, 0)            # exact: dyadic
    l = h @ W2 + b2                                                     # exact: dyadic
    p = O.policy_probs(w, D, H, N, obs)[0]
    # softmax of two logits: p0 = 1 / (1 + exp(l1 - l0)) computed as the oracle's reading
    e = np.exp(np.float32(l - l.max()).astype(np.float64)).astype(np.float32)
    ref = e / np.float32(e[0] + e[1])
    assert np.array_equal(p, ref.astype(np.float32))
    assert abs(p[0] - 1 / (1 + np.exp(l[1] - l[0]))) < 1e-7


def test_policy_softmax_closed_forms():
    D, H, N = 2, 4, 4
    w = np.zeros(D * H + H + H * N + N, np.float32)
    p = O.policy_probs(w, D, H, N, np.ones((3, D), np.float32))
    assert np.array_equal(p, np.full((3, N), 0.25, np.float32))  # equal logits: exactly uniform
    w[-N:] = [60.0, 0.0, 0.0, 0.0]                                   # exp(-60) ~ 9e-27: tiny, not zero
    p = O.policy_probs(w, D, H, N, np.ones((1, D), np.float32))[0]
    assert p[0] > 0.999999 and np.all(p[1:] < 1e-25)
    w[-N:] = [200.0, 0.0, 0.0, 0.0]                                  # exp(-200) -> 0 in fp32
    p = O.policy_probs(w, D, H, N, np.ones((1, D), np.float32))[0]
    assert np.array_equal(p, np.array([1, 0, 0, 0], np.float32))


@pytest.mark.parametrize("env,n", [("cartpole", 2), ("acrobot", 3)])
def test_zero_policy_rollout_equals_uniform_rollout(env, n):
    """All-zero weights give exactly 1/n probabilities, so the policy roll-out must reproduce
    the (separately pinned) uniform-probability roll-out element for element."""
    E, T, H = 50, 120, 16
    D = {"cartpole": 4, "acrobot": 6}[env]
    a = O.Batch(env, E, 1, W.SEED, t_capacity=T)
    assert a.rollout_policy(T, np.zeros(D * H + H + H * n + n, np.float32), H) == 0
    b = O.Batch(env, E, 1, W.SEED, t_capacity=T)
    assert b.rollout(T, W.uniform_probs(E, 1, n)) == 0
    for k in ("act", "logp", "obs", "rew", "done", "reset_count", "stats"):
        assert np.array_equal(np.array(a.array(k)), np.array(b.array(k))), k


def test_policy_rollout_uses_the_pre_step_observation():
    """Step-by-step re-derivation: at every step the action distribution is the policy of
    the logged pre-step observation obs[t] (R12), and the logged log-prob is log p[act]."""
    E, T, H, n = 40, 60, 8, 2
    w = W.policy_weights(4, H, n, seed=9, scale=3.0)
    o = O.Batch("cartpole", E, 1, W.SEED, t_capacity=T)
    assert o.rollout_policy(T, w, H, n_threads=3) == 0
    obs = np.array(o.array("obs"))[:, :, 0, :]
    act = np.array(o.array("act"))[:, :, 0]
    lp = np.array(o.array("logp"))[:, :, 0]
    p = O.policy_probs(w, 4, H, n, obs.reshape(-1, 4)).reshape(T, E, n)
    pa = np.take_along_axis(p, act[..., None], axis=2)[..., 0]
    np.testing.assert_allclose(lp, np.log(pa.astype(np.float64)), rtol=1e-6, atol=1e-6)
    # the sampled actions follow the probabilities (frequency vs mean probability, 2400 draws)
    assert abs((act == 0).mean() - p[..., 0].mean()) < 0.03


# ---------------------------------------------------------------- Gaussian policy (R34)
def gauss_params(D, H, d, seed, log_std=-0.5):
    r = np.random.default_rng(seed)
    return np.concatenate([r.standard_normal(D * H) / np.sqrt(D), r.standard_normal(H) * 0.1,
                           r.standard_normal(H * d) / np.sqrt(H), r.standard_normal(d) * 0.1,
                           np.full(d, log_std)]).astype(np.float32)


def test_gauss_policy_rows_match_fp64_network():
    D, H, d = 3, 32, 1
    w = gauss_params(D, H, d, seed=3)
    obs = np.random.default_rng(4).standard_normal((400, D)).astype(np.float32)
    rows = O.policy_gauss_rows(w, D, H, d, obs)
    W1 = w[:D * H].reshape(D, H).astype(np.float64)
    b1 = w[D * H:D * H + H].astype(np.float64)
    W2 = w[D * H + H:D * H + H + H * d].reshape(H, d).astype(np.float64)
    b2 = w[D * H + H + H * d:D * H + H + H * d + d].astype(np.float64)
    mean = np.maximum(obs @ W1 + b1, 0) @ W2 + b2
    np.testing.assert_allclose(rows[:, :d], mean, rtol=2e-5, atol=2e-6)
    assert np.all(rows[:, d:] == np.float32(-0.5))


def test_constant_gauss_policy_equals_given_rows():
    """W2 = 0: the mean is b2 exactly, so the policy roll-out must reproduce the (pinned)
    given-row Gaussian roll-out with rows (b2 | log_std) element by element."""
    D, H, d, E, T = 3, 32, 1, 64, 120
    w = gauss_params(D, H, d, seed=5, log_std=0.3)
    w[D * H + H:D * H + H + H * d] = 0.0
    a = O.Batch("pendulum", E, 1, W.SEED, t_capacity=T)
    assert a.rollout_policy_gauss(T, w, H) == 0
    rows = np.tile(np.concatenate([w[D * H + H + H * d:D * H + H + H * d + d], w[-d:]]), (E, 1, 1)).astype(np.float32)
    b = O.Batch("pendulum", E, 1, W.SEED, t_capacity=T)
    assert b.rollout(T, rows) == 0
    for k in ("obs", "act", "logp", "rew", "done", "stats", "state"):
        assert np.array_equal(a.array(k), b.array(k)), k


def test_gauss_policy_logp_is_density_at_logged_observation():
    from scipy.stats import norm
    D, H, d, E, T = 3, 32, 1, 16, 40
    w = gauss_params(D, H, d, seed=6, log_std=-0.2)
    o = O.Batch("pendulum", E, 1, W.SEED, t_capacity=T)
    assert o.rollout_policy_gauss(T, w, H) == 0
    obs = o.array("obs")[:T].reshape(-1, D)
    rows = O.policy_gauss_rows(w, D, H, d, obs)
    act = o.array("act")[:T].reshape(-1)
    ref = norm.logpdf(act.astype(np.float64), rows[:, 0].astype(np.float64), np.exp(np.float64(-0.2)))
    np.testing.assert_allclose(o.array("logp")[:T].reshape(-1), ref, rtol=1e-5, atol=1e-5)


def test_policy_second_layer_quarter_order(oracle):
    """R29': l_i = b2_i + ((P_0 + P_1) + (P_2 + P_3)) over the four quarters of the hidden units,
    pinned by the hand-derived case of tests/golden/policy_quarter_order.txt (the former single
    sequential chain gives 2^24 there, a dropped or reordered quarter another value)."""
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "policy_quarter_order.txt")) as fh:
        rows = [l for l in fh if l.strip() and not l.startswith("#")]
    assert len(rows) == 1
    head, rest = rows[0].split("|")
    D, H, N = (int(x) for x in head.split())
    b1_s, out_s = rest.split("->")
    b1 = np.array([float(x) for x in b1_s.split()], np.float32)
    want = np.array([float(x) for x in out_s.split()], np.float32)
    W1 = np.zeros((D, H), np.float32)
    W2 = np.zeros((H, N), np.float32)
    W2[:, 0] = 1.0
    b2 = np.array([0.0, 0.5], np.float32)
    w = np.concatenate([W1.ravel(), b1, W2.ravel(), b2]).astype(np.float32)
    got = oracle.policy_logits(w, D, H, N, np.zeros((1, D), np.float32))[0]
    assert np.array_equal(got, want), (got, want)
    # probabilities follow from these logits: p_1 = exp(0.5 - (2^24 + 8)) underflows to 0
    p = oracle.policy_probs(w, D, H, N, np.zeros((1, D), np.float32))[0]
    assert p[0] == 1.0 and p[1] == 0.0
