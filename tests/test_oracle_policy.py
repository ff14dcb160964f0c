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
    D, H, N = 4, 3, 2
    W1 = np.array([[1, -2, 0.5], [0.25, 1, -1], [0, 0.5, 2], [-1, 0.75, 1]], np.float32)
    b1 = np.array([0.5, -0.25, 0], np.float32)
    W2 = np.array([[1, -1], [0.5, 0.5], [-0.25, 1]], np.float32)
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
    D, H, N = 2, 2, 4
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
