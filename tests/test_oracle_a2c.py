"""Pins of the NEXT-N2 actor-critic oracle (oracle/a2c.py, DESIGN R31) against things other
than itself: central finite differences of the loss, torch autograd of an independently
written network and loss (torch.distributions.Categorical), torch.optim.Adam with
clip_grad_norm_, closed forms, and the SPEC a2c_update examples."""
import numpy as np
import pytest
import torch

from oracle import a2c as OA

SHAPES = [(4, 8, 2), (6, 16, 3), (4, 64, 2)]


def batch(D, H, n, B, seed, scale=0.7):
    r = np.random.default_rng(seed)
    params = r.standard_normal(OA.n_params(D, H, n)) * scale
    obs = r.standard_normal((B, D))
    act = r.integers(0, n, B)
    adv = r.standard_normal(B)
    ret = r.standard_normal(B)
    return params, obs, act, adv, ret


@pytest.mark.parametrize("D,H,n", SHAPES)
def test_grad_matches_central_differences(D, H, n):
    """Every component of the hand-derived backward equals the central difference of the
    loss (fp64; step 1e-6; the ReLU kinks are measure-zero for random inputs)."""
    params, obs, act, adv, ret = batch(D, H, n, 40, seed=D * 100 + H)
    c_v, c_e = 0.5, 0.03
    g = OA.grad(params, obs, act, adv, ret, D, H, n, c_v, c_e)
    fd = np.zeros_like(g)
    h = 1e-6
    for i in range(params.size):
        pp = params.copy(); pp[i] += h
        pm = params.copy(); pm[i] -= h
        fd[i] = (OA.loss(pp, obs, act, adv, ret, D, H, n, c_v, c_e)[0] -
                 OA.loss(pm, obs, act, adv, ret, D, H, n, c_v, c_e)[0]) / (2 * h)
    np.testing.assert_allclose(g, fd, rtol=1e-5, atol=1e-8)


def torch_net_loss(params, obs, act, adv_hat, ret, D, H, n, c_v, c_e, B=None):
    """Independent formulation: torch.nn.functional layers + Categorical(logits)."""
    p = torch.tensor(params, dtype=torch.float64, requires_grad=True)
    sizes = [D * H, H, H * n, n, H, 1]
    W1, b1, W2, b2, wv, bv = torch.split(p, sizes)
    o = torch.tensor(obs, dtype=torch.float64)
    h = torch.relu(torch.nn.functional.linear(o, W1.view(D, H).t(), b1))
    logits = torch.nn.functional.linear(h, W2.view(H, n).t(), b2)
    V = torch.nn.functional.linear(h, wv.view(1, H), bv).squeeze(1)
    dist = torch.distributions.Categorical(logits=logits)
    a = torch.tensor(act, dtype=torch.int64)
    ok = ((a >= 0) & (a < n)).double()
    a = a.clamp(0, n - 1)
    Ah = torch.tensor(adv_hat, dtype=torch.float64)
    R = torch.tensor(ret, dtype=torch.float64)
    B = len(act) if B is None else B
    L = (-(dist.log_prob(a) * Ah * ok).sum() + c_v * (((V - R) ** 2) * ok).sum()
         - c_e * (dist.entropy() * ok).sum()) / B
    L.backward()
    return L.item(), p.grad.numpy()


@pytest.mark.parametrize("D,H,n", SHAPES)
def test_grad_and_loss_match_torch_autograd(D, H, n):
    params, obs, act, adv, ret = batch(D, H, n, 300, seed=7 + n)
    act[::17] = -1  # R13 invalid rows contribute nothing
    L_t, g_t = torch_net_loss(params, obs, act, adv, ret, D, H, n, 0.5, 0.01, B=400)
    L = OA.loss(params, obs, act, adv, ret, D, H, n, 0.5, 0.01, batch=400)[0]
    g = OA.grad(params, obs, act, adv, ret, D, H, n, 0.5, 0.01, batch=400)
    assert abs(L - L_t) < 1e-12 * max(1.0, abs(L_t))
    np.testing.assert_allclose(g, g_t, rtol=1e-10, atol=1e-13)


def test_clip_and_adam_match_torch_optim():
    """Five Adam steps against torch.optim.Adam (exact up to rounding), and the clip against
    torch.nn.utils.clip_grad_norm_ (which divides by norm + 1e-6: agreement to ~1e-6/norm)."""
    r = np.random.default_rng(3)
    P = 50
    p = r.standard_normal(P)
    m = np.zeros(P); v = np.zeros(P)
    tp = torch.tensor(p.copy(), requires_grad=True)
    opt = torch.optim.Adam([tp], lr=3e-3, betas=(0.9, 0.999), eps=1e-8)
    for k in range(1, 6):
        g = r.standard_normal(P) * (3.0 if k % 2 else 0.01)
        gc = OA.clip(g, 0.5)
        tg = torch.tensor(g.copy(), requires_grad=False)
        tq = torch.zeros(P, dtype=torch.float64, requires_grad=True)
        tq.grad = tg.clone()
        torch.nn.utils.clip_grad_norm_([tq], 0.5)
        np.testing.assert_allclose(gc, tq.grad.numpy(), rtol=3e-6, atol=0)
        p, m, v = OA.adam(p, gc, m, v, k, 3e-3)
        tp.grad = torch.tensor(gc.copy())
        opt.step()
        np.testing.assert_allclose(p, tp.detach().numpy(), rtol=1e-12, atol=1e-14)


def test_adam_closed_forms():
    """a zero gradient leaves the parameters unchanged; at step 1 bias correction
    makes every update lr * g / (|g| + eps) -- i.e. lr * sign(g) for |g| >> eps."""
    p = np.linspace(-1, 1, 9)
    p2, _, _ = OA.adam(p, np.zeros(9), np.zeros(9), np.zeros(9), 1, 1e-2)
    assert np.array_equal(p2, p)
    g = np.array([3.0, -0.5, 1e-3, -2e-4, 7.0, 1.0, -1.0, 0.25, -4.0])
    p2, _, _ = OA.adam(p, g, np.zeros(9), np.zeros(9), 1, 1e-2)
    np.testing.assert_allclose(p - p2, 1e-2 * np.sign(g), rtol=1e-4)
    assert np.linalg.norm(OA.clip(g, 0.5)) == pytest.approx(0.5, rel=1e-15)
    assert np.array_equal(OA.clip(g * 1e-3, 0.5), g * 1e-3)


def test_normalize_moments_and_degenerate_rule():
    a = np.random.default_rng(1).standard_normal(1000) * 3 + 5
    ah = OA.normalize(a)
    assert abs(ah.mean()) < 1e-12 and abs(ah.std() - 1) < 1e-12
    c = np.full(10, 2.5)
    assert np.array_equal(OA.normalize(c), c)  # sigma < 1e-8: skipped (R31)
    # shard-wise moments summed == moments of the whole batch (the DP all-reduce)
    s1, s2 = OA.moments(a[:400]), OA.moments(a[400:])
    np.testing.assert_allclose(OA.normalize(a[:400], (s1[0] + s2[0], s1[1] + s2[1]), 1000), ah[:400],
                               rtol=1e-12, atol=1e-12)


def test_uniform_policy_entropy_closed_form():
    """W2 = 0, b2 = 0: pi uniform, entropy term = -c_e log n exactly; with zero advantages
    and V == returns (wv = 0, bv = R) every policy and value gradient vanishes (S:404 --
    and the uniform policy is the entropy maximum, so the entropy gradient vanishes too)."""
    D, H, n = 4, 8, 3
    params, obs, act, adv, ret = batch(D, H, n, 64, seed=11)
    W1, b1, W2, b2, wv, bv = OA.unpack(params, D, H, n)
    q = params.copy()
    o = D * H + H
    q[o:o + H * n + n] = 0.0
    q[o + H * n + n:o + H * n + n + H] = 0.0
    q[-1] = 0.75
    ret = np.full(64, 0.75)
    L = OA.loss(q, obs, act, np.zeros(64), ret, D, H, n, 0.5, 0.2)
    assert L[1] == 0.0 and L[2] == 0.0
    assert L[3] == pytest.approx(-0.2 * np.log(n), rel=1e-15)
    g = OA.grad(q, obs, act, np.zeros(64), ret, D, H, n, 0.5, 0.2)
    assert np.abs(g).max() < 1e-15


def test_positive_advantage_raises_its_action_probability():
    """entropy coefficient 0, uniform policy, positive advantage on action 0 ->
    pi(action 0) strictly increases after the update, for every observation."""
    D, H, n = 4, 8, 2
    params, obs, _, _, _ = batch(D, H, n, 32, seed=5)
    o = D * H + H
    params[o:o + H * n + n] = 0.0
    act = np.zeros(32, np.int64)
    adv = np.ones(32)
    V = OA.values(params, obs, D, H, n)
    g = OA.grad(params, obs, act, adv, V, D, H, n, 0.5, 0.0)
    p2, _, _ = OA.adam(params, OA.clip(g, 0.5), np.zeros_like(g), np.zeros_like(g), 1, 1e-2)
    pi0 = OA.forward(params, obs, D, H, n)[3][:, 0]
    pi1 = OA.forward(p2, obs, D, H, n)[3][:, 0]
    assert np.all(pi0 == 0.5) and np.all(pi1 > 0.5)


def test_update_decreases_loss_on_frozen_batch():
    """lr = 1e-4, 10 random batches, the loss after the update is lower >= 9 times."""
    D, H, n = 4, 16, 2
    wins = 0
    for s in range(10):
        params, obs, act, adv, ret = batch(D, H, n, 256, seed=100 + s)
        z = np.zeros_like(params)
        p2, _, _, _, L0 = OA.update(params, z, z, 1, obs, act, adv, ret, D, H, n, lr=1e-4)
        L1 = OA.loss(p2, obs, act, OA.normalize(adv), ret, D, H, n, 0.5, 0.01)
        wins += L1[0] < L0[0]
    assert wins >= 9


# ---------------------------------------------------------------- PPO (R33)
def torch_ppo_loss(params, obs, act, adv_hat, ret, logp_old, D, H, n, c_v, c_e, eps):
    p = torch.tensor(params, dtype=torch.float64, requires_grad=True)
    W1, b1, W2, b2, wv, bv = torch.split(p, [D * H, H, H * n, n, H, 1])
    o = torch.tensor(obs, dtype=torch.float64)
    h = torch.relu(o @ W1.view(D, H) + b1)
    dist = torch.distributions.Categorical(logits=h @ W2.view(H, n) + b2)
    V = h @ wv + bv
    a = torch.tensor(act, dtype=torch.int64)
    rho = torch.exp(dist.log_prob(a) - torch.tensor(logp_old, dtype=torch.float64))
    A = torch.tensor(adv_hat, dtype=torch.float64)
    surr = torch.min(rho * A, torch.clamp(rho, 1 - eps, 1 + eps) * A)
    R = torch.tensor(ret, dtype=torch.float64)
    L = -surr.mean() + c_v * ((V - R) ** 2).mean() - c_e * dist.entropy().mean()
    L.backward()
    return L.item(), p.grad.numpy()


@pytest.mark.parametrize("D,H,n", SHAPES)
def test_ppo_grad_matches_torch_and_differences(D, H, n):
    params, obs, act, adv, ret = batch(D, H, n, 200, seed=31 + H)
    # behaviour log-probs of a perturbed policy: ratios spread over both clip edges
    old = OA.forward(params + np.random.default_rng(2).standard_normal(params.size) * 0.3, obs, D, H, n)[3]
    logp_old = np.log(old[np.arange(200), act])
    L_t, g_t = torch_ppo_loss(params, obs, act, adv, ret, logp_old, D, H, n, 0.5, 0.01, 0.2)
    L = OA.ppo_loss(params, obs, act, adv, ret, logp_old, D, H, n, 0.5, 0.01, 0.2)[0]
    g = OA.ppo_grad(params, obs, act, adv, ret, logp_old, D, H, n, 0.5, 0.01, 0.2)
    assert abs(L - L_t) < 1e-12 * max(1, abs(L))
    np.testing.assert_allclose(g, g_t, rtol=1e-9, atol=1e-12)
    rho = OA.forward(params, obs, D, H, n)[3][np.arange(200), act] / old[np.arange(200), act]
    assert (rho < 0.8).any() and (rho > 1.2).any()  # both clip edges exercised


def test_ppo_identity_and_clip_rule():
    """new params = old params -> rho = 1, surrogate = mean(A_hat), gradient = A2C's;
    S:411: rho = 1.5, A_hat > 0, eps = 0.2 -> the clipped term 1.2 A_hat is used (zero
    surrogate gradient on that row)."""
    D, H, n = 4, 8, 2
    params, obs, act, adv, ret = batch(D, H, n, 64, seed=41)
    pi = OA.forward(params, obs, D, H, n)[3]
    logp_now = np.log(pi[np.arange(64), act])
    L = OA.ppo_loss(params, obs, act, adv, ret, logp_now, D, H, n, 0.5, 0.01, 0.2)
    assert L[1] == pytest.approx(-adv.mean(), rel=1e-12)
    np.testing.assert_allclose(OA.ppo_grad(params, obs, act, adv, ret, logp_now, D, H, n, 0.5, 0.01, 0.2),
                               OA.grad(params, obs, act, adv, ret, D, H, n, 0.5, 0.01), rtol=1e-10, atol=1e-14)
    one = np.array([1.0])
    lo = logp_now[:1] - np.log(1.5)  # rho = 1.5 on row 0
    Lr = OA.ppo_loss(params, obs[:1], act[:1], one, ret[:1], lo, D, H, n, 0.0, 0.0, 0.2)
    assert Lr[1] == pytest.approx(-1.2, rel=1e-12)
    g = OA.ppo_grad(params, obs[:1], act[:1], one, ret[:1], lo, D, H, n, 0.0, 0.0, 0.2)
    assert np.abs(g).max() == 0.0


# ---------------------------------------------------------------- Gaussian actor-critic (R35)
@pytest.mark.parametrize("D,H,d", [(3, 8, 1), (3, 32, 1), (5, 16, 2)])
def test_gauss_grad_matches_torch_and_differences(D, H, d):
    r = np.random.default_rng(D * 10 + d)
    params = r.standard_normal(OA.n_params_gauss(D, H, d)) * 0.5
    B = 150
    obs = r.standard_normal((B, D))
    act = r.standard_normal((B, d)) * 1.5
    act[::23] = np.nan  # rows with a non-finite action contribute nothing
    adv, ret = r.standard_normal(B), r.standard_normal(B)
    g = OA.grad_gauss(params, obs, act, adv, ret, D, H, d, 0.5, 0.03, batch=200)
    # torch autograd of an independent formulation (torch.distributions.Normal)
    p = torch.tensor(params, requires_grad=True)
    W1, b1, W2, b2, ls, wv, bv = torch.split(p, [D * H, H, H * d, d, d, H, 1])
    o = torch.tensor(obs)
    h = torch.relu(o @ W1.view(D, H) + b1)
    dist = torch.distributions.Normal(h @ W2.view(H, d) + b2, torch.exp(ls))
    ok = torch.tensor(np.isfinite(act).all(axis=1)).double()
    a = torch.tensor(np.nan_to_num(act))
    V = (h @ wv + bv)
    L = (-(dist.log_prob(a).sum(1) * torch.tensor(adv) * ok).sum() + 0.5 * (((V - torch.tensor(ret)) ** 2) * ok).sum()
         - 0.03 * (dist.entropy().sum(1) * ok).sum()) / 200
    L.backward()
    np.testing.assert_allclose(g, p.grad.numpy(), rtol=1e-9, atol=1e-12)
    assert OA.loss_gauss(params, obs, act, adv, ret, D, H, d, 0.5, 0.03, batch=200)[0] == pytest.approx(L.item(), rel=1e-12)
    # central differences of the oracle's own loss (fp64)
    fd = np.zeros_like(g)
    for i in range(0, params.size, max(1, params.size // 40)):
        pp, pm = params.copy(), params.copy()
        pp[i] += 1e-6
        pm[i] -= 1e-6
        fd[i] = (OA.loss_gauss(pp, obs, act, adv, ret, D, H, d, 0.5, 0.03, batch=200)[0] -
                 OA.loss_gauss(pm, obs, act, adv, ret, D, H, d, 0.5, 0.03, batch=200)[0]) / 2e-6
        assert abs(fd[i] - g[i]) <= 1e-5 * max(1e-3, abs(g[i])), i
