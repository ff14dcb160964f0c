"""NEXT-N2 on the GPU: the A2C update kernels (ws_ac_values, ws_a2c_moments, ws_a2c_grad,
ws_adam; DESIGN R31) against the fp64 oracle (oracle/a2c.py), and one full training
iteration (roll-out with in-kernel inference -> values -> GAE over the store -> gradient ->
Adam) against the oracle's roll-out and update.

Tolerances (derived in DESIGN section 4, R31): the GPU evaluates each row in fp32 (every
product and sum rounded, u = 2^-24) and accumulates per lane in fp32; the oracle is exact
fp64.  Each gradient component is compared against its own absolute-value scale
S_i = sum over rows of |each factor| (the same chain rule with absolute values): a row's
relative error is a few tens of u and the fp32 accumulation adds ~sqrt(rows per lane) u,
so |g - g_oracle| <= 2e-5 S_i (1e-4 S_i at 10M rows) leaves a margin of > 10x over the
observed error while a dropped term, wrong sign or transposed block fails by O(S_i)."""
import numpy as np
import pytest
import torch

import oracle as O
import wsinputs as W
from oracle import a2c as OA

pytestmark = pytest.mark.gpu
SEED = W.SEED


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2408_00930_b200 as P
    from paper_2408_00930_b200 import a2c
    return a2c


def grad_scale(params, obs, act, Ah, ret, D, H, N, c_v, c_e, B):
    """Per-component absolute-value scale of the gradient sum (tolerance denominator)."""
    W1, b1, W2, b2, wv, bv = OA.unpack(params, D, H, N)
    z, h, logits, pi, V = OA.forward(params, obs, D, H, N)
    o = np.abs(np.asarray(obs, np.float64).reshape(-1, D))
    a = np.asarray(act).astype(np.int64)
    ok = ((a >= 0) & (a < N)).astype(np.float64)
    a = np.clip(a, 0, N - 1)
    onehot = np.zeros_like(pi)
    onehot[np.arange(len(a)), a] = 1.0
    logpi = np.log(np.maximum(pi, 1e-300))
    ent = -(pi * logpi).sum(axis=1)
    dlog = (np.abs(Ah) / B)[:, None] * np.abs(pi - onehot) + (c_e / B) * pi * (np.abs(logpi) + ent[:, None])
    dlog *= ok[:, None]
    dV = 2 * c_v * np.abs(V - np.asarray(ret, np.float64)) / B * ok
    dz = (dlog @ np.abs(W2).T + dV[:, None] * np.abs(wv)[None, :]) * (z > 0)
    return np.concatenate([(o.T @ dz).ravel(), dz.sum(0), (h.T @ dlog).ravel(), dlog.sum(0), h.T @ dV, [dV.sum()]])


def loss_scale(params, obs, act, Ah, ret, D, H, N, c_v, c_e):
    """Absolute-value scales of the three loss terms: V - R cancels in fp32, so the value
    term is compared against c_v mean((|V| + |R|)^2)."""
    _, _, logits, pi, V = OA.forward(params, obs, D, H, N)
    a = np.asarray(act).astype(np.int64)
    ok = (a >= 0) & (a < N)
    B = len(a)
    lp = np.log(np.maximum(pi, 1e-300))
    ent = -(pi * lp).sum(1)
    pol = (np.abs(lp[np.arange(B), np.clip(a, 0, N - 1)]) * np.abs(Ah))[ok].sum() / B
    val = c_v * ((np.abs(V) + np.abs(np.asarray(ret, np.float64))) ** 2)[ok].sum() / B
    return np.array([pol, val, c_e * np.abs(ent[ok]).sum() / B + 1e-30])


def oracle_grad_chunked(params, obs, act, Ah, ret, D, H, N, c_v, c_e, B, chunk=400_000):
    g = 0.0
    s = 0.0
    L = np.zeros(3)
    for i in range(0, len(act), chunk):
        sl = slice(i, i + chunk)
        g = g + OA.grad(params, obs[sl], act[sl], Ah[sl], ret[sl], D, H, N, c_v, c_e, batch=B)
        s = s + grad_scale(params, obs[sl], act[sl], Ah[sl], ret[sl], D, H, N, c_v, c_e, B)
        L += np.array(OA.loss(params, obs[sl], act[sl], Ah[sl], ret[sl], D, H, N, c_v, c_e, batch=B)[1:])
    return g, s, L


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("D,H,N,rows", [(4, 64, 2, 3001), (6, 32, 3, 1000), (4, 32, 5, 129), (6, 64, 3, 77)])
def test_values_match_oracle(P, D, H, N, rows):
    params = W.a2c_params(D, H, N, seed=3)
    obs, _, _, _ = W.a2c_batch(rows, D, N, seed=4)
    v = P.ac_values(cuda(params), cuda(obs).view(-1), D, H, N).cpu().numpy()
    ref = OA.values(params, obs, D, H, N)
    W1, b1, W2, b2, wv, bv = OA.unpack(params, D, H, N)
    h = OA.forward(params, obs, D, H, N)[1]
    scale = np.abs(bv) + h @ np.abs(wv) + 1.0
    assert np.all(np.abs(v - ref) <= 1e-5 * scale)


def test_moments_exact_for_fp32_inputs(P):
    x = (np.random.default_rng(5).standard_normal(1_000_003) * 3 + 1).astype(np.float32)
    ws = P.workspace(4, 64, 2, "cuda")
    m = P.moments(cuda(x), ws).cpu().numpy()
    s1, s2 = OA.moments(x)
    assert abs(m[0] - s1) <= 1e-12 * np.abs(x).sum()
    assert abs(m[1] - s2) <= 1e-12 * s2


@pytest.mark.parametrize("D,H,N,rows,inv", [(4, 64, 2, 5000, 0.0), (4, 64, 2, 1283, 0.1), (6, 32, 3, 2000, 0.05),
                                            (6, 64, 3, 700, 0.0), (4, 32, 5, 300, 0.02), (4, 64, 5, 1, 0.0)])
def test_grad_matches_oracle(P, D, H, N, rows, inv):
    params = W.a2c_params(D, H, N, seed=11)
    obs, act, adv, ret = W.a2c_batch(rows, D, N, seed=12, invalid_frac=inv)
    c_v, c_e = 0.5, 0.02
    ws = P.workspace(D, H, N, "cuda")
    tadv = cuda(adv)
    mom = P.moments(tadv, ws)
    g, L = P.a2c_grad(cuda(params), cuda(obs).view(-1), cuda(act), tadv, cuda(ret), mom, float(rows), D, H, N,
                      c_v, c_e, ws)
    g = g.cpu().numpy().astype(np.float64)
    L = L.cpu().numpy()
    Ah = OA.normalize(adv)
    ref = OA.grad(params, obs, act, Ah, ret, D, H, N, c_v, c_e)
    scale = grad_scale(params, obs, act, Ah, ret, D, H, N, c_v, c_e, rows)
    bad = np.abs(g - ref) > 2e-5 * scale + 1e-12
    assert not bad.any(), (np.flatnonzero(bad)[:10], g[bad][:5], ref[bad][:5])
    Lref = OA.loss(params, obs, act, Ah, ret, D, H, N, c_v, c_e)
    assert np.all(np.abs(L - np.array(Lref[1:])) <= 2e-5 * loss_scale(params, obs, act, Ah, ret, D, H, N, c_v, c_e))


def test_grad_sharded_batch_sums_to_global(P):
    """DP: two shards with the global moments and batch size -> gradients that sum to the
    single-shard gradient (up to fp32 accumulation)."""
    D, H, N, rows = 4, 64, 2, 4000
    params = cuda(W.a2c_params(D, H, N, seed=21))
    obs, act, adv, ret = (cuda(x) for x in W.a2c_batch(rows, D, N, seed=22))
    ws = P.workspace(D, H, N, "cuda")
    mom = P.moments(adv, ws)
    g_all, _ = P.a2c_grad(params, obs.view(-1), act, adv, ret, mom, float(rows), D, H, N, 0.5, 0.01, ws)
    g_all = g_all.clone()
    h = rows // 2
    m1, m2 = P.moments(adv[:h].contiguous(), ws).clone(), P.moments(adv[h:].contiguous(), ws).clone()
    mg = m1 + m2
    g1, _ = P.a2c_grad(params, obs[:h].reshape(-1).contiguous(), act[:h].contiguous(), adv[:h].contiguous(),
                       ret[:h].contiguous(), mg, float(rows), D, H, N, 0.5, 0.01, ws)
    g1 = g1.clone()
    g2, _ = P.a2c_grad(params, obs[h:].reshape(-1).contiguous(), act[h:].contiguous(), adv[h:].contiguous(),
                       ret[h:].contiguous(), mg, float(rows), D, H, N, 0.5, 0.01, ws)
    np.testing.assert_allclose((g1 + g2).cpu().numpy(), g_all.cpu().numpy(), rtol=1e-4, atol=1e-7)


def test_grad_full_c2_batch(P):
    """BASELINE configs[1] scale: 10K replicas x 1000 steps = 10M rows, H = 64, in the
    launch configuration the bench uses; the oracle recomputes the whole sum in fp64 chunks."""
    D, H, N, rows = 4, 64, 2, 10_000_000
    params = W.a2c_params(D, H, N, seed=31)
    obs, act, adv, ret = W.a2c_batch(rows, D, N, seed=32, invalid_frac=0.001)
    ws = P.workspace(D, H, N, "cuda")
    tadv = cuda(adv)
    mom = P.moments(tadv, ws)
    g, L = P.a2c_grad(cuda(params), cuda(obs).view(-1), cuda(act), tadv, cuda(ret), mom, float(rows), D, H, N,
                      0.5, 0.01, ws)
    g = g.cpu().numpy().astype(np.float64)
    Ah = OA.normalize(adv)
    ref, scale, Lref = oracle_grad_chunked(params, obs, act, Ah, ret, D, H, N, 0.5, 0.01, rows)
    bad = np.abs(g - ref) > 1e-4 * scale + 1e-12
    assert not bad.any(), (np.flatnonzero(bad)[:10], g[bad][:5], ref[bad][:5])
    np.testing.assert_allclose(L.cpu().numpy(), Lref, rtol=1e-4)


def test_adam_matches_oracle(P):
    """Three clip + Adam steps on identical gradients: parameters within fp32 storage rounding
    of the fp64 oracle; one step with a large gradient exercises the clip."""
    n = 709
    r = np.random.default_rng(41)
    p = r.standard_normal(n).astype(np.float32)
    tp, tm, tv = cuda(p), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    po, mo, vo = p.astype(np.float64), np.zeros(n), np.zeros(n)
    gn = torch.zeros(1, device="cuda")
    for k, sc in ((1, 5.0), (2, 0.01), (3, 0.2)):
        g = (r.standard_normal(n) * sc).astype(np.float32)
        P.adam(tp, cuda(g), tm, tv, k, 1e-3, 0.9, 0.999, 1e-8, 0.5, grad_norm=gn)
        assert gn.item() == pytest.approx(np.linalg.norm(g.astype(np.float64)), rel=1e-6)
        po, mo, vo = OA.adam(po, OA.clip(g, 0.5), mo, vo, k, 1e-3)
        np.testing.assert_allclose(tp.cpu().numpy(), po, rtol=0, atol=1e-6 * (1 + np.abs(po)).max())
    # zero gradient with zero moments: parameters unchanged
    q = cuda(p)
    P.adam(q, torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda"), 1, 1e-3)
    assert torch.equal(q, cuda(p))


@pytest.mark.parametrize("env,H,E,T", [("cartpole", 64, 300, 128), ("acrobot", 32, 130, 64)])
def test_training_iteration_matches_oracle(P, env, H, E, T):
    """One A2C iteration: the store equals the oracle's policy roll-out bit for bit (R29), the
    critic / GAE / gradient agree with the fp64 oracle on that store, and the parameters
    after the step equal the oracle's Adam applied to the GPU's gradient."""
    import paper_2408_00930_b200 as WS
    D, N = {"cartpole": (4, 2), "acrobot": (6, 3)}[env]
    params = W.a2c_params(D, H, N, seed=51, scale=1.0)
    g = WS.Env(E, 1, env, SEED, t_capacity=T)
    tr = P.A2C(g, H, params=torch.from_numpy(params), lr=1e-3, gamma=0.99, lam=0.95, c_v=0.5, c_e=0.01,
               max_norm=0.5)
    tr.iteration(T)
    g.synchronize()
    o = O.Batch(env, E, 1, SEED, t_capacity=T)
    assert o.rollout_policy(T, params[:D * H + H + H * N + N], H, n_threads=8) == 0
    buf = {k: (v.cpu().numpy() if v is not None else None) for k, v in g.buffers().items()}
    for k in ("obs", "act", "rew", "done", "obs_live"):
        assert np.array_equal(buf[k][:T] if k != "obs_live" else buf[k], o.array(k)[:T] if k != "obs_live"
                              else o.array(k)), k
    obs = o.array("obs")[:T].reshape(-1, D)
    act = o.array("act")[:T].reshape(-1)
    vals = OA.values(params, obs, D, H, N).reshape(T, E)
    boot = OA.values(params, o.array("obs_live").reshape(-1, D), D, H, N)
    adv, ret = O.gae(o.array("rew")[:T].reshape(T, E), o.array("done")[:T], vals, boot, 0.99, 0.95, f64=True)
    Ah = OA.normalize(adv)
    ref = OA.grad(params, obs, act, Ah, ret.ravel(), D, H, N, 0.5, 0.01)
    scale = grad_scale(params, obs, act, Ah, ret.ravel(), D, H, N, 0.5, 0.01, T * E)
    gg = tr.grad.cpu().numpy().astype(np.float64)
    # advantages pass through an fp32 recursion of up to ~T terms: 1e-4 of the scale
    bad = np.abs(gg - ref) > 1e-4 * scale + 1e-10
    assert not bad.any(), (np.flatnonzero(bad)[:10], gg[bad][:5], ref[bad][:5])
    p1, _, _ = OA.adam(params.astype(np.float64), OA.clip(gg, 0.5), np.zeros_like(gg), np.zeros_like(gg), 1, 1e-3)
    np.testing.assert_allclose(tr.params.cpu().numpy(), p1, rtol=0, atol=2e-6 * (1 + np.abs(p1)).max())
    assert tr.step == 1


def test_cartpole_learns(P):
    """The paper's convergence claim in miniature (Fig 2b): A2C on 2048 CartPole replicas
    raises the mean episode length well above the random policy's ~22 steps."""
    import paper_2408_00930_b200 as WS
    E, T, H = 2048, 64, 64
    g = WS.Env(E, 1, "cartpole", SEED, t_capacity=T)
    tr = P.A2C(g, H, lr=3e-3, gamma=0.99, lam=0.95, c_v=0.5, c_e=0.01, max_norm=0.5, seed=1)
    lengths = []
    for it in range(300):
        tr.iteration(T)
        st = g.stats_f64(T).cpu().numpy().sum(0)
        if st[0] > 0:
            lengths.append(st[2] / st[0])
    first, last = np.mean(lengths[:5]), np.mean(lengths[-20:])
    print(f"cartpole A2C: mean episode length {first:.1f} -> {last:.1f}")
    assert first < 40 and last > 3 * first


@pytest.mark.parametrize("env,H,E,T", [("cartpole", 64, 1000, 200), ("acrobot", 32, 257, 64)])
def test_actor_critic_rollout_writes_critic(P, env, H, E, T):
    """ws_rollout_actor_critic: the store is bit-identical to ws_rollout_policy's (the value
    head only adds outputs), values[t] = V(obs[t]) and bootstrap = V(obs_live) within the
    critic tolerance of the fp64 oracle."""
    import paper_2408_00930_b200 as WS
    D, N = {"cartpole": (4, 2), "acrobot": (6, 3)}[env]
    params = W.a2c_params(D, H, N, seed=81)
    tp = torch.from_numpy(params).cuda()
    a = WS.Env(E, 1, env, SEED, t_capacity=T)
    b = WS.Env(E, 1, env, SEED, t_capacity=T)
    vals = torch.empty(T * E, device="cuda")
    boot = torch.empty(E, device="cuda")
    a.rollout_policy(T, tp, H)
    b.rollout_actor_critic(T, tp, H, vals, boot)
    A = {k: v.cpu().numpy() for k, v in a.buffers().items() if v is not None}
    B = {k: v.cpu().numpy() for k, v in b.buffers().items() if v is not None}
    for k in ("obs", "act", "logp", "rew", "done", "stats", "state", "obs_live"):
        assert np.array_equal(A[k], B[k], equal_nan=True), k
    obs = B["obs"][:T].reshape(-1, D)
    _, _, _, _, wv, bv = OA.unpack(params, D, H, N)
    for o, v in ((obs, vals.cpu().numpy()), (B["obs_live"].reshape(-1, D), boot.cpu().numpy())):
        ref = OA.values(params, o, D, H, N)
        h = OA.forward(params, o, D, H, N)[1]
        assert np.all(np.abs(v - ref) <= 1e-5 * (np.abs(bv) + h @ np.abs(wv) + 1.0))


def test_cartpole_solved_by_training_loop(P):
    """Paper's convergence claim ("converges to the global optimum", Fig 2(b)): the
    training loop (paper_2408_00930_b200.train: fused roll-outs with in-kernel inference +
    on-device A2C, 10K CartPole replicas) reaches a mean episodic return >= 475 (the gym
    solve threshold; 500 = never falls) within 3000 iterations of 32 steps."""
    from paper_2408_00930_b200.train import train
    curve = train("cartpole", 10000, 32, 3000, lr=3e-3, target=475.0, log_every=50)
    secs, steps, ret, length = curve[-1]
    print(f"cartpole solved: mean return {ret:.1f} after {steps:.3g} env steps, {secs:.2f} s wall-clock")
    assert ret >= 475.0 and curve[0][2] < 100.0


def test_acrobot_solved_by_training_loop(P):
    """Acrobot-v1 ("the Acrobot ... converges"): 10K replicas, T = 128, lr 1e-3 reach a
    mean episodic return >= -100 (gym's solve threshold; a random policy scores ~ -499)."""
    from paper_2408_00930_b200.train import train
    curve = train("acrobot", 10000, 128, 1500, lr=1e-3, c_e=0.01, target=-100.0, log_every=50)
    secs, steps, ret, length = curve[-1]
    print(f"acrobot solved: mean return {ret:.1f} after {steps:.3g} env steps, {secs:.2f} s wall-clock")
    assert ret >= -100.0 and curve[0][2] < -400.0


def test_ppo_grad_at_the_clip_edges(P):
    """R33's clip boundary, the rows test_ppo_grad_matches_oracle moves away: six rows whose
    behaviour log-prob puts rho exactly on an edge in fp64 (three at 1 - eps, three at 1 + eps,
    advantages of both signs).  fp32 (GPU) and fp64 (oracle) may decide such a row either way, so
    the GPU gradient must equal the oracle gradient for SOME choice of the six rows' branches
    (2^6 candidates, each row's two contributions differ by far more than the tolerance), and
    the rows away from the edges must follow the oracle's choice exactly."""
    import itertools
    D, H, N, rows = 4, 64, 2, 600
    params = W.a2c_params(D, H, N, seed=111)
    obs, act, adv, ret = W.a2c_batch(rows, D, N, seed=112)
    act = np.clip(act, 0, N - 1).astype(np.int32)
    p_new = OA.forward(params, obs, D, H, N)[3][np.arange(rows), act]
    pert = params + np.random.default_rng(113).standard_normal(params.size).astype(np.float32) * 0.3
    p_old = OA.forward(pert, obs, D, H, N)[3][np.arange(rows), act]
    rho = p_new / p_old
    for edge in (0.8, 1.2):  # the bulk stays clear of the edges
        near = np.abs(rho - edge) < 1e-3
        p_old[near] = p_new[near] / (edge + 2e-3)
    logp_old = np.log(p_old).astype(np.float32)
    edge_rows = np.array([5, 50, 100, 150, 200, 250])
    for k, r in enumerate(edge_rows):
        e = 0.8 if k < 3 else 1.2
        logp_old[r] = np.float32(np.log(p_new[r]) - np.log(e))
        adv[r] = np.float32((1.0 if k % 2 == 0 else -1.0) * (1.0 + 0.5 * k))
    ws = P.workspace(D, H, N, "cuda")
    tadv = cuda(adv)
    mom = P.moments(tadv, ws)
    g, _ = P.a2c_grad(cuda(params), cuda(obs).view(-1), cuda(act), tadv, cuda(ret), mom, float(rows), D, H, N,
                      0.5, 0.01, ws, logp_old=cuda(logp_old), clip_eps=0.2)
    g = g.cpu().numpy().astype(np.float64)
    Ah = OA.normalize(adv)
    logp64 = np.log(p_new)
    rho64 = np.exp(logp64 - logp_old.astype(np.float64))
    assert np.all(np.abs(rho64[edge_rows] - np.repeat([0.8, 1.2], 3)) < 1e-6)
    active = rho64 * Ah <= np.clip(rho64, 0.8, 1.2) * Ah
    scale = grad_scale(params, obs, act, Ah * np.maximum(rho64, 1.0), ret, D, H, N, 0.5, 0.01, rows)
    hits = 0
    for choice in itertools.product([False, True], repeat=len(edge_rows)):
        act_mask = active.copy()
        act_mask[edge_rows] = choice
        ref = OA.grad(params, obs, act, np.where(act_mask, rho64 * Ah, 0.0), ret, D, H, N, 0.5, 0.01)
        if np.all(np.abs(g - ref) <= 2e-5 * scale + 1e-12):
            hits += 1
    assert hits == 1, hits  # exactly one branch assignment of the edge rows reproduces the GPU


@pytest.mark.parametrize("D,H,N,rows", [(4, 64, 2, 3000), (6, 32, 3, 1000)])
def test_ppo_grad_matches_oracle(P, D, H, N, rows):
    """ws_a2c_grad with behaviour log-probs (PPO, R33) against oracle/a2c.py ppo_grad; the
    behaviour policy is a perturbed copy so that ratios fall on both sides of the clip range
    (rows within 1e-3 of an edge are moved away: fp32 vs fp64 may pick different branches)."""
    params = W.a2c_params(D, H, N, seed=101)
    obs, act, adv, ret = W.a2c_batch(rows, D, N, seed=102)
    pert = params + np.random.default_rng(103).standard_normal(params.size).astype(np.float32) * 0.3
    p_new = OA.forward(params, obs, D, H, N)[3][np.arange(rows), act]
    p_old = OA.forward(pert, obs, D, H, N)[3][np.arange(rows), act]
    rho = p_new / p_old
    for edge in (0.8, 1.2):
        near = np.abs(rho - edge) < 1e-3
        p_old[near] = p_new[near] / (edge + 2e-3)
    logp_old = np.log(p_old).astype(np.float32)
    assert ((p_new / p_old) < 0.8).any() and ((p_new / p_old) > 1.2).any()
    ws = P.workspace(D, H, N, "cuda")
    tadv = cuda(adv)
    mom = P.moments(tadv, ws)
    g, L = P.a2c_grad(cuda(params), cuda(obs).view(-1), cuda(act), tadv, cuda(ret), mom, float(rows), D, H, N,
                      0.5, 0.01, ws, logp_old=cuda(logp_old), clip_eps=0.2)
    g = g.cpu().numpy().astype(np.float64)
    Ah = OA.normalize(adv)
    ref = OA.ppo_grad(params, obs, act, Ah, ret, logp_old, D, H, N, 0.5, 0.01, 0.2)
    rho64 = np.exp(np.log(p_new) - logp_old)
    scale = grad_scale(params, obs, act, Ah * np.maximum(rho64, 1.0), ret, D, H, N, 0.5, 0.01, rows)
    bad = np.abs(g - ref) > 2e-5 * scale + 1e-12
    assert not bad.any(), (np.flatnonzero(bad)[:10], g[bad][:5], ref[bad][:5])
    Lref = OA.ppo_loss(params, obs, act, Ah, ret, logp_old, D, H, N, 0.5, 0.01, 0.2)
    assert abs(L.cpu().numpy()[0] - Lref[1]) <= 2e-5 * (np.abs(Ah) * np.maximum(rho64, 1.2)).mean()


def test_minibatch_normalisation_uses_whole_batch(P):
    """norm_batch: a minibatch normalises with the whole batch's moments and count while its
    means divide by its own size."""
    D, H, N, rows, r0, r1 = 4, 64, 2, 4000, 1000, 2500
    params = W.a2c_params(D, H, N, seed=111)
    obs, act, adv, ret = W.a2c_batch(rows, D, N, seed=112)
    ws = P.workspace(D, H, N, "cuda")
    mom = P.moments(cuda(adv), ws)
    g, _ = P.a2c_grad(cuda(params), cuda(obs[r0:r1]).view(-1), cuda(act[r0:r1]), cuda(adv[r0:r1]),
                      cuda(ret[r0:r1]), mom, float(r1 - r0), D, H, N, 0.5, 0.01, ws, norm_batch=float(rows))
    Ah = OA.normalize(adv)[r0:r1]
    ref = OA.grad(params, obs[r0:r1], act[r0:r1], Ah, ret[r0:r1], D, H, N, 0.5, 0.01)
    scale = grad_scale(params, obs[r0:r1], act[r0:r1], Ah, ret[r0:r1], D, H, N, 0.5, 0.01, r1 - r0)
    assert np.all(np.abs(g.cpu().numpy() - ref) <= 2e-5 * scale + 1e-12)


def test_cartpole_solved_by_ppo(P):
    """PPO (SPEC ppo_update, R33): 4 epochs x 4 minibatches per 32-step roll-out of 10K
    replicas solve CartPole (mean return >= 475) within 1000 iterations."""
    from paper_2408_00930_b200.train import train
    curve = train("cartpole", 10000, 32, 1000, lr=1e-3, target=475.0, log_every=50, algo="ppo", epochs=4,
                  minibatches=4)
    print(f"cartpole PPO solved: mean return {curve[-1][2]:.1f} after {curve[-1][1]:.3g} env steps, "
          f"{curve[-1][0]:.2f} s")
    assert curve[-1][2] >= 475.0


def gauss_grad_scale(params, obs, act, Ah, ret, D, H, d, c_v, c_e, B):
    W1, b1, W2, b2, ls, wv, bv = OA.unpack_gauss(params, D, H, d)
    z, h, mu, _, V = OA.forward_gauss(params, obs, D, H, d)
    o = np.abs(np.asarray(obs, np.float64).reshape(-1, D))
    a = np.asarray(act, np.float64).reshape(-1, d)
    iv = np.exp(-2 * ls)
    dmu = (np.abs(Ah) / B)[:, None] * np.abs(a - mu) * iv
    dls = ((np.abs(Ah) / B)[:, None] * ((a - mu) ** 2 * iv + 1)).sum(0) + c_e * len(a) / B
    dV = 2 * c_v * np.abs(V - np.asarray(ret, np.float64)) / B
    dz = (dmu @ np.abs(W2).T + dV[:, None] * np.abs(wv)[None, :]) * (z > 0)
    return np.concatenate([(o.T @ dz).ravel(), dz.sum(0), (h.T @ dmu).ravel(), dmu.sum(0), dls, h.T @ dV,
                           [dV.sum()]])


@pytest.mark.parametrize("H,rows", [(64, 5000), (32, 777)])
def test_gaussian_grad_matches_oracle(P, H, rows):
    """Continuous actor-critic (R35): ws_a2c_grad with the Gaussian head against
    oracle/a2c.py grad_gauss."""
    D, d = 3, 1
    r = np.random.default_rng(121)
    params = (r.standard_normal(OA.n_params_gauss(D, H, d)) * 0.5).astype(np.float32)
    obs = r.standard_normal((rows, D)).astype(np.float32)
    act = (r.standard_normal((rows, d)) * 1.5).astype(np.float32)
    adv = r.standard_normal(rows).astype(np.float32)
    ret = (r.standard_normal(rows) * 5).astype(np.float32)
    ws = P.workspace(D, H, d, "cuda")
    tadv = cuda(adv)
    mom = P.moments(tadv, ws)
    g, L = P.a2c_grad(cuda(params), cuda(obs).view(-1), cuda(act).view(-1), tadv, cuda(ret), mom, float(rows),
                      D, H, d, 0.5, 0.02, ws)
    Ah = OA.normalize(adv)
    ref = OA.grad_gauss(params, obs, act, Ah, ret, D, H, d, 0.5, 0.02)
    scale = gauss_grad_scale(params, obs, act, Ah, ret, D, H, d, 0.5, 0.02, rows)
    got = g.cpu().numpy().astype(np.float64)
    bad = np.abs(got - ref) > 2e-5 * scale + 1e-12
    assert not bad.any(), (np.flatnonzero(bad)[:10], got[bad][:5], ref[bad][:5])
    Lref = OA.loss_gauss(params, obs, act, Ah, ret, D, H, d, 0.5, 0.02)
    np.testing.assert_allclose(L.cpu().numpy(), Lref[1:], rtol=1e-4, atol=1e-5)


def test_gaussian_training_iteration_matches_oracle(P):
    """One A2C iteration on Pendulum: Gaussian policy roll-out with the fused critic, GAE,
    gradient -- the store equals the oracle's Gaussian policy roll-out and the gradient the
    oracle's on that store."""
    import paper_2408_00930_b200 as WS
    D, d, H, E, T = 3, 1, 32, 256, 100
    r = np.random.default_rng(131)
    params = (r.standard_normal(OA.n_params_gauss(D, H, d)) * 0.4).astype(np.float32)
    params[D * H + H + H * d + d] = -0.5  # log_std
    g = WS.Env(E, 1, "pendulum", SEED, t_capacity=T)
    tr = P.A2C(g, H, params=torch.from_numpy(params), lr=1e-3)
    assert tr.gaussian
    tr.iteration(T)
    g.synchronize()
    o = O.Batch("pendulum", E, 1, SEED, t_capacity=T)
    assert o.rollout_policy_gauss(T, params[:D * H + H + H * d + 2 * d], H, n_threads=8) == 0
    buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    for k in ("obs", "act", "rew", "done"):
        assert np.array_equal(buf[k][:T], o.array(k)[:T]), k
    obs = o.array("obs")[:T].reshape(-1, D)
    act = o.array("act")[:T].reshape(-1, d)
    vals = OA.forward_gauss(params, obs, D, H, d)[4].reshape(T, E)
    boot = OA.forward_gauss(params, o.array("obs_live").reshape(-1, D), D, H, d)[4]
    adv, ret = O.gae(o.array("rew")[:T].reshape(T, E), o.array("done")[:T], vals, boot, 0.99, 0.95, f64=True)
    Ah = OA.normalize(adv)
    ref = OA.grad_gauss(params, obs, act, Ah, ret.ravel(), D, H, d, 0.5, 0.01)
    scale = gauss_grad_scale(params, obs, act, Ah, ret.ravel(), D, H, d, 0.5, 0.01, T * E)
    got = tr.grad.cpu().numpy().astype(np.float64)
    bad = np.abs(got - ref) > 1e-4 * scale + 1e-10
    assert not bad.any(), (np.flatnonzero(bad)[:10], got[bad][:5], ref[bad][:5])


def test_pendulum_learns_with_gaussian_a2c(P):
    """Continuous control ("both discrete and continuous actions"): the Gaussian
    actor-critic on 10K Pendulum replicas lifts the mean episodic return from the random
    policy's ~ -1100 to above -600 within 600 iterations of 64 steps."""
    from paper_2408_00930_b200.train import train
    curve = train("pendulum", 10000, 64, 600, lr=1e-3, c_e=0.0, log_every=50)
    first, best = curve[0][2], max(c[2] for c in curve)
    print(f"pendulum A2C: mean return {first:.1f} -> best {best:.1f}")
    assert first < -900.0 and best > -600.0


def test_truncation_bootstraps_from_post_step_value(P):
    """S:185 "truncation ... flagged so the trainer bootstraps": with max_steps = 20 the
    critic roll-out writes V(post-step state) at every truncated slot (the oracle recomputes
    the post-step state with its pinned cartpole_step from the logged pre-step observation --
    CartPole observes its state), and the A2C gradient uses it through GAE's v_trunc."""
    import paper_2408_00930_b200 as WS
    D, N, H, E, T = 4, 2, 64, 300, 60
    params = W.a2c_params(D, H, N, seed=161)
    g = WS.Env(E, 1, "cartpole", SEED, t_capacity=T, max_steps=20)
    tr = P.A2C(g, H, params=torch.from_numpy(params), lr=1e-3)
    tr.iteration(T)
    g.synchronize()
    o = O.Batch("cartpole", E, 1, SEED, t_capacity=T, max_steps=20)
    assert o.rollout_policy(T, params[:D * H + H + H * N + N], H, n_threads=8) == 0
    done = o.array("done")[:T]
    assert np.array_equal(g.buffers()["done"].cpu().numpy()[:T], done)
    obs, act = o.array("obs")[:T], o.array("act")[:T]
    trunc = np.argwhere(done == 2)
    assert len(trunc) > 100
    post = np.stack([O.cartpole_step(obs[t, e, 0], int(act[t, e, 0]))[1] for t, e in trunc])
    v_ref = OA.values(params, post, D, H, N)
    v_gpu = tr._vtrunc.view(T, E).cpu().numpy()[trunc[:, 0], trunc[:, 1]]
    h = OA.forward(params, post, D, H, N)[1]
    wv = OA.unpack(params, D, H, N)[4]
    assert np.all(np.abs(v_gpu - v_ref) <= 1e-5 * (10.0 + h @ np.abs(wv)))
    # gradient with GAE bootstrapping from those terminal values
    vt = np.zeros((T, E))
    vt[trunc[:, 0], trunc[:, 1]] = v_ref
    flat = obs.reshape(-1, D)
    vals = OA.values(params, flat, D, H, N).reshape(T, E)
    boot = OA.values(params, o.array("obs_live").reshape(-1, D), D, H, N)
    adv, ret = O.gae(o.array("rew")[:T].reshape(T, E), done, vals, boot, 0.99, 0.95, v_trunc=vt, f64=True)
    Ah = OA.normalize(adv)
    ref = OA.grad(params, flat, act.reshape(-1), Ah, ret.ravel(), D, H, N, 0.5, 0.01)
    scale = grad_scale(params, flat, act.reshape(-1), Ah, ret.ravel(), D, H, N, 0.5, 0.01, T * E)
    got = tr.grad.cpu().numpy().astype(np.float64)
    assert not (np.abs(got - ref) > 1e-4 * scale + 1e-10).any()


def test_multi_agent_a2c_iteration_matches_oracle(P):
    """Multi-agent A2C on tag (P:71 agents on threads; every agent is a row): a policy with a
    zero output layer is exactly uniform in both torch and R29, so the single-step roll-out
    equals the oracle's uniform-probability tag roll-out bit for bit; the critic, the GAE over
    [T, E, A] with the per-replica done flag (R26) and the gradient then agree with the oracle."""
    import paper_2408_00930_b200 as WS
    D, N, H, E, A, T = 4, 5, 32, 6, 100, 40
    params = W.a2c_params(D, H, N, seed=171)
    params[D * H + H:D * H + H + H * N + N] = 0.0  # W2, b2 = 0: uniform policy
    g = WS.Env(E, A, "tag", SEED, t_capacity=T)
    tr = P.A2C(g, H, params=torch.from_numpy(params), lr=1e-3)
    assert tr.A == A
    tr.iteration(T)
    g.synchronize()
    o = O.Batch("tag", E, A, SEED, t_capacity=T)
    assert o.rollout(T, np.full((E, A, N), 0.2, np.float32)) == 0
    buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    for k in ("obs", "act", "rew", "done"):
        assert np.array_equal(buf[k][:T], o.array(k)[:T]), k
    obs = o.array("obs")[:T].reshape(-1, D)
    act = o.array("act")[:T].reshape(-1)
    vals = OA.values(params, obs, D, H, N).reshape(T, E, A)
    boot = OA.values(params, o.array("obs_live").reshape(-1, D), D, H, N).reshape(E, A)
    adv, ret = O.gae(o.array("rew")[:T], o.array("done")[:T], vals, boot, 0.99, 0.95, f64=True)
    Ah = OA.normalize(adv)
    ref = OA.grad(params, obs, act, Ah, ret.ravel(), D, H, N, 0.5, 0.01)
    scale = grad_scale(params, obs, act, Ah, ret.ravel(), D, H, N, 0.5, 0.01, T * E * A)
    got = tr.grad.cpu().numpy().astype(np.float64)
    bad = np.abs(got - ref) > 1e-4 * scale + 1e-10
    assert not bad.any(), (np.flatnonzero(bad)[:10], got[bad][:5], ref[bad][:5])
