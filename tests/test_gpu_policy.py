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
    t = P.Env(2, 200, "tag", SEED, t_capacity=4)
    with pytest.raises(P.WSError):
        t.rollout_policy(4, w, 32)  # tag policy roll-out: at most 128 agents per replica
    p = P.Env(4, 1, "surface", SEED, t_capacity=4, param0=20)
    with pytest.raises(P.WSError):
        p.rollout_policy(4, w, 32)  # continuous actions beyond Pendulum (R34): not supported


@pytest.mark.parametrize("H,E,T", [(32, 300, 200), (64, 129, 150)])
def test_gaussian_policy_rollout_parity(P, H, E, T):
    """NEXT-N1 continuous (R34): Pendulum with the Gaussian MLP policy in the fused loop
    against the oracle's policy roll-out: obs / act / rew / done / state bit-identical,
    log-probs within 2 ulp (R18); with the critic, values within the critic tolerance."""
    from test_oracle_policy import gauss_params
    D, d = 3, 1
    w = gauss_params(D, H, d, seed=17, log_std=-0.3)
    g = P.Env(E, 1, "pendulum", SEED, t_capacity=T)
    g.rollout_policy(T, torch.from_numpy(w).cuda(), H)
    assert g.status() == 0
    o = O.Batch("pendulum", E, 1, SEED, t_capacity=T)
    assert o.rollout_policy_gauss(T, w, H, n_threads=8) == 0
    buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    for k in ("obs", "act", "rew", "done", "state", "obs_live", "reset_count"):
        ref = o.array(k)[:T] if k in ("obs", "act", "rew", "done") else o.array(k)
        got = buf[k][:T] if k in ("obs", "act", "rew", "done") else buf[k]
        assert np.array_equal(got, ref), k
    lg, lo = buf["logp"][:T].ravel(), o.array("logp")[:T].ravel()
    assert np.all(np.abs(lg.view(np.int32).astype(np.int64) - lo.view(np.int32).astype(np.int64)) <= 2)
    st_g, st_o = g.stats_f64(T).cpu().numpy(), np.array(o.array("stats"))[:T]
    assert np.array_equal(st_g[:, [0, 2]], st_o[:, [0, 2]])
    # R20: per-replica rewards rounded to multiples of 2^-32 (Pendulum rewards can be < 2^-8)
    np.testing.assert_allclose(st_g[:, [1, 3]], st_o[:, [1, 3]], rtol=1e-12, atol=E * 2.0 ** -32)
    # critic variant: same store, values = wv^T h + bv of the logged observations
    r = np.random.default_rng(18)
    head = np.concatenate([r.standard_normal(H) / np.sqrt(H), [-3.0]]).astype(np.float32)
    wc = np.concatenate([w, head])
    gc = P.Env(E, 1, "pendulum", SEED, t_capacity=T)
    vals, boot = torch.empty(T * E, device="cuda"), torch.empty(E, device="cuda")
    gc.rollout_actor_critic(T, torch.from_numpy(wc).cuda(), H, vals, boot)
    assert np.array_equal(gc.buffers()["act"].cpu().numpy(), buf["act"])
    obs = buf["obs"][:T].reshape(-1, D).astype(np.float64)
    W1 = w[:D * H].reshape(D, H).astype(np.float64)
    b1 = w[D * H:D * H + H].astype(np.float64)
    h = np.maximum(obs @ W1 + b1, 0.0)
    ref = h @ head[:H].astype(np.float64) + head[H]
    assert np.all(np.abs(vals.cpu().numpy() - ref) <= 1e-5 * (3.0 + h @ np.abs(head[:H])))


def test_torch_policy_rollout(P):
    """paper_2408_00930_b200.policy.rollout_with: (1) a torch policy returning fixed rows
    reproduces the fused ws_rollout on those rows bit for bit (single-step sample + step ==
    fused roll-out, R28); (2) an observation-dependent torch network drives the roll-out:
    every logged log-prob is the log of the policy's probability of the logged action at the
    logged (pre-step) observation."""
    from paper_2408_00930_b200.policy import rollout_with
    E, T = 300, 64
    probs = torch.from_numpy(W.random_probs(E, 1, 3, seed=141, zero_frac=0.2)).cuda()
    a = P.Env(E, 1, "acrobot", SEED, t_capacity=T)
    rollout_with(a, lambda obs: probs, T)
    b = P.Env(E, 1, "acrobot", SEED, t_capacity=T)
    b.rollout(T, probs)
    A = {k: v.cpu().numpy() for k, v in a.buffers().items() if v is not None}
    B = {k: v.cpu().numpy() for k, v in b.buffers().items() if v is not None}
    for k in ("obs", "act", "logp", "rew", "done", "state", "obs_live", "reset_count", "stats"):
        assert np.array_equal(A[k], B[k], equal_nan=True), k
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(4, 32), torch.nn.Tanh(), torch.nn.Linear(32, 2)).cuda()
    pol = lambda obs: torch.softmax(net(obs), dim=-1)  # noqa: E731
    c = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    with torch.no_grad():
        rollout_with(c, pol, T)
        C_ = c.buffers()
        p_all = pol(C_["obs"][:T])                       # [T, E, 1, 2] at the logged observations
        act = C_["act"][:T].long()
        lp_ref = torch.log(torch.gather(p_all, -1, act.unsqueeze(-1)).squeeze(-1))
    assert torch.allclose(C_["logp"][:T], lp_ref, atol=1e-5)
    assert 0.05 < (act == 0).float().mean().item() < 0.95


@pytest.mark.parametrize("env,A", [("cartpole", 1), ("tag", 20)])
def test_policy_graph_replays_equal_eager_rollouts(P, env, A):
    """policy.PolicyGraph (SURVEY 8(f) N1 "captured in a CUDA Graph"): the T-step loop of a
    torch policy captured once and replayed three times writes, after every replay, exactly
    the store, live state and statistics of three eager rollout_with calls (the device clock
    advances the ACTION draw index per step, R15); fused roll-outs are refused while the graph
    holds the clock, and closing it hands the step index (3 T) back to the host."""
    from paper_2408_00930_b200.policy import PolicyGraph, rollout_with
    E, T = 96, 40
    D, n = (4, 2) if env == "cartpole" else (4, 5)
    g = torch.Generator(device="cpu").manual_seed(7)
    Wt = (torch.randn(D, n, generator=g) * 2.0).cuda()
    b = torch.randn(n, generator=g).cuda()
    pol = lambda obs: torch.softmax((obs[..., :, None] * Wt).sum(-2) + b, dim=-1)  # noqa: E731  (no cuBLAS)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    a = P.Env(E, A, env, SEED, t_capacity=T, stream=sa)
    e = P.Env(E, A, env, SEED, t_capacity=T, stream=sb)
    keys = ("obs", "act", "logp", "rew", "done", "state", "tstate", "obs_live", "reset_count", "ep_step", "stats")
    pg = PolicyGraph(a, pol, T)
    with pytest.raises(P.WSError):
        a.rollout(T, torch.full((E, A, n), 1.0 / n, device="cuda"))
    for k in range(3):
        pg.rollout()
        with torch.cuda.stream(sb):
            rollout_with(e, pol, T)
        torch.cuda.synchronize()
        A_ = {q: v.cpu().numpy() for q, v in a.buffers().items() if v is not None}
        B_ = {q: v.cpu().numpy() for q, v in e.buffers().items() if v is not None}
        for q in keys:
            if q in A_:
                assert np.array_equal(A_[q], B_[q], equal_nan=True), (env, k, q)
    assert a.info().t == 3 * T
    pg.close()
    assert a.info().t == 3 * T and e.info().t == 3 * T
    a.rollout(T, torch.full((E, A, n), 1.0 / n, device="cuda"))  # the host owns the clock again
    assert a.status() == 0


@pytest.mark.parametrize("H,E,A,T", [(32, 20, 100, 60), (64, 7, 37, 80)])
def test_tag_policy_rollout_parity(P, H, E, A, T):
    """Multi-agent policy inference inside the CTA-per-replica tag kernel (P:65 / P:71:
    every agent thread samples from the policy; R29, R36) against the oracle's per-agent
    policy roll-out: bit-identical store (log-probs within 2 ulp, R18); with the critic,
    values / bootstrap within the critic tolerance."""
    w = W.policy_weights(4, H, 5, seed=181, scale=2.0)
    g = P.Env(E, A, "tag", SEED, t_capacity=T)
    g.rollout_policy(T, torch.from_numpy(w).cuda(), H)
    assert g.status() == 0
    o = O.Batch("tag", E, A, SEED, t_capacity=T)
    assert o.rollout_policy(T, w, H, n_threads=4) == 0
    buf = {k: v.cpu().numpy() for k, v in g.buffers().items() if v is not None}
    for k in ("obs", "act", "rew", "done", "obs_live", "reset_count"):
        ref = o.array(k)[:T] if k in ("obs", "act", "rew", "done") else o.array(k)
        got = buf[k][:T] if k in ("obs", "act", "rew", "done") else buf[k]
        assert np.array_equal(got, ref), k
    lg, lo = buf["logp"][:T].ravel(), o.array("logp")[:T].ravel()
    assert np.all(np.abs(lg.view(np.int32).astype(np.int64) - lo.view(np.int32).astype(np.int64)) <= 2)
    assert len(np.unique(buf["act"][:T])) >= 3  # the policy really varies the actions
    # critic variant: same store, values of the logged observations
    head = np.concatenate([np.random.default_rng(182).standard_normal(H) / np.sqrt(H), [0.5]]).astype(np.float32)
    gc = P.Env(E, A, "tag", SEED, t_capacity=T)
    vals, boot = torch.empty(T * E * A, device="cuda"), torch.empty(E * A, device="cuda")
    gc.rollout_actor_critic(T, torch.from_numpy(np.concatenate([w, head])).cuda(), H, vals, boot)
    assert np.array_equal(gc.buffers()["act"].cpu().numpy(), buf["act"])
    obs = buf["obs"][:T].reshape(-1, 4).astype(np.float64)
    W1 = w[:4 * H].reshape(4, H).astype(np.float64)
    b1 = w[4 * H:4 * H + H].astype(np.float64)
    h = np.maximum(obs @ W1 + b1, 0.0)
    ref = h @ head[:H].astype(np.float64) + head[H]
    assert np.all(np.abs(vals.cpu().numpy() - ref) <= 1e-5 * (1.0 + h @ np.abs(head[:H])))
