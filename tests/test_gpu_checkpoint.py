"""Checkpoint / resume on the GPU: a run interrupted after a roll-out and resumed
in a fresh handle + trainer continues bit-identically (store, statistics, parameters) -- the
counter-based streams (R15) make the live state plus the step index a complete checkpoint."""
import numpy as np
import pytest
import torch

import wsinputs as W

pytestmark = pytest.mark.gpu
SEED = W.SEED


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2408_00930_b200 as P
    return P


@pytest.mark.parametrize("env,A,kw", [("cartpole", 1, {}), ("acrobot", 1, {}), ("pendulum", 1, {}),
                                      ("tag", 50, {"param0": 20, "param1": 5})])
def test_env_resume_is_bit_exact(P, env, A, kw, tmp_path):
    from paper_2408_00930_b200 import checkpoint as ck
    E, T = 200, 80
    n = {"cartpole": 2, "acrobot": 3, "tag": 5}.get(env)
    probs = (W.random_probs(E, A, n, seed=191) if n else W.gaussian_params(E, A, 1, 0.0, 0.0))
    probs = torch.from_numpy(probs).cuda()
    a = P.Env(E, A, env, SEED, t_capacity=T, **kw)
    a.rollout(T, probs)
    snap = ck.env_state(a)
    torch.save(snap, tmp_path / "env.pt")
    a.rollout(T, probs)
    ref = {k: v.cpu().numpy() for k, v in a.buffers().items() if v is not None}
    b = P.Env(E, A, env, SEED, t_capacity=T, **kw)
    ck.load_env_state(b, torch.load(tmp_path / "env.pt"))
    b.rollout(T, probs)
    got = {k: v.cpu().numpy() for k, v in b.buffers().items() if v is not None}
    for k in ("obs", "act", "logp", "rew", "done", "stats", "obs_live", "reset_count", "ep_step", "ep_ret"):
        assert np.array_equal(got[k], ref[k], equal_nan=True), k
    assert b.info().t == a.info().t


def test_training_resume_is_bit_exact(P, tmp_path):
    from paper_2408_00930_b200 import checkpoint as ck
    from paper_2408_00930_b200.a2c import A2C
    E, T, H = 500, 32, 64
    a = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    tr = A2C(a, H, lr=3e-3, seed=3)
    for _ in range(3):
        tr.iteration(T)
    ck.save_params(str(tmp_path / "p.wsac"), tr.params, 4, H, 2)
    e_snap, t_snap = ck.env_state(a), ck.trainer_state(tr)
    for _ in range(2):
        tr.iteration(T)
    ref = tr.params.cpu().numpy()
    b = P.Env(E, 1, "cartpole", SEED, t_capacity=T)
    tr2 = A2C(b, H, lr=3e-3, seed=99)
    ck.load_env_state(b, e_snap)
    ck.load_trainer_state(tr2, t_snap)
    p_file, _ = ck.load_params(str(tmp_path / "p.wsac"))
    assert np.array_equal(p_file.numpy(), t_snap["params"].numpy())
    for _ in range(2):
        tr2.iteration(T)
    assert np.array_equal(tr2.params.cpu().numpy(), ref)
