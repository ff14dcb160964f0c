"""Small launches of the kernels added late in round 1, for compute-sanitizer racecheck /
synccheck (shared-memory hazards): the tag kernel with in-kernel policy + critic, the
composer's policy / continuous templates, the A2C gradient kernel, the peer-free Adam."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import wsinputs as W  # noqa: E402
import wsinputs.user_envs as U  # noqa: E402
import paper_2408_00930_b200 as P  # noqa: E402
from paper_2408_00930_b200 import a2c  # noqa: E402

E, A, T, H = 3, 40, 12, 32
w = torch.from_numpy(np.concatenate([W.policy_weights(4, H, 5, seed=1), np.zeros(H + 1, np.float32)])).cuda()
g = P.Env(E, A, "tag", W.SEED, t_capacity=T)
v, b = torch.empty(T * E * A, device="cuda"), torch.empty(E * A, device="cuda")
g.rollout_actor_critic(T, w, H, v, b)
g.rollout_policy(T, w[:4 * H + H + H * 5 + 5].contiguous(), H)
for name in ("u_cartpole", "u_pendulum"):
    src, dims = U.ENVS[name]
    P.register_env(name, src, **dims)
u = P.Env(64, 1, "u_cartpole", W.SEED, t_capacity=T)
u.rollout_policy(T, torch.from_numpy(W.policy_weights(4, H, 2, seed=2)).cuda(), H)
c = P.Env(64, 1, "u_pendulum", W.SEED, t_capacity=T)
c.rollout(T, torch.from_numpy(W.gaussian_params(64, 1, 1, 0.0, 0.0)).cuda())
e = P.Env(256, 1, "cartpole", W.SEED, t_capacity=T)
tr = a2c.A2C(e, H, lr=1e-3)
tr.iteration(T)
p = P.Env(256, 1, "pendulum", W.SEED, t_capacity=T)
tg = a2c.A2C(p, H, lr=1e-3)
tg.iteration(T)
torch.cuda.synchronize()
print("racecheck_small: done")
