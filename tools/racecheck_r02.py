"""Small launches of the kernels added or restructured in round 2, for compute-sanitizer
racecheck / synccheck / memcheck: the warp-specialised policy roll-out (named-barrier hand-over
between the env warp and the inference warps, with and without the critic, truncations), the
plan-driven composer kernel (per-warp statistics window), the segmented surface kernel (shuffled
energy, statistics window + CTA accumulator), the plan kernel clearing the statistics slab, and
the ws_test_surface_energy hook."""
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

T, H = 40, 32
# policy roll-out (ws kernel), 70 replicas: a full and a partial 32-replica group
e = P.Env(70, 1, "cartpole", W.SEED, t_capacity=T, max_steps=9)   # truncations every 9 steps
wts = torch.from_numpy(W.a2c_params(4, H, 2, seed=3)).cuda()
v, b, vt = (torch.empty(T * 70, device="cuda"), torch.empty(70, device="cuda"), torch.zeros(T * 70, device="cuda"))
e.rollout_actor_critic(T, wts, H, v, b, vt)
e.rollout_policy(T, wts[:4 * H + H + 2 * H + 2].contiguous(), H)
ac = P.Env(40, 1, "acrobot", W.SEED, t_capacity=T)
ac.rollout_policy(T, torch.from_numpy(W.policy_weights(6, H, 3, seed=4)).cuda(), H)
# composer: plan-driven template
src, dims = U.ENVS["u_cartpole"]
P.register_env("u_cartpole", src, **dims)
u = P.Env(45, 1, "u_cartpole", W.SEED, t_capacity=T)
u.rollout(T, torch.from_numpy(W.uniform_probs(45, 1, 2)).cuda())
# surface-D segmented kernel (13 replicas: a partial last warp)
s = P.Env(13, 1, "surface", W.SEED, t_capacity=T, param0=20, max_steps=17)
s.rollout(T, torch.from_numpy(W.gaussian_params(13, 1, 20, 0.0, float(np.log(0.025)))).cuda())
q = torch.randn(10, 20, device="cuda")
P.ws_test_surface_energy(q)
# discrete roll-out (plan kernel clears the statistics)
c = P.Env(50, 1, "cartpole", W.SEED, t_capacity=T)
c.rollout(T, torch.from_numpy(W.uniform_probs(50, 1, 2)).cuda())
tr = a2c.A2C(P.Env(64, 1, "cartpole", W.SEED, t_capacity=T), H, lr=1e-3)
tr.iteration(T)
# round 2, last session: the policy kernel's store warp (named barriers 5 / 6) is exercised above;
# the surface kernel's fast 4-step trips with goal terminations (per-step steering heads), the
# Gaussian plan (one Philox block per lane, lane = step log-densities), and a CUDA-graph-captured
# torch-policy roll-out on the device clock (sample / step kernels reading / advancing t_dev)
D = 20
g0 = P.Env(40, 1, "surface", W.SEED, t_capacity=T, param0=D, max_steps=30)
hd = np.zeros((T, 40, 1, 2 * D), np.float32)
hd[..., D:] = np.log(1e-6)
hd[:, :, 0, 0], hd[:, :, 0, 1] = -0.05 * 1.181 / 1.414, 0.05
g0.rollout(T, torch.from_numpy(hd).cuda(), row_stride=2 * D, step_stride=40 * 2 * D)
from paper_2408_00930_b200.policy import PolicyGraph  # noqa: E402
st = torch.cuda.Stream()
pg_env = P.Env(33, 1, "cartpole", W.SEED, t_capacity=T, stream=st)
Wt = torch.randn(4, 2, device="cuda")
pg = PolicyGraph(pg_env, lambda o: torch.softmax((o[..., :, None] * Wt).sum(-2), -1), T)
pg.rollout()
pg.rollout()
pg.close()
torch.cuda.synchronize()
for x in (e, ac, u, s, c, g0, pg_env):
    assert x.status() == 0, x.status()
print("racecheck_r02: done")
