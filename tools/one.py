"""One warm roll-out of a config (for ncu captures): python tools/one.py env E block T [reps]."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import wsinputs as W
from paper_2408_00930_b200 import Env

env, E, b, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
n = {"cartpole": 2, "acrobot": 3, "dummy": 2}.get(env, 0)
g = Env(E, 1, env, W.SEED, t_capacity=T, block_size=b)
p = torch.from_numpy(W.uniform_probs(E, 1, n) if n else W.gaussian_params(E, 1, 1)).cuda()
for _ in range(reps):
    g.rollout(T, p)
torch.cuda.synchronize()
print("ok")
