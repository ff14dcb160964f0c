"""Timing sweep of ws_rollout (CUDA events, warm) over replica counts and CTA sizes."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import wsinputs as W
from paper_2408_00930_b200 import Env

env = sys.argv[1] if len(sys.argv) > 1 else "cartpole"
Es = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "10000").split(",")]
blocks = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "128").split(",")]
T = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
n = {"cartpole": 2, "acrobot": 3, "dummy": 2}.get(env, 0)
out = []
for E in Es:
    for b in blocks:
        g = Env(E, 1, env, W.SEED, t_capacity=T, block_size=b)
        p = torch.from_numpy(W.uniform_probs(E, 1, n) if n else W.gaussian_params(E, 1, 1)).cuda()
        for _ in range(3):
            g.rollout(T, p)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        K = 10
        for _ in range(K):
            g.rollout(T, p)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / K
        r = {"env": env, "E": E, "block": b, "T": T, "ms": round(ms, 4), "Gsteps_s": round(E * T / ms / 1e6, 2)}
        print(json.dumps(r), flush=True)
        out.append(r)
        del g
        torch.cuda.empty_cache()
