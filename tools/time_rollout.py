"""Quick device timing of ws_rollout (CUDA events, warm): python tools/time_rollout.py env E T [reps] [block]
Prints ms per roll-out and env-steps/s (diagnostic sweeps; bench.py is the reported measurement)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import wsinputs as W  # noqa: E402
from paper_2408_00930_b200 import Env  # noqa: E402

env, E, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
block = int(sys.argv[5]) if len(sys.argv) > 5 else 0
n = {"cartpole": 2, "acrobot": 3, "dummy": 2}.get(env, 0)
p = {"surface": (20, 0)}.get(env, (0, 0))
g = Env(E, 1, env, W.SEED, t_capacity=T, block_size=block, param0=p[0])
import numpy as np  # noqa: E402
pr = W.uniform_probs(E, 1, n) if n else (W.gaussian_params(E, 1, 20, 0.0, float(np.log(0.025))) if env == "surface"
                                       else W.gaussian_params(E, 1, 1))
pt = torch.from_numpy(pr).cuda()
for _ in range(3):
    g.rollout(T, pt)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize()
ev[0].record()
for _ in range(reps):
    g.rollout(T, pt)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / reps
print(f"{env} E={E} T={T} block={block}: {ms:.4f} ms/rollout, {E * T / ms * 1e3:.4g} env-steps/s, status {g.status()}")
