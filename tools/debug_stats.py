import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O, wsinputs as W
from paper_2408_00930_b200 import Env
E, T = int(sys.argv[1]), int(sys.argv[2])
probs = W.uniform_probs(E, 1, 2)
o = O.Batch("cartpole", E, 1, W.SEED, t_capacity=T); o.rollout(T, probs, n_threads=8)
so = np.array(o.array("stats"))
for block in (32, 64, 128, 256):
    for rep in range(2):
        g = Env(E, 1, "cartpole", W.SEED, t_capacity=T, block_size=block)
        g.rollout(T, torch.from_numpy(probs).cuda())
        sg = g.stats_f64(T).cpu().numpy()
        bad = np.nonzero(np.any(sg != so, axis=1))[0]
        print(block, rep, "bad slots", len(bad), bad[:10], (sg - so)[bad[:3]] if len(bad) else "")
