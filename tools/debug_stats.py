import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O, wsinputs as W
from paper_2408_00930_b200 import Env
E, T = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 500
probs = W.uniform_probs(E, 1, 2)
g = Env(E, 1, "cartpole", W.SEED, t_capacity=T)
g.rollout(T, torch.from_numpy(probs).cuda())
o = O.Batch("cartpole", E, 1, W.SEED, t_capacity=T)
o.rollout(T, probs)
sg = g.buffers()["stats"].cpu().numpy(); so = np.array(o.array("stats"))
bad = np.nonzero((sg[:, 0] != so[:, 0]) | (sg[:, 2] != so[:, 2]))[0]
print("mismatching slots:", len(bad), bad[:20])
for t in bad[:8]:
    print(t, sg[t], so[t])
d = g.buffers()["done"].cpu().numpy()
print("done per slot gpu-count vs stats:", [(t, int((d[t] != 0).sum())) for t in bad[:8]])
