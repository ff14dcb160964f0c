"""Diagnostic: arbitrary torch policy roll-outs (policy.rollout_with) eager vs captured in a CUDA
graph (policy.PolicyGraph): python tools/time_policy_graph.py [E T reps].  CartPole, a 4-64-2 MLP
(torch.nn) policy; CUDA events on the handle's stream."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import wsinputs as W  # noqa: E402
from paper_2408_00930_b200 import Env  # noqa: E402
from paper_2408_00930_b200.policy import PolicyGraph, rollout_with  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
torch.manual_seed(0)
net = torch.nn.Sequential(torch.nn.Linear(4, 64), torch.nn.ReLU(), torch.nn.Linear(64, 2)).cuda()
pol = lambda obs: torch.softmax(net(obs), dim=-1)  # noqa: E731
s = torch.cuda.Stream()


def timeit(fn):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.no_grad():
        fn()
        torch.cuda.synchronize()
        ev[0].record(s)
        for _ in range(reps):
            fn()
        ev[1].record(s)
        torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


with torch.no_grad():
    a = Env(E, 1, "cartpole", W.SEED, t_capacity=T, stream=s)
    with torch.cuda.stream(s):
        ms_eager = timeit(lambda: rollout_with(a, pol, T))
    b = Env(E, 1, "cartpole", W.SEED, t_capacity=T, stream=s)
    g = PolicyGraph(b, pol, T)
    ms_graph = timeit(g.rollout)
    g.close()
print(f"cartpole E={E} T={T} 4-64-2 torch MLP: eager {ms_eager:.3f} ms ({E * T / ms_eager * 1e3:.3g} env-steps/s), "
      f"CUDA graph {ms_graph:.3f} ms ({E * T / ms_graph * 1e3:.3g} env-steps/s); in-kernel policy: bench C2P")
