"""Worker of tests/test_gpu_a2c_dp.py: one rank of a data-parallel A2C run (torchrun, gloo,
ranks sharing one GPU).  Each rank owns a contiguous replica shard of the global batch; the
moments and the gradient are summed across ranks inside A2C.update.  Writes, per rank, the
all-reduced gradient of the first iteration and the parameters after the last one."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import wsinputs as W  # noqa: E402
from paper_2408_00930_b200 import Env  # noqa: E402
from paper_2408_00930_b200.a2c import A2C  # noqa: E402
from paper_2408_00930_b200.parallel import shard  # noqa: E402


def main():
    out, E_g, T, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    peer = len(sys.argv) > 5 and sys.argv[5] == "peer"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    off, n = shard(E_g, world, rank)
    env = Env(n, 1, "cartpole", W.SEED, env_offset=off, n_envs_global=E_g, t_capacity=T)
    params = torch.from_numpy(W.a2c_params(4, 64, 2, seed=71))
    tr = A2C(env, 64, params=params, lr=1e-3, peer=peer)  # peer=False: the torch.distributed path
    assert (tr._pg_grad is not None) == peer
    grads = []
    for _ in range(iters):
        tr.iteration(T)
        torch.cuda.synchronize()
        grads.append(tr.grad.cpu().numpy().copy())
    np.savez(os.path.join(out, f"rank{rank}.npz"), grad0=grads[0], params=tr.params.cpu().numpy(),
             mom=tr.mom.cpu().numpy(), peer_status=(tr._pg_grad.status() if peer else 0))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
