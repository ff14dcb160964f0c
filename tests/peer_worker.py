"""Worker for tests/test_gpu_multirank.py::test_peer_memory_stats_allreduce (run by torchrun
with 2 ranks on one GPU, gloo for the handle exchange): each rank rolls out its contiguous
shard, the statistics are merged by libws's peer-memory kernel (CUDA IPC), and every rank
saves its merged [T,4] slab of each roll-out."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import wsinputs as W  # noqa: E402
from paper_2408_00930_b200 import Env  # noqa: E402
from paper_2408_00930_b200.parallel import attach_peer_stats, shard  # noqa: E402


def main():
    out_dir, env_name, E_g, T, n_roll = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    off, n = shard(E_g, world, rank)
    n_act = {"cartpole": 2, "acrobot": 3}[env_name]
    probs_all = W.random_probs(E_g, 1, n_act, seed=41, zero_frac=0.2)
    g = Env(n, 1, env_name, W.SEED, env_offset=off, n_envs_global=E_g, t_capacity=T)
    assert attach_peer_stats(g), "peer-memory statistics path unavailable"
    p = torch.from_numpy(probs_all[off:off + n]).cuda()
    slabs = []
    for _ in range(n_roll):
        g.rollout(T, p)
        g.synchronize()
        slabs.append(g.buffers()["stats"][:T].cpu().numpy().copy())
    np.save(os.path.join(out_dir, f"stats_rank{rank}.npy"), np.stack(slabs))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
