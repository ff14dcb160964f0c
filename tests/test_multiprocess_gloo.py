"""World-size-2 and -4 CPU coverage of the multi-GPU path with the
gloo backend: each rank owns a contiguous replica shard (parallel.shard) and the only
exchange is the sum all-reduce of the per-slot statistics (parallel.allreduce_stats).  The
per-rank roll-outs are computed by the oracle here (no GPU); the merged statistics must
equal those of one process simulating all replicas, and every replica's trajectory must be
independent of the sharding (Philox keyed by the global index, DESIGN R15)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
E_GLOBAL, T, SEED = 37, 150, 0x24080930


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, env, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2408_00930_b200.parallel import allreduce_stats, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    off, n = shard(E_GLOBAL, world, rank)
    A = 10 if env == "tag" else 1
    b = O.Batch(env, n, A, SEED, env_offset=off, n_envs_global=E_GLOBAL, t_capacity=T)
    inf = b.info()
    probs = (np.full((n, A, inf["n_actions"]), 1.0 / inf["n_actions"], np.float32) if inf["n_actions"]
             else np.zeros((n, A, 2 * inf["act_dim"]), np.float32))
    assert b.rollout(T, probs) == 0
    stats = torch.from_numpy(np.array(b.array("stats")))
    allreduce_stats(stats)
    np.save(os.path.join(out_dir, f"stats_{rank}.npy"), stats.numpy())
    np.save(os.path.join(out_dir, f"obs_{rank}.npy"), np.array(b.array("obs")))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("env", ["cartpole", "tag"])
def test_multi_rank_stats_allreduce_matches_single_process(env, world, tmp_path):
    """world 2 (shards 18 / 19) and world 4 (9 / 9 / 9 / 10): uneven contiguous shards of
    E = 37."""
    import oracle as O
    mp.start_processes(_worker, args=(world, _free_port(), env, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    A = 10 if env == "tag" else 1
    full = O.Batch(env, E_GLOBAL, A, SEED, t_capacity=T)
    inf = full.info()
    probs = (np.full((E_GLOBAL, A, inf["n_actions"]), 1.0 / inf["n_actions"], np.float32) if inf["n_actions"]
             else np.zeros((E_GLOBAL, A, 2 * inf["act_dim"]), np.float32))
    assert full.rollout(T, probs) == 0
    ref = np.array(full.array("stats"))
    for r in range(world):
        got = np.load(tmp_path / f"stats_{r}.npy")
        assert np.array_equal(got[:, [0, 2]], ref[:, [0, 2]])      # counts / lengths exact
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-9)
    obs = np.concatenate([np.load(tmp_path / f"obs_{r}.npy") for r in range(world)], axis=1)
    assert np.array_equal(obs, np.array(full.array("obs")))
