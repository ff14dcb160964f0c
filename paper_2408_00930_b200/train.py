"""NEXT-N2: the training loop (SPEC train S:418-421; A2C or PPO; P:86 / P:95 convergence claims, Fig 2(b)):
alternate fused roll-outs with in-kernel inference and on-device A2C updates until a budget
of iterations or a target mean episodic return, emitting the learning curve as CSV with the
SPEC columns wall_clock_s, env_steps, mean_episodic_reward, mean_episodic_length, policy_loss,
value_loss, entropy (the last update's loss terms) and the episode count.  No data
leaves the GPU between the phases; the statistics of each iteration (exact fixed-point
per-slot sums, R20) are read back once per `log_every` iterations.

    python -m paper_2408_00930_b200.train --env cartpole --envs 10000 --T 32 --iters 3000
    torchrun --nproc-per-node 8 -m paper_2408_00930_b200.train ...   (data parallel)
"""
from __future__ import annotations

import argparse
import csv
import os
import sys
import time

import torch
import torch.distributed as dist

from .a2c import A2C, PPO
from .env import Env
from .parallel import shard


def train(env_name: str = "cartpole", n_envs: int = 10000, T: int = 32, iters: int = 1000, hidden: int = 64,
          lr: float = 3e-3, gamma: float = 0.99, lam: float = 0.95, c_v: float = 0.5, c_e: float = 0.01,
          max_norm: float = 0.5, seed: int = 0x24080930, target: float | None = None, log_every: int = 10,
          out=None, algo: str = "a2c", epochs: int = 4, minibatches: int = 4, clip_eps: float = 0.2,
          n_agents: int = 1) -> list[tuple]:
    """Returns the learning curve [(seconds, env_steps, mean_return, mean_length)]."""
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    off, n = shard(n_envs, world, rank)
    env = Env(n, n_agents, env_name, seed, env_offset=off, n_envs_global=n_envs, t_capacity=T)
    kw = dict(lr=lr, gamma=gamma, lam=lam, c_v=c_v, c_e=c_e, max_norm=max_norm, seed=seed & 0xFFFF)
    if algo == "ppo":
        tr = PPO(env, hidden, epochs=epochs, minibatches=minibatches, clip_eps=clip_eps, **kw)
    else:
        tr = A2C(env, hidden, **kw)
    stats = torch.zeros((log_every, 4), dtype=torch.int64, device=env.device)
    curve = []
    writer = csv.writer(out) if out is not None and rank == 0 else None
    if writer:
        writer.writerow(["wall_clock_s", "env_steps", "mean_episodic_reward", "mean_episodic_length", "policy_loss",
                         "value_loss", "entropy", "episodes"])
    torch.cuda.synchronize(env.device)
    t0 = time.perf_counter()
    st_view = env.buffers()["stats"]
    for it in range(iters):
        tr.iteration(T)
        stats[it % log_every] = st_view[:T].sum(dim=0)  # exact int64 sums of this iteration's slots
        if (it + 1) % log_every == 0 or it == iters - 1:
            s = stats.sum(dim=0)
            if world > 1:
                dist.all_reduce(s)
            s = s.tolist()  # synchronises
            stats.zero_()
            ep = s[0]
            mean_ret = s[1] * 2.0 ** -32 / ep if ep else float("nan")
            mean_len = s[2] / ep if ep else float("nan")
            row = (time.perf_counter() - t0, (it + 1) * T * n_envs, mean_ret, mean_len, ep)
            curve.append(row[:4])
            if writer:
                pl, vl, ent = tr.loss.tolist()  # the last update's policy / value / entropy terms
                writer.writerow([f"{row[0]:.4f}", row[1], f"{row[2]:.3f}", f"{row[3]:.3f}", f"{pl:.6g}",
                                 f"{vl:.6g}", f"{ent:.6g}", row[4]])
            if target is not None and ep and mean_ret >= target:
                break
    return curve


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--env", default="cartpole")
    ap.add_argument("--envs", type=int, default=10000)
    ap.add_argument("--T", type=int, default=32)
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--hidden", type=int, default=64)
    ap.add_argument("--lr", type=float, default=3e-3)
    ap.add_argument("--gamma", type=float, default=0.99)
    ap.add_argument("--lam", type=float, default=0.95)
    ap.add_argument("--entropy", type=float, default=0.01)
    ap.add_argument("--target", type=float, default=None)
    ap.add_argument("--log-every", type=int, default=10)
    ap.add_argument("--csv", default="-")
    ap.add_argument("--seed", type=lambda x: int(x, 0), default=0x24080930)
    ap.add_argument("--algo", choices=["a2c", "ppo"], default="ppo")  # SPEC: PPO is the default trainer
    ap.add_argument("--epochs", type=int, default=4)
    ap.add_argument("--minibatches", type=int, default=4)
    ap.add_argument("--clip", type=float, default=0.2)
    ap.add_argument("--agents", type=int, default=1)
    a = ap.parse_args(argv)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) > 1:
        local = int(os.environ.get("LOCAL_RANK", 0))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = sys.stdout if a.csv == "-" else open(a.csv, "w", newline="")
    train(a.env, a.envs, a.T, a.iters, a.hidden, a.lr, a.gamma, a.lam, c_e=a.entropy, target=a.target,
          log_every=a.log_every, seed=a.seed, out=out, algo=a.algo, epochs=a.epochs, minibatches=a.minibatches,
          clip_eps=a.clip, n_agents=a.agents)
    if out is not sys.stdout:
        out.close()
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
