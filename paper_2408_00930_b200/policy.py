"""Roll-outs driven by an arbitrary PyTorch policy (first stage): every step
the policy maps the live observations (a zero-copy view of libws's obs_live) to action
probabilities on the handle's stream, then libws samples (ws_sample, R13) and steps
(ws_step) -- the same kernels and results as the fused ws_rollout fed the same rows (R28).
For the in-kernel MLP policy use Env.rollout_policy / rollout_actor_critic instead (one
launch for all T steps); this path trades launch overhead for any network architecture.
"""
from __future__ import annotations

from typing import Callable

import torch

from .env import Env


def rollout_with(env: Env, policy: Callable[[torch.Tensor], torch.Tensor], T: int) -> None:
    """T single steps into store slots [0, T): probs = policy(obs_live [E, A, D]) -> [E, A, n]
    (or [E, A, 2d] Gaussian rows), sampled and stepped by libws.  Rewinds the store cursor."""
    env.rewind()
    obs_live = env.buffers()["obs_live"]
    with torch.cuda.stream(env.stream):
        for _ in range(T):
            probs = policy(obs_live)
            if probs.dtype != torch.float32 or not probs.is_contiguous():
                probs = probs.float().contiguous()
            env.sample(probs)
            env.step()
            env._keep_probs = probs  # alive until the stream consumed it
