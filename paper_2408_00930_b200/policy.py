"""Roll-outs driven by an arbitrary PyTorch policy (first stage): every step
the policy maps the live observations (a zero-copy view of libws's obs_live) to action
probabilities on the handle's stream, then libws samples (ws_sample, R13) and steps
(ws_step) -- the same kernels and results as the fused ws_rollout fed the same rows (R28).
For the in-kernel MLP policy use Env.rollout_policy / rollout_actor_critic instead (one
launch for all T steps); this path trades launch overhead for any network architecture.
PolicyGraph captures the T-step loop (policy, sample, step) once in a CUDA graph and replays
it per roll-out (SURVEY 8(f) N1 "captured in a CUDA Graph"): the handle's step index lives on
the device while the graph exists (ws_enable_device_clock), so every replay draws the actions
of the steps it runs -- the same trajectory as calling rollout_with T steps at a time.
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


class PolicyGraph:
    """rollout_with(env, policy, T) captured once in a CUDA graph, replayed by `rollout()`.

    Requirements: the handle was created on a non-default stream (Env(..., stream=
    torch.cuda.Stream())) -- CUDA graphs cannot capture the legacy default stream; the policy is
    a pure function of its input that runs on the current stream without host synchronisation
    (a torch.nn.Module under no_grad, say); its parameters may change between replays in place.
    While the graph exists the step index is device-resident: fused ws_rollout* calls on the
    handle are refused until `close()` (which copies the step index back to the host).
    The capture itself runs nothing: replay k of the graph performs roll-out k."""

    def __init__(self, env: Env, policy: Callable[[torch.Tensor], torch.Tensor], T: int):
        if env.stream.cuda_stream == 0:
            raise ValueError("PolicyGraph needs a handle created on a non-default stream "
                             "(Env(..., stream=torch.cuda.Stream()))")
        info = env.info()
        if T < 1 or T > info.t_capacity:
            raise ValueError(f"T must be in [1, t_capacity = {info.t_capacity}]")
        self.env, self.T = env, T
        self.obs_live = env.buffers()["obs_live"]
        env.synchronize()
        with torch.cuda.stream(env.stream):
            policy(self.obs_live)  # lazy initialisation of the policy's kernels / workspaces
        env.stream.synchronize()
        env.enable_device_clock(True)
        try:
            env.rewind()
            self.graph = torch.cuda.CUDAGraph()
            keep = []
            with torch.cuda.graph(self.graph, stream=env.stream):
                for _ in range(T):
                    probs = policy(self.obs_live)
                    if probs.dtype != torch.float32 or not probs.is_contiguous():
                        probs = probs.float().contiguous()
                    env.sample(probs)
                    env.step()
                    keep.append(probs)
            self._keep = keep  # the graph's memory pool owns them; keep the tensors alive
        except Exception:
            env.enable_device_clock(False)
            raise
        # the host cursor now reads T: exactly the state after every replay (slots 0 .. T-1)

    def rollout(self) -> None:
        """One roll-out of T steps into store slots [0, T) (asynchronous on the handle's stream)."""
        with torch.cuda.stream(self.env.stream):
            self.graph.replay()

    def close(self) -> None:
        """Release the graph and move the step index back to the host."""
        if getattr(self, "graph", None) is not None:
            self.env.stream.synchronize()
            self.graph = None
            self._keep = None
            self.env.enable_device_clock(False)
