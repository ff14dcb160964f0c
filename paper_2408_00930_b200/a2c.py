"""NEXT-N2: on-device A2C training over the GPU-resident roll-out store (include/ws.h
"NEXT-N2: A2C update", DESIGN reading R31; SPEC a2c_update S:402-406, train S:419;
P:41 "supports actor-critic algorithms", "roll-outs, action inference, reset and
training" in one GPU-resident store, P:106 / P:122 "zero data transfer").

Argument marshalling only: every arithmetic step runs in libws's kernels --
ws_rollout_actor_critic (roll-out with in-kernel policy inference that also writes the
critic's values from the same hidden layer), ws_ac_values (stand-alone critic),
ws_gae_store (advantages over the store, in place), ws_a2c_moments / ws_a2c_grad
(normalised-advantage actor-critic gradient) and ws_adam (clip + Adam).  Data parallel:
each rank trains on its replica shard; the two fp64 moments and the gradient are summed
across ranks with torch.distributed (NCCL on GPUs), so every rank applies the same update.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _abi
from ._abi import WSError, check, lib
from .env import Env


def n_params(obs_dim: int, hidden: int, n_actions: int, gaussian: bool = False) -> int:
    """Packed parameter count (R31; gaussian: the R35 layout with log_std after b2)."""
    return int(lib().ws_a2c_n_params_ex(obs_dim, hidden, n_actions, 1 if gaussian else 0))


def workspace(obs_dim: int, hidden: int, n_actions: int, device) -> torch.Tensor:
    nbytes = int(lib().ws_a2c_workspace_bytes(obs_dim, hidden, n_actions))
    if nbytes == 0:
        raise WSError(_abi.INVALID_ARGUMENT, f"unsupported network shape D={obs_dim} H={hidden} n={n_actions}")
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


def _s(stream: Optional[torch.cuda.Stream], t: torch.Tensor):
    st = stream if stream is not None else torch.cuda.current_stream(t.device)
    return C.c_void_p(st.cuda_stream)


def _f32(name, t, n=None):
    if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous() or (n is not None and t.numel() != n):
        raise WSError(_abi.INVALID_ARGUMENT, f"{name}: contiguous float32 device tensor" +
                      (f" with {n} elements" if n is not None else ""))


def ac_values(params: torch.Tensor, obs: torch.Tensor, obs_dim: int, hidden: int, n_actions: int,
              out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """V(o) of every row of obs (ws_ac_values) -> float32 [rows]."""
    rows = obs.numel() // obs_dim
    _f32("params", params, n_params(obs_dim, hidden, n_actions))
    _f32("obs", obs, rows * obs_dim)
    out = torch.empty(rows, dtype=torch.float32, device=obs.device) if out is None else out
    check(lib().ws_ac_values(params.data_ptr(), obs_dim, hidden, n_actions, obs.data_ptr(), rows, out.data_ptr(),
                             _s(stream, obs)))
    return out


def moments(x: torch.Tensor, ws: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """(sum x, sum x^2) in fp64 (ws_a2c_moments) -> float64 [2] device tensor."""
    _f32("x", x)
    out = torch.empty(2, dtype=torch.float64, device=x.device) if out is None else out
    check(lib().ws_a2c_moments(x.data_ptr(), x.numel(), out.data_ptr(), ws.data_ptr(), _s(stream, x)))
    return out


def a2c_grad(params, obs, act, adv, ret, mom, batch: float, obs_dim: int, hidden: int, n_actions: int,
             c_v: float, c_e: float, ws: torch.Tensor, grad: Optional[torch.Tensor] = None,
             loss: Optional[torch.Tensor] = None, stream=None, logp_old: Optional[torch.Tensor] = None,
             clip_eps: float = 0.2, norm_batch: float = 0.0):
    """This shard's gradient of the S:405 loss (ws_a2c_grad) -> (grad f32 [P], loss f64 [3]).
    logp_old given: the PPO clipped surrogate (R33) instead of the A2C policy term.  act float32
    [rows, n_actions]: continuous actions, Gaussian head (R35)."""
    rows = adv.numel()
    gaussian = act.dtype == torch.float32
    P = n_params(obs_dim, hidden, n_actions, gaussian)
    _f32("params", params, P)
    _f32("obs", obs, rows * obs_dim)
    _f32("adv", adv, rows)
    _f32("ret", ret, rows)
    if gaussian:
        _f32("act", act, rows * n_actions)
    elif act.dtype != torch.int32 or not act.is_contiguous() or act.numel() != rows:
        raise WSError(_abi.INVALID_ARGUMENT, "act: contiguous int32 with one entry per row")
    grad = torch.empty(P, dtype=torch.float32, device=adv.device) if grad is None else grad
    loss = torch.empty(3, dtype=torch.float64, device=adv.device) if loss is None else loss
    if logp_old is not None:
        _f32("logp_old", logp_old, rows)
    a = _abi.ws_a2c_args(obs_dim, hidden, n_actions, rows, params.data_ptr(), obs.data_ptr(),
                         None if gaussian else act.data_ptr(),
                         adv.data_ptr(), ret.data_ptr(), mom.data_ptr(), float(batch), c_v, c_e, ws.data_ptr(),
                         grad.data_ptr(), loss.data_ptr(),
                         None if logp_old is None else logp_old.data_ptr(), clip_eps, float(norm_batch),
                         1 if gaussian else 0, act.data_ptr() if gaussian else None)
    check(lib().ws_a2c_grad(C.byref(a), _s(stream, adv)))
    return grad, loss


def adam(params, grad, m, v, step: int, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
         max_norm: float = 0.0, grad_norm: Optional[torch.Tensor] = None, stream=None):
    """Clip + one Adam step in place (ws_adam)."""
    n = params.numel()
    for name, t in (("params", params), ("grad", grad), ("m", m), ("v", v)):
        _f32(name, t, n)
    check(lib().ws_adam(params.data_ptr(), grad.data_ptr(), m.data_ptr(), v.data_ptr(), n, step, lr, beta1, beta2,
                        eps, max_norm, None if grad_norm is None else grad_norm.data_ptr(), _s(stream, params)))


def init_params(obs_dim: int, hidden: int, n_actions: int, seed: int = 0, device=None,
                gaussian: bool = False) -> torch.Tensor:
    """Initial weights: W1 ~ N(0, 1/D), W2 ~ N(0, 0.01^2/H) (near-uniform policy / near-zero
    mean), log_std = 0 (Gaussian head), wv ~ N(0, 1/H), zero biases; seeded on the host,
    copied once to the device."""
    g = torch.Generator().manual_seed(seed)
    D, H, N = obs_dim, hidden, n_actions
    parts = [torch.randn(D * H, generator=g) / D ** 0.5, torch.zeros(H),
             torch.randn(H * N, generator=g) * (0.01 / H ** 0.5), torch.zeros(N)]
    if gaussian:
        parts.append(torch.zeros(N))
    parts += [torch.randn(H, generator=g) / H ** 0.5, torch.zeros(1)]
    return torch.cat(parts).float().to(device)


class A2C:
    """Synchronous advantage actor-critic on one Env (one rank's replica shard).

    iteration(T): T fused roll-out steps with in-kernel policy inference, then one update
    consuming the store in place (no copy of obs / act / rew / done anywhere)."""

    def __init__(self, env: Env, hidden: int = 64, *, lr: float = 1e-3, gamma: float = 0.99, lam: float = 0.95,
                 c_v: float = 0.5, c_e: float = 0.01, max_norm: float = 0.5, beta1: float = 0.9,
                 beta2: float = 0.999, eps: float = 1e-8, seed: int = 0, params: Optional[torch.Tensor] = None,
                 group: Optional[dist.ProcessGroup] = None, bootstrap_truncation: bool = True,
                 peer="auto"):
        info = env.info()
        self.gaussian = int(info.n_actions) == 0  # continuous actions: Gaussian head (R34 / R35)
        self.A = int(info.n_agents)  # multi-agent (tag): every agent is a row; rolled out by a torch policy
        if self.A != 1 and int(info.n_actions) < 1:
            raise WSError(_abi.INVALID_ARGUMENT, "A2C: multi-agent envs need discrete actions")
        self.env, self.H = env, hidden
        self.D, self.E = int(info.obs_dim), int(info.n_envs) * self.A  # E counts agent columns (E * A)
        self.N = int(info.act_dim) if self.gaussian else int(info.n_actions)
        self.P = n_params(self.D, hidden, self.N, self.gaussian)
        if self.P == 0 or int(lib().ws_a2c_workspace_bytes(self.D, hidden, self.N)) == 0:
            raise WSError(_abi.INVALID_ARGUMENT, f"A2C: unsupported network shape D={self.D} H={hidden} n={self.N}")
        dev = env.device
        self.params = (init_params(self.D, hidden, self.N, seed, dev, self.gaussian) if params is None
                       else params.detach().to(dev, torch.float32).contiguous().clone())
        if self.params.numel() != self.P:
            raise WSError(_abi.INVALID_ARGUMENT, f"params: {self.P} floats")
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.ws = workspace(self.D, hidden, self.N, dev)
        self.grad = torch.empty_like(self.params)
        self.loss = torch.zeros(3, dtype=torch.float64, device=dev)
        self.mom = torch.zeros(2, dtype=torch.float64, device=dev)
        self.grad_norm = torch.zeros(1, dtype=torch.float32, device=dev)
        self.bootstrap = torch.empty(self.E, dtype=torch.float32, device=dev)
        self.hp = dict(lr=lr, gamma=gamma, lam=lam, c_v=c_v, c_e=c_e, max_norm=max_norm, beta1=beta1, beta2=beta2,
                       eps=eps)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.step = 0
        self._values = None
        # global agent columns (sum of every rank's E * A): shards may differ by one replica
        # (parallel.shard), so the global batch is counted, not assumed to be E * world
        self.E_global = self.E
        if self.world > 1:
            n = torch.tensor([self.E], dtype=torch.int64, device=dev if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(n, op=dist.ReduceOp.SUM, group=group)
            self.E_global = int(n.item())
        # peer=True (world > 1): moments and gradient reduced over CUDA-IPC peer memory, the
        # gradient all-reduce fused with clip + Adam in one kernel (ws_pgroup_*), no NCCL
        # ("auto": use it when CUDA IPC works on every rank, else torch.distributed / NCCL)
        self._pg_mom = self._pg_grad = None
        if peer and self.world > 1:
            from .parallel import PeerGroup
            try:
                self._pg_mom = PeerGroup(2, group)
                self._pg_grad = PeerGroup(self.P, group)
                self._mom_sum = torch.zeros(2, dtype=torch.float64, device=dev)
            except RuntimeError:
                if peer != "auto":
                    raise
                for g in (self._pg_mom, self._pg_grad):
                    if g is not None:
                        g.close()
                self._pg_mom = self._pg_grad = None
        # truncated episodes bootstrap from V(post-step state) written by the roll-out kernel
        # (GAE's v_trunc, R30); registered envs treat truncation as termination (R31)
        self.bootstrap_truncation = bootstrap_truncation and env.env in ("cartpole", "acrobot", "dummy",
                                                                         "pendulum")
        self._vtrunc = None

    def _allreduce(self, t: torch.Tensor):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def _value_buf(self, rows: int) -> torch.Tensor:
        if self._values is None or self._values.numel() != rows:
            self._values = torch.empty(rows, dtype=torch.float32, device=self.env.device)
            self._vtrunc = torch.zeros(rows, dtype=torch.float32, device=self.env.device)
        return self._values

    def _advantages(self, T: int, values_ready: bool):
        """Critic values (unless the roll-out wrote them), GAE over the store in place, and the
        global-batch moments of the advantages.  Returns (obs, act, adv, ret, rows)."""
        env, D, H, N, hp = self.env, self.D, self.H, self.N, self.hp
        s = env.stream
        buf = env.buffers()
        rows = T * self.E
        obs = buf["obs"][:T].reshape(rows * D)
        act = buf["act"][:T].reshape(rows * N if self.gaussian else rows)
        self._value_buf(rows)
        if not values_ready:
            if self.gaussian:
                raise WSError(_abi.INVALID_ARGUMENT, "Gaussian A2C: the critic comes from the roll-out kernel")
            ac_values(self.params, obs, D, H, N, out=self._values, stream=s)
            ac_values(self.params, buf["obs_live"].reshape(-1), D, H, N, out=self.bootstrap, stream=s)
        vtr = self._vtrunc.view(T, self.E, 1) if (values_ready and self.bootstrap_truncation) else None
        if vtr is not None:
            vtr = vtr.view(T, self.E // self.A, self.A)
        adv, ret = env.gae_store(T, self._values.view(T, self.E // self.A, self.A),
                                 self.bootstrap.view(self.E // self.A, self.A), hp["gamma"], hp["lam"], v_trunc=vtr)
        moments(adv.view(-1), self.ws, out=self.mom, stream=s)
        if self._pg_mom is not None:
            self._pg_mom.allreduce(self.mom, self._mom_sum, stream=s)
            self.mom.copy_(self._mom_sum)
        else:
            self._allreduce(self.mom)
        self._adv = adv  # alive until the stream consumed it
        return obs, act, adv.view(-1), ret.view(-1), rows

    def _step(self, obs, act, adv, ret, slots, norm_slots, logp_old=None, clip_eps=0.2):
        """One gradient (this shard's rows of `slots` store slots) -> all-reduce -> clip + Adam.
        The loss averages over the GLOBAL batch (slots x every rank's columns) and the advantages
        are normalised with the global moments over norm_slots slots."""
        hp, s = self.hp, self.env.stream
        a2c_grad(self.params, obs, act, adv, ret, self.mom, float(slots * self.E_global), self.D, self.H, self.N,
                 hp["c_v"], hp["c_e"], self.ws, grad=self.grad, loss=self.loss, stream=s, logp_old=logp_old,
                 clip_eps=clip_eps, norm_batch=float(norm_slots * self.E_global))
        self.step += 1
        if self._pg_grad is not None:  # fused peer-memory all-reduce + clip + Adam (one kernel)
            self._pg_grad.allreduce_adam(self.grad, self.params, self.m, self.v, self.step, hp["lr"], hp["beta1"],
                                         hp["beta2"], hp["eps"], hp["max_norm"], grad_out=self.grad,
                                         grad_norm=self.grad_norm, stream=s)
        else:
            self._allreduce(self.grad)
            adam(self.params, self.grad, self.m, self.v, self.step, hp["lr"], hp["beta1"], hp["beta2"], hp["eps"],
                 hp["max_norm"], grad_norm=self.grad_norm, stream=s)
        if self.gaussian:  # SPEC policy invariant: log_std in [-5, 2] (ws_clamp on the log_std slice)
            o = self.D * self.H + self.H + self.H * self.N + self.N
            ls = self.params[o:o + self.N]
            check(lib().ws_clamp(ls.data_ptr(), self.N, -5.0, 2.0, C.c_void_p(s.cuda_stream)))

    def update(self, T: int, values_ready: bool = False):
        """One A2C update on store slots [0, T) (already rolled out with self.params).
        values_ready: the roll-out already wrote the critic (ws_rollout_actor_critic)."""
        with torch.cuda.stream(self.env.stream):
            obs, act, adv, ret, rows = self._advantages(T, values_ready)
            self._step(obs, act, adv, ret, T, T)

    def torch_policy(self):
        """The R29 policy of self.params as a torch function (for the single-step roll-out of
        multi-agent envs, which have no fused policy kernel): probs = softmax(relu(o W1 + b1) W2 + b2)."""
        D, H, N = self.D, self.H, self.N

        def pol(obs):
            p = self.params
            W1 = p[:D * H].view(D, H)
            b1 = p[D * H:D * H + H]
            W2 = p[D * H + H:D * H + H + H * N].view(H, N)
            b2 = p[D * H + H + H * N:D * H + H + H * N + N]
            return torch.softmax(torch.relu(obs @ W1 + b1) @ W2 + b2, dim=-1)
        return pol

    def iteration(self, T: int):
        """Roll out T steps with the current policy (the fused kernels also write the critic's
        values from the hidden layer they already compute -- single-agent lanes, tag's agent
        threads; other multi-agent cases: the torch policy through ws_sample / ws_step), then
        update (train)."""
        vals = self._value_buf(T * self.E)
        if self.A == 1 or (self.env.env == "tag" and self.A <= 128 and not self.gaussian):
            # fused roll-out with in-kernel policy + critic (tag: agent threads of the CTA kernel)
            self.env.rollout_actor_critic(T, self.params, self.H, vals, self.bootstrap,
                                          self._vtrunc if self.bootstrap_truncation else None)
            self.update(T, values_ready=True)
        else:
            from .policy import rollout_with
            with torch.no_grad():
                rollout_with(self.env, self.torch_policy(), T)
            self.update(T, values_ready=False)


class PPO(A2C):
    """SPEC ppo_update (DESIGN R33): after each roll-out, `epochs` passes of
    `minibatches` clipped-surrogate steps.  Minibatch m is the contiguous slot range
    [m T / M, (m + 1) T / M) of the time-major store (every replica's rows of those slots; no
    copy, pointer offsets into the store), in a fixed order; the behaviour log-probabilities
    are the store's logp slab written by the roll-out; advantages are normalised once with the
    whole (global) batch's moments; one all-reduce + clip + Adam step per minibatch."""

    def __init__(self, env: Env, hidden: int = 64, *, epochs: int = 4, minibatches: int = 4, clip_eps: float = 0.2,
                 **kw):
        super().__init__(env, hidden, **kw)
        if epochs < 1 or minibatches < 1:
            raise WSError(_abi.INVALID_ARGUMENT, "epochs, minibatches >= 1")
        self.epochs, self.minibatches, self.clip_eps = epochs, minibatches, clip_eps
        self.ppo_seed = int(kw.get("seed", 0)) & 0xFFFFFFFF

    def update(self, T: int, values_ready: bool = False):
        if T < self.minibatches:
            raise WSError(_abi.INVALID_ARGUMENT, "T must be >= minibatches")
        with torch.cuda.stream(self.env.stream):
            obs, act, adv, ret, rows = self._advantages(T, values_ready)
            logp = self.env.buffers()["logp"][:T].reshape(rows)
            E, D, M = self.E, self.D, self.minibatches
            for ep in range(self.epochs):
                # minibatch order shuffled per epoch from a dedicated stream ("minibatch
                # shuffling from a dedicated RngStream"): Philox-free host permutation keyed by
                # (update count, epoch), identical on every rank
                order = np.random.Generator(np.random.PCG64([self.ppo_seed, self.step, ep])).permutation(M)
                for m in order.tolist():
                    t0, t1 = T * m // M, T * (m + 1) // M
                    r0, r1 = t0 * E, t1 * E
                    na = self.N if self.gaussian else 1
                    self._step(obs[r0 * D:r1 * D], act[r0 * na:r1 * na], adv[r0:r1], ret[r0:r1], t1 - t0, T,
                               logp_old=logp[r0:r1], clip_eps=self.clip_eps)
