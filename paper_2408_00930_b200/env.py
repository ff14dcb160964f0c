"""Thin Python binding of libws (include/ws.h): same call names, argument marshalling only.

PyTorch provides device memory (libws's allocator hooks are routed to torch's caching
allocator, so every byte is a torch tensor), the CUDA stream, and -- in parallel.py -- the
process group; every step of the roll-out runs in libws's sm_100a kernels.

    env = Env(10_000, 1, "cartpole", seed=0x24080930)
    probs = torch.full((10_000, 1, 2), 0.5, device="cuda")
    env.rollout(1000, probs)            # ws_rollout: one fused kernel + stats finalize
    buf = env.buffers()                 # zero-copy torch views of the store (ws_get_buffers)
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _abi
from ._abi import WSError, check, lib

_TORCH_DTYPE = {_abi.F32: torch.float32, _abi.I32: torch.int32, _abi.U8: torch.uint8,
                _abi.F64: torch.float64, _abi.U32: torch.uint32, _abi.I64: torch.int64}


class _TorchAllocator:
    """libws allocation hooks backed by torch's caching allocator; counts calls so the
    zero-steady-state-allocation invariant can be asserted."""

    def __init__(self, device: torch.device):
        self.device = device
        self.live: dict[int, torch.Tensor] = {}
        self.n_alloc = 0
        self.n_free = 0
        self.bytes = 0

        def _alloc(nbytes, stream, user):
            t = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
            p = t.data_ptr()
            self.live[p] = t
            self.n_alloc += 1
            self.bytes += int(nbytes)
            return p

        def _free(ptr, nbytes, stream, user):
            self.live.pop(int(ptr), None)
            self.n_free += 1

        self.c_alloc = _abi.ALLOC_FN(_alloc)
        self.c_free = _abi.FREE_FN(_free)


def decode_stats(st: torch.Tensor) -> torch.Tensor:
    """Fixed-point int64 stats [T, 4] (include/ws.h, DESIGN R20) -> float64 [T, 4]."""
    out = st.to(torch.float64)
    out[:, 1] *= _abi.FX_SCALE
    out[:, 3] *= _abi.FX_SCALE
    return out


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


class Env:
    """A handle of libws (ws_env*): E replicas of `env` on one GPU."""

    def __init__(self, n_envs: int, n_agents: int = 1, env: str = "cartpole", seed: int = 0, *,
                 env_offset: int = 0, n_envs_global: int = 0, device=None, stream: Optional[torch.cuda.Stream] = None,
                 t_capacity: int = 0, max_steps: int = 0, write_logp: bool = True, param0: int = 0,
                 param1: int = 0, block_size: int = 0, torch_allocator: bool = True,
                 env_prm: Optional[torch.Tensor] = None, env_shared: Optional[torch.Tensor] = None):
        L = lib()
        if not torch.cuda.is_available():
            raise WSError(_abi.CUDA_ERROR, "no CUDA device: libws runs on the GPU only (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        cfg = _abi.ws_config()
        L.ws_config_init(C.byref(cfg))
        cfg.n_envs = n_envs
        cfg.env_offset = env_offset
        cfg.n_envs_global = n_envs_global
        cfg.n_agents = n_agents
        self._env_name = env.encode()
        cfg.env = self._env_name
        cfg.seed = seed & 0xFFFFFFFFFFFFFFFF
        cfg.device = self.device.index
        cfg.stream = self.stream.cuda_stream
        cfg.t_capacity = t_capacity
        cfg.max_steps = max_steps
        cfg.write_logp = 1 if write_logp else 0
        cfg.param0 = param0
        cfg.param1 = param1
        cfg.block_size = block_size
        for name, t in (("env_prm", env_prm), ("env_shared", env_shared)):  # NEXT-N4 registered envs
            if t is not None:
                if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
                    raise WSError(_abi.INVALID_ARGUMENT, f"{name}: contiguous float32 device tensor")
                setattr(cfg, name, t.data_ptr())
        self._env_data = (env_prm, env_shared)
        self.allocator = _TorchAllocator(self.device) if torch_allocator else None
        if self.allocator is not None:
            cfg.alloc = self.allocator.c_alloc
            cfg.free = self.allocator.c_free
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            st = L.ws_create_ex(C.byref(cfg), C.byref(h))
        check(st)
        self._h = h
        self.env = env
        self.n_envs, self.n_agents = n_envs, n_agents
        self._views = None

    # ------------------------------------------------------------------ lifetime
    def close(self):
        h = getattr(self, "_h", None)
        if h:
            lib().ws_destroy(h)
            self._h = None
            self._views = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # ------------------------------------------------------------------ calls
    def _row_stride(self, probs: torch.Tensor, row_stride: Optional[int]) -> int:
        if row_stride is not None:
            return row_stride
        return 0 if probs.dim() == 1 else probs.shape[-1]

    def _check_probs(self, probs: torch.Tensor):
        if probs.device != self.device or probs.dtype != torch.float32 or not probs.is_contiguous():
            raise WSError(_abi.INVALID_ARGUMENT, "probs must be a contiguous float32 tensor on the handle's device")

    def reset(self):
        check(lib().ws_reset(self._h), self._h)

    def rewind(self):
        check(lib().ws_rewind(self._h), self._h)

    def sample(self, probs: torch.Tensor, row_stride: Optional[int] = None):
        self._check_probs(probs)
        check(lib().ws_sample(self._h, _ptr(probs), self._row_stride(probs, row_stride)), self._h)

    def step(self, actions: Optional[torch.Tensor] = None):
        if actions is not None:
            info = self.info()
            want = torch.int32 if info.n_actions else torch.float32
            if actions.device != self.device or actions.dtype != want or not actions.is_contiguous():
                raise WSError(_abi.INVALID_ARGUMENT, f"actions must be contiguous {want} on the handle's device")
        check(lib().ws_step(self._h, _ptr(actions)), self._h)

    def rollout(self, T: int, probs: torch.Tensor, row_stride: Optional[int] = None, step_stride: int = 0):
        self._check_probs(probs)
        check(lib().ws_rollout(self._h, T, _ptr(probs), self._row_stride(probs, row_stride), step_stride), self._h)

    def rollout_host(self, T: int, host_probs: torch.Tensor, row_stride: Optional[int] = None,
                     step_stride: int = 0) -> _abi.ws_stats:
        """ws_rollout_host: host (ideally pinned) probabilities in, statistics out."""
        if host_probs.device.type != "cpu" or host_probs.dtype != torch.float32 or not host_probs.is_contiguous():
            raise WSError(_abi.INVALID_ARGUMENT, "host_probs must be a contiguous float32 CPU tensor")
        out = _abi.ws_stats()
        check(lib().ws_rollout_host(self._h, T, _ptr(host_probs), host_probs.numel(),
                                    self._row_stride(host_probs, row_stride), step_stride, C.byref(out)), self._h)
        return out

    def rollout_host_submit(self, T: int, host_probs: torch.Tensor, slot: int, row_stride: Optional[int] = None,
                            step_stride: int = 0) -> None:
        """ws_rollout_host_submit: enqueue a host-buffered roll-out into result slot 0 / 1 (pinned
        host_probs, left unchanged until the matching rollout_host_wait)."""
        if host_probs.device.type != "cpu" or host_probs.dtype != torch.float32 or not host_probs.is_contiguous():
            raise WSError(_abi.INVALID_ARGUMENT, "host_probs must be a contiguous float32 CPU tensor")
        check(lib().ws_rollout_host_submit(self._h, T, _ptr(host_probs), host_probs.numel(),
                                           self._row_stride(host_probs, row_stride), step_stride, slot), self._h)

    def rollout_host_wait(self, slot: int) -> _abi.ws_stats:
        """ws_rollout_host_wait: the statistics of the submission in `slot`."""
        out = _abi.ws_stats()
        check(lib().ws_rollout_host_wait(self._h, slot, C.byref(out)), self._h)
        return out

    def rollout_staged(self, T: int, host_probs: torch.Tensor, dst: dict, row_stride: Optional[int] = None,
                       step_stride: int = 0) -> dict:
        """NEXT-N3 copy-based baseline (ws.h ws_rollout_staged): the same T steps as rollout(),
        with the step's probabilities copied host -> device and the slot's obs / act / logp /
        rew / done copied device -> host into `dst` (pinned CPU tensors shaped like the store
        slabs' first T slots) every step.  Returns the transfer report."""
        if host_probs.is_cuda or host_probs.dtype != torch.float32 or not host_probs.is_contiguous():
            raise WSError(_abi.INVALID_ARGUMENT, "host_probs: contiguous float32 host tensor")
        if step_stride:
            per_step = host_probs.numel() - (T - 1) * step_stride
        else:
            per_step = host_probs.numel()
        hs = _abi.ws_host_store(*[(dst[k].data_ptr() if dst.get(k) is not None else None)
                                  for k in ("obs", "act", "logp", "rew", "done")])
        rep = _abi.ws_staged_report()
        check(lib().ws_rollout_staged(self._h, T, host_probs.data_ptr(), per_step,
                                      self._row_stride(host_probs, row_stride), step_stride, C.byref(hs),
                                      C.byref(rep)), self._h)
        return {"total_ms": rep.total_ms, "transfer_ms": rep.transfer_ms, "h2d_bytes": rep.h2d_bytes,
                "d2h_bytes": rep.d2h_bytes}

    def host_store(self, T: int) -> dict:
        """Pinned host tensors shaped like the first T slots of the store slabs (for rollout_staged)."""
        return {k: torch.empty((T,) + tuple(v.shape[1:]), dtype=v.dtype).pin_memory()
                for k, v in self.buffers().items() if k in ("obs", "act", "logp", "rew", "done") and v is not None}

    def set_env_data(self, prm: Optional[torch.Tensor] = None, shared: Optional[torch.Tensor] = None):
        """NEXT-N4: per-replica parameters [E, n_params] and shared read-only data of a
        registered env (float32 device tensors, kept alive by the handle; ws_set_env_data)."""
        for name, t in (("prm", prm), ("shared", shared)):
            if t is not None and (t.dtype != torch.float32 or t.device != self.device or not t.is_contiguous()):
                raise WSError(_abi.INVALID_ARGUMENT, f"{name}: contiguous float32 tensor on the handle's device")
        check(lib().ws_set_env_data(self._h, _ptr(prm), _ptr(shared)), self._h)
        self._env_data = (prm, shared)

    def synchronize(self):
        check(lib().ws_synchronize(self._h), self._h)

    def enable_device_clock(self, enable: bool = True):
        """ws.h ws_enable_device_clock: the step index lives on the device (CUDA-graph capture of
        sample / step sequences, policy.PolicyGraph)."""
        check(lib().ws_enable_device_clock(self._h, 1 if enable else 0), self._h)

    def status(self) -> int:
        """ws_synchronize without raising: returns the ws_status."""
        return lib().ws_synchronize(self._h)

    def read_stats(self, t0: int = 0, t1: Optional[int] = None) -> _abi.ws_stats:
        info = self.info()
        out = _abi.ws_stats()
        check(lib().ws_read_stats(self._h, t0, info.cursor if t1 is None else t1, C.byref(out)), self._h)
        return out

    def enable_kernel_timing(self, enable=True, period: int = 1):
        """True / 1: events around every kernel; 2: around the fused roll-out kernel only;
        3: roll-out and GAE; False / 0: off; period P > 1: only every P-th launch of a timed
        class is bracketed (ws.h ws_enable_kernel_timing)."""
        mode = 0 if enable is False else (1 if enable is True else int(enable))
        if not 1 <= int(period) <= 255:
            raise ValueError("period must be in [1, 255]")
        check(lib().ws_enable_kernel_timing(self._h, mode | (int(period) << 8 if period > 1 else 0)), self._h)

    def rollout_policy(self, T: int, weights: torch.Tensor, hidden: int) -> None:
        """NEXT-N1: T fused steps whose actions are drawn from an in-kernel MLP policy
        (ws.h ws_rollout_policy); weights: packed fp32 device tensor."""
        w = weights.contiguous()
        if w.dtype != torch.float32 or w.device != self.device:
            raise ValueError("weights: float32 on the handle's device")
        check(lib().ws_rollout_policy(self._h, T, w.data_ptr(), hidden), self._h)
        self._keep = w  # alive until the stream has consumed it

    def rollout_actor_critic(self, T: int, params: torch.Tensor, hidden: int, values: torch.Tensor,
                             bootstrap: torch.Tensor, values_trunc: Optional[torch.Tensor] = None) -> None:
        """NEXT-N2: the policy roll-out that also writes the critic's values [T, E] and the
        bootstrap values [E] (ws.h ws_rollout_actor_critic); params: R31 packed float32."""
        w = params.contiguous()
        for name, t in (("params", w), ("values", values), ("bootstrap", bootstrap)):
            if t.dtype != torch.float32 or t.device != self.device or not t.is_contiguous():
                raise WSError(_abi.INVALID_ARGUMENT, f"{name}: contiguous float32 on the handle's device")
        if values.numel() < T * self.n_envs or bootstrap.numel() < self.n_envs:
            raise WSError(_abi.INVALID_ARGUMENT, "values [T, E] / bootstrap [E]")
        if values_trunc is not None and (values_trunc.dtype != torch.float32 or values_trunc.device != self.device
                                         or values_trunc.numel() < T * self.n_envs):
            raise WSError(_abi.INVALID_ARGUMENT, "values_trunc: float32 [T, E] on the handle's device")
        check(lib().ws_rollout_actor_critic(self._h, T, w.data_ptr(), hidden, values.data_ptr(),
                                            bootstrap.data_ptr(), _ptr(values_trunc)), self._h)
        self._keep = w

    def gae_store(self, T: int, values: torch.Tensor, bootstrap: torch.Tensor, gamma: float, lam: float,
                  v_trunc: Optional[torch.Tensor] = None, out: Optional[tuple] = None):
        """NEXT-N2: advantages and returns of store slots [0, T) (ws.h ws_gae_store), reading
        the handle's rew / done slabs in place.  values / v_trunc [T, E, A], bootstrap [E, A]
        float32 on the handle's device.  -> (adv, ret) [T, E, A] float32."""
        info = self.info()
        shape = (T, int(info.n_envs), int(info.n_agents))
        for name, t, shp in (("values", values, shape), ("bootstrap", bootstrap, shape[1:]),
                             ("v_trunc", v_trunc, shape)):
            if t is not None and (t.dtype != torch.float32 or t.device != self.device or not t.is_contiguous()
                                  or t.numel() != _numel(shp)):
                raise WSError(_abi.INVALID_ARGUMENT, f"{name}: contiguous float32 {shp} on the handle's device")
        adv, ret = out if out is not None else (torch.empty(shape, dtype=torch.float32, device=self.device),
                                                torch.empty(shape, dtype=torch.float32, device=self.device))
        check(lib().ws_gae_store(self._h, T, _ptr(values), _ptr(bootstrap), _ptr(v_trunc), gamma, lam,
                                 _ptr(adv), _ptr(ret)), self._h)
        return adv, ret

    # ---- cross-GPU statistics over peer memory (ws.h "multi-GPU statistics")
    def peer_export(self, world: int) -> bytes:
        """Allocate this rank's IPC-exportable gather buffer; returns its 64-byte handle."""
        hd = _abi.ws_ipc_handle()
        check(lib().ws_peer_export(self._h, world, C.byref(hd)), self._h)
        return bytes(hd.bytes)

    def peer_attach(self, rank: int, handles) -> None:
        """Open every other rank's buffer; each later rollout() merges the statistics."""
        arr = (_abi.ws_ipc_handle * len(handles))()
        for i, b in enumerate(handles):
            C.memmove(arr[i].bytes, b, 64)
        check(lib().ws_peer_attach(self._h, rank, len(handles), arr), self._h)
        self.peers_attached = len(handles) > 1

    def peer_detach(self) -> None:
        check(lib().ws_peer_detach(self._h), self._h)
        self.peers_attached = False

    def kernel_times(self) -> dict:
        """{kernel class: (launches, mean_ms)} since the last call (ws_kernel_times)."""
        arr = (_abi.ws_kernel_time * 8)()
        n = C.c_int32(0)
        check(lib().ws_kernel_times(self._h, arr, 8, C.byref(n)), self._h)
        return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].mean_ms)) for i in range(n.value)}

    def info(self) -> _abi.ws_info:
        out = _abi.ws_info()
        check(lib().ws_get_info(self._h, C.byref(out)))
        return out

    def stats_f64(self, t1: Optional[int] = None) -> torch.Tensor:
        """Per-slot statistics [t1, 4] as float64 (episodes, sum of returns, sum of lengths,
        sum of rewards), decoded from the exact fixed-point int64 slab."""
        st = self.buffers()["stats"]
        st = st[: (self.info().cursor if t1 is None else t1)]
        return decode_stats(st)

    # ------------------------------------------------------------------ zero-copy views
    def buffers(self) -> dict[str, torch.Tensor]:
        """ws_get_buffers as torch tensors aliasing libws's device memory (no copy)."""
        raw = _abi.ws_buffers()
        check(lib().ws_get_buffers(self._h, C.byref(raw)))
        out = {}
        for name in _abi.BUFFER_NAMES:
            t = getattr(raw, name)
            shape = tuple(int(t.shape[i]) for i in range(t.ndim))
            out[name] = self._view(t.ptr, _TORCH_DTYPE[t.dtype], shape)
        return out

    def _view(self, ptr, dtype, shape) -> Optional[torch.Tensor]:
        if not ptr:
            return None
        n = 1
        for s in shape:
            n *= s
        if self.allocator is not None and ptr in self.allocator.live:
            owner = self.allocator.live[ptr]
            nbytes = n * torch.empty((), dtype=dtype).element_size()
            return owner[:nbytes].view(dtype).view(shape)

        class _CAI:  # __cuda_array_interface__ for buffers libws allocated itself
            pass
        typestr = {torch.float32: "<f4", torch.int32: "<i4", torch.uint8: "|u1", torch.float64: "<f8",
                   torch.uint32: "<u4", torch.int64: "<i8"}[dtype]
        obj = _CAI()
        obj.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (int(ptr), False),
                                        "version": 3, "strides": None}
        return torch.as_tensor(obj, device=self.device)


def register_env(name: str, source: str, state_dim: int, obs_dim: int, n_actions: int, n_reset_draws: int,
                 max_steps: int, n_params: int = 0, act_dim: int = 0) -> str:
    """NEXT-N4: compile a C-source environment with NVRTC into the fused roll-out template
    (ws.h ws_register_env); afterwards Env(E, 1, name, ...) runs it.  Returns the NVRTC log;
    raises WSError (with the log) on a compile error.  Re-registering the same name with the
    same source is a no-op."""
    L = lib()
    if L.ws_registered_env(name.encode()):
        if _REGISTERED.get(name, (source, state_dim, obs_dim, n_actions, act_dim)) != \
                (source, state_dim, obs_dim, n_actions, act_dim):
            raise WSError(_abi.INVALID_ARGUMENT, f"env {name!r} is already registered with a different definition")
        return ""
    d = _abi.ws_env_def(name.encode(), source.encode(), state_dim, obs_dim, n_actions, n_reset_draws, max_steps,
                        n_params, act_dim)
    buf = C.create_string_buffer(1 << 16)
    st = L.ws_register_env(C.byref(d), buf, len(buf))
    log = buf.value.decode(errors="replace")
    if st != _abi.OK:
        raise WSError(st, log)
    _REGISTERED[name] = (source, state_dim, obs_dim, n_actions, act_dim)
    return log


_REGISTERED: dict = {}


def _numel(shape) -> int:
    n = 1
    for s in shape:
        n *= int(s)
    return n


# ---------------------------------------------------------------------- C-ABI-named functions
def ws_create(n_envs: int, n_agents: int, env: str, seed: int) -> Env:
    return Env(n_envs, n_agents, env, seed)


def ws_create_ex(**cfg) -> Env:
    n_envs = cfg.pop("n_envs")
    return Env(n_envs, cfg.pop("n_agents", 1), cfg.pop("env", "cartpole"), cfg.pop("seed", 0), **cfg)


def ws_destroy(h: Env):
    h.close()


def ws_reset(h: Env):
    h.reset()


def ws_rewind(h: Env):
    h.rewind()


def ws_sample(h: Env, probs: torch.Tensor, row_stride: Optional[int] = None):
    h.sample(probs, row_stride)


def ws_step(h: Env, actions: Optional[torch.Tensor] = None):
    h.step(actions)


def ws_rollout(h: Env, T: int, probs: torch.Tensor, row_stride: Optional[int] = None, step_stride: int = 0):
    h.rollout(T, probs, row_stride, step_stride)


def ws_rollout_host(h: Env, T: int, host_probs: torch.Tensor, row_stride: Optional[int] = None, step_stride: int = 0):
    return h.rollout_host(T, host_probs, row_stride, step_stride)


def ws_get_buffers(h: Env) -> dict:
    return h.buffers()


def ws_get_info(h: Env):
    return h.info()


def ws_synchronize(h: Env):
    h.synchronize()


def ws_read_stats(h: Env, t0: int = 0, t1: Optional[int] = None):
    return h.read_stats(t0, t1)


def ws_gae(rew: torch.Tensor, done: torch.Tensor, values: torch.Tensor, bootstrap: torch.Tensor, gamma: float,
           lam: float, v_trunc: Optional[torch.Tensor] = None, out: Optional[tuple] = None):
    """NEXT-N2 generalised advantage estimation (ws.h ws_gae, DESIGN R30) on device arrays:
    rew / values / v_trunc [T, E, A] (or [T, E]) float32, done [T, E] uint8, bootstrap [E, A]
    -> (adv, ret) shaped like rew, enqueued on torch's current stream."""
    T, E = int(rew.shape[0]), int(rew.shape[1])
    A = _numel(rew.shape[2:])
    for name, t, dt, n in (("rew", rew, torch.float32, T * E * A), ("values", values, torch.float32, T * E * A),
                           ("done", done, torch.uint8, T * E), ("bootstrap", bootstrap, torch.float32, E * A),
                           ("v_trunc", v_trunc, torch.float32, T * E * A)):
        if t is not None and (t.dtype != dt or not t.is_cuda or not t.is_contiguous() or t.numel() != n):
            raise WSError(_abi.INVALID_ARGUMENT, f"{name}: contiguous {dt} device tensor with {n} elements")
    adv, ret = out if out is not None else (torch.empty_like(rew), torch.empty_like(rew))
    args = _abi.ws_gae_args(T, A, E, rew.data_ptr(), done.data_ptr(), values.data_ptr(), bootstrap.data_ptr(),
                            v_trunc.data_ptr() if v_trunc is not None else None, gamma, lam,
                            adv.data_ptr(), ret.data_ptr())
    check(lib().ws_gae(C.byref(args), C.c_void_p(torch.cuda.current_stream(rew.device).cuda_stream)))
    return adv, ret


def ws_test_philox(rows: torch.Tensor) -> torch.Tensor:
    """rows: [n, 6] int32/uint32 device (c0..c3, k0, k1) -> [n, 4] Philox words (int32 view)."""
    rows = rows.contiguous()
    out = torch.empty((rows.shape[0], 4), dtype=torch.int32, device=rows.device)
    check(lib().ws_test_philox(_ptr(rows), rows.shape[0], _ptr(out), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out


def ws_test_sample_grid(p: torch.Tensor) -> torch.Tensor:
    """Exhaustive 2^24-grid counts of the library sampler for one row p (n <= 8) -> [n + 1]
    (the last entry counts direct-vs-hoisted search disagreements)."""
    p = p.contiguous().float()
    counts = torch.zeros(p.numel() + 1, dtype=torch.int64, device=p.device)
    check(lib().ws_test_sample_grid(_ptr(p), p.numel(), _ptr(counts), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return counts


def ws_test_unary(fn: int, x: torch.Tensor, param: float = 0.0) -> torch.Tensor:
    """Device elementary function fn (see ws.h) on float32 x (device)."""
    x = x.contiguous().float()
    out = torch.empty_like(x)
    check(lib().ws_test_unary(fn, param, _ptr(x), x.numel(), _ptr(out),
                              C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out


def ws_test_surface_energy(q: torch.Tensor) -> tuple:
    """(energy f32 [n], spring f64 [n]) of the device states q [n, D] by the segmented kernel's code."""
    q = q.contiguous().float()
    n, D = q.shape
    en = torch.empty(n, dtype=torch.float32, device=q.device)
    sp = torch.empty(n, dtype=torch.float64, device=q.device)
    check(lib().ws_test_surface_energy(_ptr(q), D, n, _ptr(en), _ptr(sp),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return en, sp


def ws_test_exhaustive(fn_a: int, fn_b: int, lo_bits: int, hi_bits: int, param: float = 0.0) -> int:
    """Number of fp32 bit patterns in [lo_bits, hi_bits] where device functions differ."""
    m = C.c_uint64(0)
    check(lib().ws_test_exhaustive(fn_a, fn_b, param, lo_bits, hi_bits, C.byref(m),
                                   C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return int(m.value)
