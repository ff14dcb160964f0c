"""Multi-GPU plumbing: one process per GPU, replicas
sharded contiguously across ranks, and the one real exchange of the path -- the sum
all-reduce of the per-slot episode statistics (BJ:5 "NCCL over NVLink used only for the
per-step episode-return and statistics all-reduce").

Every Philox stream is keyed by the GLOBAL replica index (DESIGN R15), so each replica's
trajectory is bit-identical whatever the number of ranks; only the statistics cross GPUs.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def shard(n_envs_global: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced replica range of `rank` (S:167-175 partition_lanes): sizes differ
    by at most 1; returns (env_offset, n_envs)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need world >= 1 and 0 <= rank < world")
    lo = n_envs_global * rank // world
    hi = n_envs_global * (rank + 1) // world
    return lo, hi - lo


def allreduce_stats(stats: torch.Tensor, group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """In-place SUM all-reduce of a [T, 4] statistics view across ranks (NCCL on the GPU
    path; gloo in the CPU tests).  libws's slab is exact fixed-point int64 (DESIGN R20), so
    the merged statistics are bit-identical for any number of ranks.  (Handles attached with
    attach_peer_stats already merge inside ws_rollout; their callers skip this.)"""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def attach_peer_stats(env, group: Optional[dist.ProcessGroup] = None) -> bool:
    """Collective: switch `env` to the NCCL-free statistics all-reduce over CUDA-IPC peer
    memory (libws ws_peer_export / ws_peer_attach): from now on every env.rollout() leaves
    the merged [T,4] statistics of all ranks in its stats slab.  Returns False (and leaves
    the NCCL path in place) when IPC is unavailable on any rank."""
    if not (dist.is_available() and dist.is_initialized()):
        return False
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world < 2:
        return False
    try:
        h = env.peer_export(world)
        err = None
    except Exception as ex:  # noqa: BLE001 -- reported collectively below
        h, err = b"", repr(ex)
    handles = [None] * world
    dist.all_gather_object(handles, (h, err), group=group)
    if any(e for _, e in handles):
        return False
    ok = True
    try:
        env.peer_attach(rank, [hh for hh, _ in handles])
    except Exception:  # noqa: BLE001
        ok = False
    flags = [None] * world
    dist.all_gather_object(flags, ok, group=group)
    if not all(flags):
        if ok:
            env.peer_detach()
        return False
    dist.barrier(group)
    return True


def summarize(stats: torch.Tensor) -> dict:
    """Episode statistics over slots (P:93 average episodic reward, P:132 episodic step).
    Accepts libws's fixed-point int64 slab or already-decoded float64 rows."""
    if stats.dtype == torch.int64:
        s = stats.sum(dim=0).tolist()
        s = [s[0], s[1] * 2.0 ** -32, s[2], s[3] * 2.0 ** -32]
    else:
        s = stats.double().sum(dim=0).tolist()
    n = s[0]
    return {"episodes": n, "mean_return": s[1] / n if n else float("nan"),
            "mean_length": s[2] / n if n else float("nan"), "sum_reward": s[3]}


class PeerGroup:
    """Collective: a libws peer group (ws.h "peer groups") of `n` values across the ranks of
    `group` on their current devices -- fp64 sums over CUDA-IPC peer memory, optionally fused
    with the clip + Adam step.  Raises RuntimeError (on every rank) if IPC is unavailable."""

    def __init__(self, n: int, group: Optional[dist.ProcessGroup] = None):
        import ctypes as C
        from . import _abi
        from ._abi import lib
        self._C, self._abi, self._lib = C, _abi, lib()
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        h = _abi.ws_ipc_handle()
        g = C.c_void_p()
        st = self._lib.ws_pgroup_create(world, n, C.byref(g), C.byref(h))
        blobs = [None] * world
        dist.all_gather_object(blobs, (bytes(h.bytes), st), group=group)
        if any(s != 0 for _, s in blobs):
            if g:
                self._lib.ws_pgroup_destroy(g)
            raise RuntimeError("peer group: cudaIpc export failed on some rank")
        arr = (_abi.ws_ipc_handle * world)()
        for r, (b, _) in enumerate(blobs):
            C.memmove(arr[r].bytes, b, 64)
        st = self._lib.ws_pgroup_attach(g, rank, arr)
        oks = [None] * world
        dist.all_gather_object(oks, st == 0, group=group)
        if not all(oks):
            self._lib.ws_pgroup_destroy(g)
            raise RuntimeError("peer group: cudaIpcOpenMemHandle failed on some rank")
        dist.barrier(group)
        self._g, self.n, self.world, self.rank = g, n, world, rank

    def allreduce(self, x: torch.Tensor, out: torch.Tensor, stream=None):
        """out (fp64) = sum over ranks of x (fp32 or fp64), identical on every rank."""
        s = self._C.c_void_p((stream or torch.cuda.current_stream(x.device)).cuda_stream)
        st = self._lib.ws_pgroup_allreduce(self._g, x.data_ptr(), 1 if x.dtype == torch.float32 else 0,
                                           out.data_ptr(), s)
        if st != 0:
            raise RuntimeError(f"ws_pgroup_allreduce: {st}")

    def allreduce_adam(self, grad, params, m, v, step, lr, beta1, beta2, eps, max_norm, grad_out=None,
                       grad_norm=None, stream=None):
        s = self._C.c_void_p((stream or torch.cuda.current_stream(grad.device)).cuda_stream)
        st = self._lib.ws_pgroup_allreduce_adam(
            self._g, grad.data_ptr(), params.data_ptr(), m.data_ptr(), v.data_ptr(), step, lr, beta1, beta2, eps,
            max_norm, None if grad_out is None else grad_out.data_ptr(),
            None if grad_norm is None else grad_norm.data_ptr(), s)
        if st != 0:
            raise RuntimeError(f"ws_pgroup_allreduce_adam: {st}")

    def status(self) -> int:
        return int(self._lib.ws_pgroup_status(self._g))

    def close(self):
        if getattr(self, "_g", None):
            self._lib.ws_pgroup_destroy(self._g)
            self._g = None
