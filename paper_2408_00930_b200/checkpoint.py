"""Checkpoint / resume ("parameter checkpoint format: flat
little-endian float32 file with a small header (magic, layer sizes, head type); bit-exact
round-trip required").

* save_params / load_params -- the packed actor-critic parameters (R31 / R35 layout) as
  header + float32 LE payload; the round trip is bit-exact.
* env_state / load_env_state -- a handle's live state (per-replica state, observations,
  episode counters, the step index t); because every draw is keyed by (seed, replica, agent,
  t, reset count) (R15), a restored handle continues bit-identically.
* trainer_state / load_trainer_state -- parameters, Adam moments and step of an A2C / PPO.
"""
from __future__ import annotations

import struct
from typing import Optional

import numpy as np
import torch

from ._abi import check, lib

MAGIC = b"WSAC"
VERSION = 1
HEADS = {"softmax": 0, "gaussian": 1}
_HDR = struct.Struct("<4sIIIIIQ")  # magic, version, obs_dim, hidden, n_actions, head, n_floats


def save_params(path: str, params: torch.Tensor, obs_dim: int, hidden: int, n_actions: int,
                head: str = "softmax") -> None:
    p = params.detach().to("cpu", torch.float32).contiguous().numpy()
    with open(path, "wb") as f:
        f.write(_HDR.pack(MAGIC, VERSION, obs_dim, hidden, n_actions, HEADS[head], p.size))
        f.write(p.astype("<f4", copy=False).tobytes())


def load_params(path: str, device=None) -> tuple[torch.Tensor, dict]:
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < _HDR.size:
        raise ValueError("checkpoint: truncated header")
    magic, ver, D, H, N, head, n = _HDR.unpack_from(raw)
    if magic != MAGIC or ver != VERSION:
        raise ValueError("checkpoint: not a WSAC v1 parameter file")
    if len(raw) != _HDR.size + 4 * n:
        raise ValueError("checkpoint: payload size does not match the header")
    p = np.frombuffer(raw, dtype="<f4", offset=_HDR.size, count=n).astype(np.float32)
    meta = {"obs_dim": D, "hidden": H, "n_actions": N, "head": {v: k for k, v in HEADS.items()}[head]}
    t = torch.from_numpy(p.copy())
    return (t.to(device) if device is not None else t), meta


_LIVE = ("state", "obs_live", "ep_step", "reset_count", "ep_ret")


def env_state(env) -> dict:
    """CPU copy of a handle's live state and step index (call after the stream is idle)."""
    env.synchronize()
    buf = env.buffers()
    d = {k: buf[k].detach().cpu().clone() for k in _LIVE if buf.get(k) is not None}
    d["t"] = int(env.info().t)
    return d


def load_env_state(env, d: dict) -> None:
    """Restore env_state(...) into a handle created with the same configuration."""
    buf = env.buffers()
    for k in _LIVE:
        if k in d:
            if buf[k] is None or buf[k].shape != d[k].shape:
                raise ValueError(f"checkpoint: {k} does not match this handle")
            buf[k].copy_(d[k].to(buf[k].device))
    torch.cuda.synchronize(env.device)
    check(lib().ws_set_time(env.handle, int(d["t"])), env.handle)


def trainer_state(tr) -> dict:
    return {"params": tr.params.detach().cpu().clone(), "m": tr.m.detach().cpu().clone(),
            "v": tr.v.detach().cpu().clone(), "step": tr.step}


def load_trainer_state(tr, d: dict) -> None:
    for k in ("params", "m", "v"):
        getattr(tr, k).copy_(d[k].to(tr.params.device))
    tr.step = int(d["step"])
