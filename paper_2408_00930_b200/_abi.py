"""ctypes mirror of include/ws.h (argument marshalling only -- every step of the roll-out
runs in libws's CUDA kernels).  Loading fails loudly if libws.so is missing: there is no
CPU fallback on the product path."""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WS_LIBWS") or os.path.join(HERE, "lib", "libws.so")  # override: profiling experiments
HEADER = os.path.join(os.path.dirname(HERE), "include", "ws.h")

# ws_status
(OK, INVALID_ARGUMENT, UNKNOWN_ENV, INVALID_ACTION, INVALID_PROBS, OUT_OF_RANGE, BAD_STATE, OUT_OF_MEMORY, CUDA_ERROR,
 PEER_ERROR) = range(10)
STATUS_NAMES = {0: "WS_OK", 1: "WS_ERR_INVALID_ARGUMENT", 2: "WS_ERR_UNKNOWN_ENV", 3: "WS_ERR_INVALID_ACTION",
                4: "WS_ERR_INVALID_PROBS", 5: "WS_ERR_OUT_OF_RANGE", 6: "WS_ERR_BAD_STATE",
                7: "WS_ERR_OUT_OF_MEMORY", 8: "WS_ERR_CUDA", 9: "WS_ERR_PEER"}
# ws_dtype
F32, I32, U8, F64, U32, I64 = range(6)
FX_SCALE = 2.0 ** -32  # fixed-point scale of stats[:, 1] and stats[:, 3]

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class ws_config(C.Structure):
    _fields_ = [
        ("n_envs", C.c_int64), ("env_offset", C.c_int64), ("n_envs_global", C.c_int64),
        ("n_agents", C.c_int32), ("env", C.c_char_p), ("seed", C.c_uint64),
        ("device", C.c_int32), ("stream", C.c_void_p),
        ("t_capacity", C.c_int32), ("max_steps", C.c_int32), ("write_logp", C.c_int32),
        ("param0", C.c_int32), ("param1", C.c_int32), ("block_size", C.c_int32),
        ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_user", C.c_void_p),
        ("env_prm", C.c_void_p), ("env_shared", C.c_void_p),
    ]


class ws_ipc_handle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64)]


class ws_tensor(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("dtype", C.c_int32), ("ndim", C.c_int32), ("shape", C.c_int64 * 5)]


BUFFER_NAMES = ["obs", "act", "logp", "rew", "done", "stats", "state", "obs_live", "ep_step", "reset_count", "ep_ret"]


class ws_buffers(C.Structure):
    _fields_ = [(n, ws_tensor) for n in BUFFER_NAMES]


class ws_info(C.Structure):
    _fields_ = [
        ("obs_dim", C.c_int32), ("n_actions", C.c_int32), ("act_dim", C.c_int32), ("state_dim", C.c_int32),
        ("max_steps", C.c_int32), ("n_agents", C.c_int32), ("t_capacity", C.c_int32), ("cursor", C.c_int32),
        ("n_envs", C.c_int64), ("env_offset", C.c_int64), ("n_envs_global", C.c_int64),
        ("t", C.c_uint64), ("launches", C.c_uint64), ("probs_width", C.c_int32), ("reserved", C.c_int32),
    ]


class ws_stats(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("episodes", "sum_return", "sum_length", "sum_reward", "mean_return", "mean_length")]


class ws_kernel_time(C.Structure):
    _fields_ = [("name", C.c_char_p), ("launches", C.c_int32), ("mean_ms", C.c_float), ("total_ms", C.c_float)]


class ws_gae_args(C.Structure):
    _fields_ = [("T", C.c_int32), ("n_agents", C.c_int32), ("n_envs", C.c_int64),
                ("rew", C.c_void_p), ("done", C.c_void_p), ("values", C.c_void_p), ("bootstrap", C.c_void_p),
                ("v_trunc", C.c_void_p), ("gamma", C.c_float), ("lam", C.c_float),
                ("adv", C.c_void_p), ("ret", C.c_void_p)]


class ws_a2c_args(C.Structure):
    _fields_ = [("obs_dim", C.c_int32), ("hidden", C.c_int32), ("n_actions", C.c_int32), ("rows", C.c_int64),
                ("params", C.c_void_p), ("obs", C.c_void_p), ("act", C.c_void_p), ("adv", C.c_void_p),
                ("ret", C.c_void_p), ("moments", C.c_void_p), ("batch", C.c_double), ("c_v", C.c_float),
                ("c_e", C.c_float), ("workspace", C.c_void_p), ("grad", C.c_void_p), ("loss", C.c_void_p),
                ("logp_old", C.c_void_p), ("clip_eps", C.c_float), ("norm_batch", C.c_double),
                ("gaussian", C.c_int32), ("act_f", C.c_void_p)]


class ws_host_store(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("obs", "act", "logp", "rew", "done")]


class ws_staged_report(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("total_ms", "transfer_ms", "h2d_bytes", "d2h_bytes")]


class ws_env_def(C.Structure):
    _fields_ = [("name", C.c_char_p), ("source", C.c_char_p), ("state_dim", C.c_int32), ("obs_dim", C.c_int32),
                ("n_actions", C.c_int32), ("n_reset_draws", C.c_int32), ("max_steps", C.c_int32),
                ("n_params", C.c_int32), ("act_dim", C.c_int32)]


_SIGS = {
    "ws_config_init": (C.c_int, [C.POINTER(ws_config)]),
    "ws_create": (C.c_int, [C.c_int64, C.c_int32, C.c_char_p, C.c_uint64, C.POINTER(C.c_void_p)]),
    "ws_create_ex": (C.c_int, [C.POINTER(ws_config), C.POINTER(C.c_void_p)]),
    "ws_destroy": (C.c_int, [C.c_void_p]),
    "ws_reset": (C.c_int, [C.c_void_p]),
    "ws_rewind": (C.c_int, [C.c_void_p]),
    "ws_sample": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "ws_step": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ws_rollout": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int64]),
    "ws_rollout_host": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                  C.POINTER(ws_stats)]),
    "ws_rollout_staged": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                    C.POINTER(ws_host_store), C.POINTER(ws_staged_report)]),
    "ws_register_env": (C.c_int, [C.POINTER(ws_env_def), C.c_char_p, C.c_size_t]),
    "ws_registered_env": (C.c_int32, [C.c_char_p]),
    "ws_set_env_data": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ws_set_time": (C.c_int, [C.c_void_p, C.c_uint64]),
    "ws_rollout_host_submit": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int32]),
    "ws_rollout_host_wait": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "ws_enable_device_clock": (C.c_int, [C.c_void_p, C.c_int32]),
    "ws_pgroup_create": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(ws_ipc_handle)]),
    "ws_pgroup_attach": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(ws_ipc_handle)]),
    "ws_pgroup_destroy": (C.c_int, [C.c_void_p]),
    "ws_pgroup_status": (C.c_int, [C.c_void_p]),
    "ws_pgroup_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "ws_pgroup_allreduce_adam": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                           C.c_float, C.c_float, C.c_float, C.c_float, C.c_float, C.c_void_p,
                                           C.c_void_p, C.c_void_p]),
    "ws_get_buffers": (C.c_int, [C.c_void_p, C.POINTER(ws_buffers)]),
    "ws_get_info": (C.c_int, [C.c_void_p, C.POINTER(ws_info)]),
    "ws_synchronize": (C.c_int, [C.c_void_p]),
    "ws_read_stats": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(ws_stats)]),
    "ws_status_string": (C.c_char_p, [C.c_int]),
    "ws_last_error": (C.c_char_p, [C.c_void_p]),
    "ws_abi_version": (C.c_int32, []),
    "ws_enable_kernel_timing": (C.c_int, [C.c_void_p, C.c_int32]),
    "ws_rollout_policy": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32]),
    "ws_rollout_actor_critic": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_void_p]),
    "ws_gae": (C.c_int, [C.POINTER(ws_gae_args), C.c_void_p]),
    "ws_gae_store": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_float,
                               C.c_void_p, C.c_void_p]),
    "ws_a2c_n_params": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32]),
    "ws_a2c_n_params_ex": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "ws_a2c_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32]),
    "ws_ac_values": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                               C.c_void_p]),
    "ws_a2c_moments": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ws_a2c_grad": (C.c_int, [C.POINTER(ws_a2c_args), C.c_void_p]),
    "ws_clamp": (C.c_int, [C.c_void_p, C.c_int32, C.c_float, C.c_float, C.c_void_p]),
    "ws_adam": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_float,
                          C.c_float, C.c_float, C.c_float, C.c_float, C.c_void_p, C.c_void_p]),
    "ws_peer_export": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(ws_ipc_handle)]),
    "ws_peer_attach": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(ws_ipc_handle)]),
    "ws_peer_detach": (C.c_int, [C.c_void_p]),
    "ws_kernel_times": (C.c_int, [C.c_void_p, C.POINTER(ws_kernel_time), C.c_int32, C.POINTER(C.c_int32)]),
    "ws_test_philox": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "ws_test_sample_grid": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "ws_test_unary": (C.c_int, [C.c_int32, C.c_float, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "ws_test_surface_energy": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ws_test_exhaustive": (C.c_int, [C.c_int32, C.c_int32, C.c_float, C.c_uint32, C.c_uint32,
                                     C.POINTER(C.c_uint64), C.c_void_p]),
}

_lib = None


def declared_functions(header: str = HEADER) -> list[str]:
    """Names of the functions include/ws.h declares."""
    src = open(header).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ws_[a-z_0-9]+)\s*\(", src)) - {"ws_alloc_fn", "ws_free_fn"})


def lib() -> C.CDLL:
    """Load libws.so (built by paper_2408_00930_b200.build / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libws.so not found at {LIB_PATH}: build it with `python paper_2408_00930_b200/build.py` "
                "(there is no CPU fallback on the product path)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class WSError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        self.status = status
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {detail}" if detail else STATUS_NAMES.get(status, str(status)))


def check(status: int, handle=None):
    if status != OK:
        detail = ""
        if handle:
            raw = lib().ws_last_error(handle)
            detail = raw.decode() if raw else ""
        raise WSError(status, detail)
