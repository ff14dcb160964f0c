"""paper_2408_00930_b200 -- B200-native (sm_100a) batched environment roll-out engine of
WarpSci (arXiv 2408.00930): GPU-resident replicas, Philox-driven warp-scan sampling,
fused multi-step roll-out with auto-reset into a time-major in-place store, behind the
C ABI of include/ws.h (libws.so).  See DESIGN.md.

Importing this package never falls back to a CPU implementation: the binding raises if
libws.so has not been built (`python paper_2408_00930_b200/build.py`).
"""
from ._abi import WSError, declared_functions, lib  # noqa: F401
from .env import (Env, register_env, ws_gae, ws_create, ws_create_ex, ws_destroy, ws_get_buffers, ws_get_info,  # noqa: F401
                  ws_read_stats, ws_reset, ws_rewind, ws_rollout, ws_rollout_host, ws_sample, ws_step,
                  ws_synchronize, ws_test_exhaustive, ws_test_philox, ws_test_sample_grid, ws_test_surface_energy, ws_test_unary)

lib()  # load libws.so now: a missing extension is an ImportError, never a silent fallback

__all__ = ["Env", "register_env", "WSError", "ws_gae", "lib", "declared_functions", "ws_create", "ws_create_ex", "ws_destroy",
           "ws_reset", "ws_rewind", "ws_sample", "ws_step", "ws_rollout", "ws_rollout_host", "ws_get_buffers",
           "ws_get_info", "ws_synchronize", "ws_read_stats", "ws_test_philox", "ws_test_sample_grid", "ws_test_unary", "ws_test_exhaustive",
           "ws_test_surface_energy"]
