"""CPU oracle of the WarpSci roll-out hot path -- ctypes binding of ``oracle/wso.cpp``.

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and its ``--impl reference`` arm) may import this
package.  The product package ``paper_2408_00930_b200`` never imports it, and this
package never imports the product package: the two share no code.

Every numerical function of ``wso.cpp`` cites the PAPER.md / SPEC.md passage it follows
and is pinned by ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wso.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

# Same status numbering as the written contract in DESIGN.md (restated here, not shared).
OK, INVALID_ARGUMENT, UNKNOWN_ENV, INVALID_ACTION, INVALID_PROBS, OUT_OF_RANGE, BAD_STATE = range(7)


def build(force: bool = False) -> str:
    """Compile wso.cpp with -O2 -ffp-contract=off (no FMA contraction, DESIGN R4)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lpthread"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P, I, I64, U32, U64, F, D = C.c_void_p, C.c_int, C.c_int64, C.c_uint32, C.c_uint64, C.c_float, C.c_double
        sig = {
            "wso_philox4x32_10": (None, [P, P, P]),
            "wso_draw": (U32, [U64, U64, U32, U32, U64]),
            "wso_u01": (F, [U32]),
            "wso_gauss": (F, [U64, U64, U32, U64, I, I]),
            "wso_box_muller": (F, [U32, U32, I]),
            "wso_sample_discrete": (I, [P, I, F, P, P, P]),
            "wso_sample_grid": (I64, [P, I, P]),
            "wso_sincos_f32": (None, [P, I64, P, P]),
            "wso_cartpole_step_f32": (I, [P, I, P, P, P]),
            "wso_cartpole_step_f64": (I, [P, I, P, P, P]),
            "wso_acrobot_step_f32": (I, [P, I, P, P, P]),
            "wso_acrobot_step_f64": (I, [P, I, P, P, P]),
            "wso_acrobot_dsdt_f64": (None, [P, D, P]),
            "wso_acrobot_terminal_f32": (I, [P]),
            "wso_pendulum_step_f32": (I, [P, F, P, P]),
            "wso_pendulum_step_f64": (I, [P, D, P, P]),
            "wso_mb_energy": (D, [D, D, P, P]),
            "wso_surface_energy": (F, [P, I]),
            "wso_surface_spring": (D, [P, I]),
            "wso_surface_step": (I, [P, P, I, P, P, P]),
            "wso_tag_step": (I, [I, I, I, P, P, P, P, P, P]),
            "wso_create": (P, [C.c_char_p, I64, I, U64, I64, I64, I, I, I, P]),
            "wso_destroy": (None, [P]),
            "wso_set_capacity": (I, [P, I]),
            "wso_reset": (I, [P]),
            "wso_register_user": (I, [C.c_char_p, C.c_char_p, I, I, I, I, I, I, I]),
            "wso_policy_gauss_rows": (I, [P, I, I, I, P, I64, P]),
            "wso_rollout_policy_gauss": (I, [P, I, P, I, I]),
            "wso_set_env_data": (I, [P, P, I64, P, I64]),
            "wso_sample": (I, [P, P, I64, P, P]),
            "wso_step": (I, [P, P]),
            "wso_rollout": (I, [P, I, P, I64, I64, P, P, I]),
            "wso_rollout_policy": (I, [P, I, P, I, I]),
            "wso_policy_probs": (I, [P, I, I, I, P, I64, P]),
            "wso_policy_logits": (I, [P, I, I, I, P, I64, P]),
            "wso_gae_f32": (I, [I, I64, I, P, P, P, P, P, F, F, P, P]),
            "wso_gae_f64": (I, [I, I64, I, P, P, P, P, P, D, D, P, P]),
            "wso_synchronize": (I, [P]),
            "wso_info": (None, [P, P]),
            "wso_get": (P, [P, C.c_char_p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------------------- unit functions
def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().wso_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def draw(seed: int, env_global: int, agent: int, purpose: int, j: int) -> int:
    return int(lib().wso_draw(seed, env_global, agent, purpose, j))


def u01(w: int) -> float:
    return float(lib().wso_u01(w))


def box_muller(wa: int, wb: int, odd: int) -> float:
    """Box-Muller on the word pair (wa, wb): the cos (odd = 0) or sin (odd = 1) normal."""
    return float(lib().wso_box_muller(wa, wb, odd))


def gauss(seed: int, env_global: int, agent: int, t: int, d: int, k: int) -> float:
    return float(lib().wso_gauss(seed, env_global, agent, t, d, k))


def sample_discrete(p, u: float):
    """-> (status, action, logp, ambiguous)"""
    pa = np.ascontiguousarray(p, dtype=np.float32)
    a = np.zeros(1, np.int32); lp = np.zeros(1, np.float32); amb = np.zeros(1, np.int32)
    st = lib().wso_sample_discrete(_p(pa), len(pa), np.float32(u), _p(a), _p(lp), _p(amb))
    return st, int(a[0]), float(lp[0]), bool(amb[0])


def policy_logits(weights, D: int, H: int, N: int, obs) -> np.ndarray:
    """Second-layer outputs (R29' quarter sums) of observations [n, D] -> [n, N]."""
    weights = np.ascontiguousarray(weights, dtype=np.float32)
    obs = np.ascontiguousarray(obs, dtype=np.float32).reshape(-1, D)
    out = np.zeros((obs.shape[0], N), np.float32)
    assert lib().wso_policy_logits(_p(weights), D, H, N, _p(obs), obs.shape[0], _p(out)) == 0
    return out


def policy_probs(weights, D: int, H: int, N: int, obs) -> np.ndarray:
    """MLP policy probabilities (R29) of observations [n, D] -> [n, N]."""
    weights = np.ascontiguousarray(weights, dtype=np.float32)
    obs = np.ascontiguousarray(obs, dtype=np.float32).reshape(-1, D)
    out = np.zeros((obs.shape[0], N), np.float32)
    assert lib().wso_policy_probs(_p(weights), D, H, N, _p(obs), obs.shape[0], _p(out)) == 0
    return out


def policy_gauss_rows(weights, D: int, H: int, d: int, obs) -> np.ndarray:
    """Gaussian policy head rows (mean | log_std, R34) of observations [n, D] -> [n, 2d]."""
    weights = np.ascontiguousarray(weights, dtype=np.float32)
    obs = np.ascontiguousarray(obs, dtype=np.float32).reshape(-1, D)
    out = np.zeros((obs.shape[0], 2 * d), np.float32)
    assert lib().wso_policy_gauss_rows(_p(weights), D, H, d, _p(obs), obs.shape[0], _p(out)) == 0
    return out


def gae(rew, done, values, bootstrap, gamma, lam, v_trunc=None, f64=False):
    """NEXT-N2 GAE (wso.cpp gae, DESIGN R30): rew / values / v_trunc [T, E, A] (or [T, E]),
    done [T, E] u8, bootstrap [E, A] -> (advantages, returns), same shape as rew."""
    dt = np.float64 if f64 else np.float32
    rew = np.ascontiguousarray(rew, dtype=dt)
    T, E = rew.shape[0], rew.shape[1]
    A = int(np.prod(rew.shape[2:])) if rew.ndim > 2 else 1
    done = np.ascontiguousarray(done, dtype=np.uint8).reshape(T, E)
    values = np.ascontiguousarray(values, dtype=dt).reshape(rew.shape)
    bootstrap = np.ascontiguousarray(bootstrap, dtype=dt).reshape(E * A)
    vt = None if v_trunc is None else np.ascontiguousarray(v_trunc, dtype=dt).reshape(rew.shape)
    adv = np.zeros(rew.shape, dt); ret = np.zeros(rew.shape, dt)
    fn = lib().wso_gae_f64 if f64 else lib().wso_gae_f32
    st = fn(T, E, A, _p(rew), _p(done), _p(values), _p(bootstrap), _p(vt), dt(gamma), dt(lam),
            _p(adv), _p(ret))
    assert st == 0, st
    return adv, ret


def sample_grid(p):
    """Exhaustive u = k 2^-24 grid -> (counts[n], n_ambiguous)."""
    pa = np.ascontiguousarray(p, dtype=np.float32)
    counts = np.zeros(len(pa), np.int64)
    amb = lib().wso_sample_grid(_p(pa), len(pa), _p(counts))
    return counts, int(amb)


def sincos_f32(x):
    """(float)sin((double)x), (float)cos((double)x) with the host libm (reading Q3)."""
    xa = np.ascontiguousarray(x, dtype=np.float32)
    s = np.empty_like(xa); c = np.empty_like(xa)
    lib().wso_sincos_f32(_p(xa), xa.size, _p(s), _p(c))
    return s, c


def _step4(fn32, fn64, s, a, f64):
    dt = np.float64 if f64 else np.float32
    sa = np.ascontiguousarray(s, dtype=dt)
    out = np.zeros(4, dt); r = np.zeros(1, dt); term = np.zeros(1, np.int32)
    st = (fn64 if f64 else fn32)(_p(sa), int(a), _p(out), _p(r), _p(term))
    return st, out, r[0], bool(term[0])


def cartpole_step(s, a, f64=False):
    L = lib()
    return _step4(L.wso_cartpole_step_f32, L.wso_cartpole_step_f64, s, a, f64)


def acrobot_step(s, a, f64=False):
    L = lib()
    return _step4(L.wso_acrobot_step_f32, L.wso_acrobot_step_f64, s, a, f64)


def acrobot_dsdt(s, torque) -> np.ndarray:
    sa = np.ascontiguousarray(s, dtype=np.float64)
    d = np.zeros(4, np.float64)
    lib().wso_acrobot_dsdt_f64(_p(sa), float(torque), _p(d))
    return d


def acrobot_terminal(s) -> bool:
    sa = np.ascontiguousarray(s, dtype=np.float32)
    return bool(lib().wso_acrobot_terminal_f32(_p(sa)))


def pendulum_step(s, u, f64=False):
    dt = np.float64 if f64 else np.float32
    sa = np.ascontiguousarray(s, dtype=dt)
    out = np.zeros(2, dt); r = np.zeros(1, dt)
    fn = lib().wso_pendulum_step_f64 if f64 else lib().wso_pendulum_step_f32
    st = fn(_p(sa), dt(u), _p(out), _p(r))
    return st, out, r[0]


def mb_energy(x, y):
    gx = np.zeros(1); gy = np.zeros(1)
    e = lib().wso_mb_energy(float(x), float(y), _p(gx), _p(gy))
    return e, gx[0], gy[0]


def surface_spring(q) -> float:
    """The fp64 spring sum of q_i^2 (i >= 2) in R23's pairwise order."""
    qa = np.ascontiguousarray(q, np.float32)
    return float(lib().wso_surface_spring(_p(qa), len(qa)))


def surface_energy(q) -> float:
    qa = np.ascontiguousarray(q, dtype=np.float32)
    return float(lib().wso_surface_energy(_p(qa), len(qa)))


def surface_step(q, a):
    qa = np.ascontiguousarray(q, dtype=np.float32)
    aa = np.ascontiguousarray(a, dtype=np.float32)
    out = np.zeros_like(qa); r = np.zeros(1, np.float32); term = np.zeros(1, np.int32)
    st = lib().wso_surface_step(_p(qa), _p(aa), len(qa), _p(out), _p(r), _p(term))
    return st, out, float(r[0]), bool(term[0])


def tag_step(G, n_taggers, x, y, active, act):
    x = np.array(x, dtype=np.int32); y = np.array(y, dtype=np.int32)
    active = np.array(active, dtype=np.uint8); act = np.ascontiguousarray(act, dtype=np.int32)
    A = len(x)
    rew = np.zeros(A, np.float32); term = np.zeros(1, np.int32)
    st = lib().wso_tag_step(A, G, n_taggers, _p(x), _p(y), _p(active), _p(act), _p(rew), _p(term))
    return st, x, y, active, rew, bool(term[0])


# ----------------------------------------------------------------------------- batch
class _View(np.ndarray):
    """ndarray view that holds a reference to its owning Batch."""

    def __new__(cls, arr, owner):
        v = arr.view(cls)
        v._owner = owner
        return v

    def __array_finalize__(self, obj):
        self._owner = getattr(obj, "_owner", None)


# ------------------------------------------------------------------ NEXT-N4 registered envs
# The oracle's own prelude for a user environment's C source (the composer's input, contract
# in include/ws.h): transcendental contract R3 (fp64 evaluation, one rounding), correctly
# rounded sqrt, the same min / max / clip definitions; compiled without FMA contraction.
_USER_PRELUDE = r"""
#include <cmath>
#define WS_FN static inline
static inline float ws_sin(float x) { return (float)std::sin((double)x); }
static inline float ws_cos(float x) { return (float)std::cos((double)x); }
static inline float ws_exp(float x) { return (float)std::exp((double)x); }
static inline float ws_log(float x) { return (float)std::log((double)x); }
static inline float ws_tanh(float x) { return (float)std::tanh((double)x); }
static inline float ws_sqrt(float x) { return std::sqrt(x); }
static inline float ws_min(float a, float b) { return b < a ? b : a; }
static inline float ws_max(float a, float b) { return a < b ? b : a; }
static inline float ws_clip(float x, float lo, float hi) { return x < lo ? lo : (hi < x ? hi : x); }
static inline float ws_abs(float x) { return std::fabs(x); }
static inline float ws_floor(float x) { return std::floor(x); }
static inline float ws_fmod(float x, float y) { return std::fmod(x, y); }
static inline void ws_sincos(float x, float* s, float* c) { *s = (float)std::sin((double)x); *c = (float)std::cos((double)x); }
#line 1 "user_env.c"
"""
_USER_EPILOGUE = r"""
extern "C" {
void wsu_init(float* s, const float* u, const float* p, const float* sh) { ws_env_init(s, u, p, sh); }
void wsu_obs(const float* s, float* o, const float* p, const float* sh) { ws_env_obs(s, o, p, sh); }
#if WS_C > 0
int wsu_step(float* s, const float* a, float* r, const float* p, const float* sh) { return ws_env_step(s, a, r, p, sh); }
#else
int wsu_step(float* s, int a, float* r, const float* p, const float* sh) { return ws_env_step(s, a, r, p, sh); }
#endif
}
"""
_USER_ENVS = set()


def register_user_env(name: str, source: str, state_dim: int, obs_dim: int, n_actions: int, n_reset_draws: int,
                      max_steps: int, n_params: int = 0, act_dim: int = 0) -> str:
    """Compile a user environment's C source with g++ (-O2 -ffp-contract=off) and register it
    with the oracle under `name`; Batch(name, ...) then simulates it.  Returns the .so path."""
    import hashlib
    defs = (f"#define WS_S {state_dim}\n#define WS_D {obs_dim}\n#define WS_N {n_actions}\n"
            f"#define WS_R {n_reset_draws}\n#define WS_P {n_params}\n#define WS_C {act_dim}\n")
    text = defs + _USER_PRELUDE + source + "\n" + _USER_EPILOGUE
    key = hashlib.sha1(text.encode()).hexdigest()[:12]
    d = os.path.join(_HERE, "build_user")
    os.makedirs(d, exist_ok=True)
    so = os.path.join(d, f"{name}_{key}.so")
    if not os.path.exists(so):
        src = so[:-3] + ".cpp"
        with open(src, "w") as f:
            f.write(text)
        subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                        "-o", so + ".tmp", src], check=True)
        os.replace(so + ".tmp", so)
    st = lib().wso_register_user(name.encode(), so.encode(), state_dim, obs_dim, n_actions, n_reset_draws,
                                 max_steps, n_params, act_dim)
    if st != OK:
        raise ValueError(f"wso_register_user failed ({st})")
    _USER_ENVS.add(name)
    return so


class Batch:
    """make_batch .. run_rollout on the CPU; arrays are numpy views of the
    oracle's own storage (valid until the next set_capacity / destroy)."""

    def __init__(self, env: str, n_envs: int, n_agents: int = 1, seed: int = 0, *,
                 env_offset: int = 0, n_envs_global: int = 0, max_steps: int = 0,
                 p0: int = 0, p1: int = 0, t_capacity: int = 0, env_prm=None, env_shared=None):
        st = np.zeros(1, np.int32)
        self._h = lib().wso_create(env.encode(), n_envs, n_agents, seed & (2**64 - 1), env_offset,
                                   n_envs_global, max_steps, p0, p1, _p(st))
        self.status = int(st[0])
        if not self._h:
            raise ValueError(f"wso_create failed with status {self.status}")
        self.env = env
        if env in _USER_ENVS:  # registered env: parameters / shared data, then the initial reset
            prm = np.ascontiguousarray(np.zeros(0) if env_prm is None else env_prm, dtype=np.float32).ravel()
            sh = np.ascontiguousarray(np.zeros(0) if env_shared is None else env_shared, dtype=np.float32).ravel()
            assert lib().wso_set_env_data(self._h, _p(prm), prm.size, _p(sh), sh.size) == OK
            assert self.reset() == OK
        if t_capacity:
            self.set_capacity(t_capacity)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            try:
                _lib.wso_destroy(h)
            except Exception:  # interpreter teardown
                pass
            self._h = None

    def info(self) -> dict:
        v = np.zeros(10, np.int64)
        lib().wso_info(self._h, _p(v))
        keys = ["obs_dim", "n_actions", "act_dim", "state_dim", "T_max", "T_cap", "cursor", "t", "A", "E"]
        return {k: int(x) for k, x in zip(keys, v)}

    def set_capacity(self, T: int) -> int:
        return lib().wso_set_capacity(self._h, T)

    def reset(self) -> int:
        return lib().wso_reset(self._h)

    def sample(self, probs: np.ndarray, row_stride: Optional[int] = None, override=None, ambiguous=None) -> int:
        probs = np.ascontiguousarray(probs, dtype=np.float32)
        if row_stride is None:
            row_stride = probs.shape[-1]
        return lib().wso_sample(self._h, _p(probs), row_stride, _p(override), _p(ambiguous))

    def step(self, actions: Optional[np.ndarray] = None) -> int:
        if actions is not None:
            inf = self.info()
            actions = np.ascontiguousarray(actions, dtype=np.int32 if inf["n_actions"] else np.float32)
        return lib().wso_step(self._h, _p(actions))

    def rollout(self, T: int, probs: np.ndarray, row_stride: Optional[int] = None, step_stride: int = 0,
                override: Optional[np.ndarray] = None, ambiguous: Optional[np.ndarray] = None,
                n_threads: int = 1) -> int:
        probs = np.ascontiguousarray(probs, dtype=np.float32)
        if row_stride is None:
            row_stride = probs.shape[-1]
        if override is not None:
            override = np.ascontiguousarray(override, dtype=np.int32)
        return lib().wso_rollout(self._h, T, _p(probs), row_stride, step_stride, _p(override),
                                 _p(ambiguous), n_threads)

    def rollout_policy(self, T: int, weights: np.ndarray, hidden: int, n_threads: int = 1) -> int:
        """NEXT-N1: roll-out driven by the MLP policy (wso.cpp policy_probs, DESIGN R29)."""
        weights = np.ascontiguousarray(weights, dtype=np.float32)
        return lib().wso_rollout_policy(self._h, T, _p(weights), hidden, n_threads)

    def rollout_policy_gauss(self, T: int, weights: np.ndarray, hidden: int, n_threads: int = 1) -> int:
        """NEXT-N1 continuous (R34): roll-out whose Gaussian head rows come from the policy."""
        w = np.ascontiguousarray(weights, dtype=np.float32)
        return lib().wso_rollout_policy_gauss(self._h, T, _p(w), hidden, n_threads)

    def synchronize(self) -> int:
        return lib().wso_synchronize(self._h)

    def array(self, name: str) -> np.ndarray:
        inf = self.info()
        E, A, T = inf["E"], inf["A"], inf["T_cap"]
        D, n, d, S = inf["obs_dim"], inf["n_actions"], inf["act_dim"], inf["state_dim"]
        spec = {
            "obs": ((T, E, A, D), np.float32),
            "act": ((T, E, A) if n else (T, E, A, d), np.int32 if n else np.float32),
            "logp": ((T, E, A), np.float32),
            "rew": ((T, E, A), np.float32),
            "done": ((T, E), np.uint8),
            "stats": ((T, 4), np.float64),
            "state": ((E, S), np.float32),
            "obs_live": ((E, A, D), np.float32),
            "ep_step": ((E,), np.int32),
            "reset_count": ((E,), np.uint32),
            "ep_ret": ((E, A), np.float32),
            "tag_x": ((E, A), np.int32),
            "tag_y": ((E, A), np.int32),
            "tag_active": ((E, A), np.uint8),
        }[name]
        shape, dt = spec
        ptr = lib().wso_get(self._h, name.encode())
        count = int(np.prod(shape))
        if count == 0 or not ptr:
            return np.zeros(shape, dt)
        buf = (C.c_char * (count * np.dtype(dt).itemsize)).from_address(ptr)
        arr = np.frombuffer(buf, dtype=dt).reshape(shape)
        # keep the batch alive as long as the view is (the view aliases oracle storage)
        return _View(arr, self)
