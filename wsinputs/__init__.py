"""Seeded synthetic inputs shared by the oracle-side tests and the product-side tests and
bench (the one module both sides may use).  It holds NONE of the method's arithmetic:
no Philox, no sampling, no dynamics -- only the workload shapes of BASELINE.json's
configs and numpy-generated policy inputs.

Random numbers the METHOD draws (actions, resets, Gaussian noise) come from the
counter-based Philox streams each side implements on its own (reading Q15); the numbers
generated here are only the *given* inputs: probabilities, Gaussian head parameters and
fixed-action tables.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED = 0x24080930  # one seed for every config


@dataclass(frozen=True)
class Workload:
    name: str
    env: str
    n_envs: int          # global env count (E_g)
    n_agents: int
    T: int
    n_actions: int       # 0 for continuous
    act_dim: int
    params: dict = field(default_factory=dict)   # env params (tag grid/taggers, surface dim)
    note: str = ""


# BASELINE.json configs (BJ:7-11) made concrete
CONFIGS = {
    "C1": Workload("C1", "cartpole", 64, 1, 500, 2, 1, note="CartPole-v1 64 envs x 500 steps (BJ:7)"),
    "C2": Workload("C2", "cartpole", 10000, 1, 1000, 2, 1, note="CartPole-v1 10K envs x 1000 steps (BJ:8)"),
    "C3a": Workload("C3a", "acrobot", 100000, 1, 500, 3, 1, note="Acrobot-v1 100K envs x 500 (BJ:9)"),
    "C3b": Workload("C3b", "pendulum", 100000, 1, 200, 0, 1, note="Pendulum-v1 100K envs x 200 (BJ:9)"),
    "C4": Workload("C4", "tag", 1000, 100, 200, 5, 1, {"grid": 20, "taggers": 10},
                   note="tag 1K envs x 100 agents x 200 (BJ:10)"),
    "C5": Workload("C5", "surface", 2000, 1, 200, 0, 20, {"dim": 20},
                   note="surface-20 2K envs x 200 (BJ:11)"),
    "D0": Workload("D0", "dummy", 1000000, 1, 100, 2, 1, note="store-write calibration"),
    # saturation points of SURVEY 8(d).1's sweep (where the >= 60 % roofline target is assessed:
    # enough replicas per GPU to fill every scheduler; same per-replica work as C2 / C3a)
    "C2S": Workload("C2S", "cartpole", 640000, 1, 1000, 2, 1,
                    note="CartPole-v1 640K envs x 1000 steps (saturation point, SURVEY 8(d).1 sweep)"),
    "C3S": Workload("C3S", "acrobot", 400000, 1, 500, 3, 1,
                    note="Acrobot-v1 400K envs x 500 steps (saturation point, SURVEY 8(d).1 sweep)"),
    # NEXT-N1: C2's shape with the actions drawn from an in-kernel MLP policy
    "C2P": Workload("C2P", "cartpole", 10000, 1, 1000, 2, 1, {"policy_hidden": 64},
                    note="CartPole-v1 10K envs x 1000 steps, in-kernel MLP policy 4-64-2 (NEXT-N1)"),
    # NEXT-N2: C2's roll-out followed by GAE over the store it wrote
    "C2G": Workload("C2G", "cartpole", 10000, 1, 1000, 2, 1, {"gae": (0.99, 0.95)},
                    note="CartPole-v1 10K envs x 1000 steps + GAE(0.99, 0.95) over the store (NEXT-N2)"),
    # NEXT-N2: a full A2C iteration -- C2's roll-out with in-kernel inference of
    # a 4-64-2 actor-critic, then critic values, GAE over the store, gradient, clip + Adam
    "C2T": Workload("C2T", "cartpole", 10000, 1, 1000, 2, 1, {"policy_hidden": 64, "a2c": True},
                    note="CartPole-v1 10K envs x 1000 steps + A2C update of a 4-64-2 actor-critic (NEXT-N2)"),
    "C2O": Workload("C2O", "cartpole", 10000, 1, 1000, 2, 1, {"policy_hidden": 64, "a2c": True, "ppo": (4, 4)},
                    note="CartPole-v1 10K envs x 1000 steps + PPO update (4 epochs x 4 minibatches) of a 4-64-2 "
                         "actor-critic (NEXT-N2)"),
    # NEXT-N2 continuous (R34 / R35): C3b's Pendulum shape with a Gaussian actor-critic iteration
    "C3T": Workload("C3T", "pendulum", 100000, 1, 200, 0, 1, {"policy_hidden": 64, "a2c": True},
                    note="Pendulum-v1 100K envs x 200 steps + A2C update of a 3-64-1 Gaussian actor-critic (NEXT-N2)"),
    # NEXT-N2 multi-agent (R36): C4's tag shape with every agent's policy in the kernel + A2C
    "C4T": Workload("C4T", "tag", 1000, 100, 200, 5, 1, {"grid": 20, "taggers": 10, "policy_hidden": 64, "a2c": True},
                    note="tag 1K envs x 100 agents x 200 + multi-agent A2C update of a 4-64-5 actor-critic (NEXT-N2)"),
    # NEXT-N3: C2 through the copy-based baseline pipeline (per-step H2D of the
    # probabilities and D2H of the slot, synchronised every step) -- the "data transfer"
    # cost WarpSci removes
    "C2X": Workload("C2X", "cartpole", 10000, 1, 1000, 2, 1, {"staged": True},
                    note="CartPole-v1 10K envs x 1000 steps through the copy-based baseline pipeline (NEXT-N3)"),
    # NEXT-N4: C2 with CartPole supplied as user C source through the runtime
    # env composer (NVRTC-compiled generic template) instead of the hand-written kernel
    "C2U": Workload("C2U", "u_cartpole", 10000, 1, 1000, 2, 1, {"user": "u_cartpole"},
                    note="CartPole-v1 10K envs x 1000 steps, env registered as C source (NVRTC composer, NEXT-N4)"),
    "C4G": Workload("C4G", "tag", 1000, 100, 200, 5, 1, {"grid": 20, "taggers": 10, "gae": (0.99, 0.95)},
                    note="tag 1K envs x 100 agents x 200 + GAE(0.99, 0.95) over the store (NEXT-N2)"),
}


def uniform_probs(E: int, A: int, n: int) -> np.ndarray:
    """Reading Q25: uniform 1/n probabilities, [E, A, n] float32."""
    return np.full((E, A, n), 1.0 / n, dtype=np.float32)


def random_probs(E: int, A: int, n: int, seed: int = SEED, zero_frac: float = 0.0,
                 T: int | None = None) -> np.ndarray:
    """Random unnormalised probability rows ([T,]E, A, n) with a fraction of exact zeros
    (at least one nonzero per row) -- exercises Q13 (rows need not sum to 1, zeros are
    never drawn)."""
    rng = np.random.default_rng(seed)
    shape = (E, A, n) if T is None else (T, E, A, n)
    p = rng.gamma(0.7, 1.0, size=shape).astype(np.float32)
    if zero_frac > 0:
        z = rng.random(shape) < zero_frac
        p[z] = 0.0
        flat = p.reshape(-1, n)
        dead = flat.sum(axis=1) == 0
        flat[dead, rng.integers(0, n, dead.sum())] = 1.0
    return p


def gaussian_params(E: int, A: int, d: int, mean: float = 0.0, log_std: float = 0.0,
                    jitter: float = 0.0, seed: int = SEED) -> np.ndarray:
    """Continuous head input [E, A, 2d] = mean[d] | log_std[d] (reading Q25: Pendulum
    mean 0, log_std 0; surface mean 0, log_std ln 0.025)."""
    rng = np.random.default_rng(seed)
    p = np.empty((E, A, 2 * d), np.float32)
    p[..., :d] = mean + jitter * rng.standard_normal((E, A, d))
    p[..., d:] = log_std + jitter * rng.standard_normal((E, A, d))
    return p


def action_table(T: int, E: int, A: int, n: int, seed: int = SEED, p1: float | None = None) -> np.ndarray:
    """Fixed-action parity table [T, E, A] int32 (reading Q27)."""
    rng = np.random.default_rng(seed)
    if p1 is not None and n == 2:
        return (rng.random((T, E, A)) < p1).astype(np.int32)
    return rng.integers(0, n, size=(T, E, A), dtype=np.int32)


def continuous_action_table(T: int, E: int, A: int, d: int, scale: float, seed: int = SEED) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return (scale * rng.standard_normal((T, E, A, d))).astype(np.float32)


def workload_policy(w: Workload):
    """(hidden, packed weights) of a policy-driven workload, else None."""
    H = w.params.get("policy_hidden")
    if not H:
        return None
    D = {"cartpole": 4, "acrobot": 6, "dummy": 4, "pendulum": 3, "tag": 4}[w.env]
    if w.params.get("a2c") and w.n_actions == 0:  # Gaussian actor-critic (R35)
        return H, a2c_params_gauss(D, H, w.act_dim, seed=SEED)
    if w.params.get("a2c"):  # actor-critic: the policy prefix followed by the value head
        return H, a2c_params(D, H, w.n_actions, seed=SEED, scale=1.0)
    return H, policy_weights(D, H, w.n_actions, seed=SEED, scale=2.0)


def workload_probs(w: Workload) -> np.ndarray:
    """The bench / parity input of a config: per-env given probabilities, step stride 0."""
    if w.n_actions:
        return uniform_probs(w.n_envs, w.n_agents, w.n_actions)
    if w.env == "surface":
        return gaussian_params(w.n_envs, w.n_agents, w.act_dim, 0.0, float(np.log(0.025)))
    return gaussian_params(w.n_envs, w.n_agents, w.act_dim, 0.0, 0.0)


def gae_inputs(T: int, E: int, A: int, seed: int = SEED, with_trunc: bool = False):
    """NEXT-N2 given inputs of GAE (reading R30): values [T, E, A], bootstrap [E, A] and,
    optionally, terminal values v_trunc [T, E, A] (float32) -- value estimates of the scale
    of CartPole returns (mean 10, std 5; SPEC S:433 defaults gamma 0.99 give returns <= 100)."""
    rng = np.random.default_rng(seed)
    values = (10.0 + 5.0 * rng.standard_normal((T, E, A))).astype(np.float32)
    boot = (10.0 + 5.0 * rng.standard_normal((E, A))).astype(np.float32)
    vtr = (10.0 + 5.0 * rng.standard_normal((T, E, A))).astype(np.float32) if with_trunc else None
    return values, boot, vtr


def policy_weights(D: int, H: int, N: int, seed: int = SEED, scale: float = 1.0) -> np.ndarray:
    """NEXT-N1 MLP policy weights, packed W1 [D][H] | b1 [H] | W2 [H][N] | b2 [N] (float32,
    reading R29): Glorot-like normal draws times `scale`."""
    rng = np.random.default_rng(seed)
    W1 = rng.standard_normal((D, H)) * (scale / np.sqrt(D))
    b1 = rng.standard_normal(H) * 0.1 * scale
    W2 = rng.standard_normal((H, N)) * (scale / np.sqrt(H))
    b2 = rng.standard_normal(N) * 0.1 * scale
    return np.concatenate([W1.ravel(), b1, W2.ravel(), b2]).astype(np.float32)


def a2c_params(D: int, H: int, N: int, seed: int = SEED, scale: float = 1.0) -> np.ndarray:
    """NEXT-N2 actor-critic parameters (reading R31): the R29 policy weights followed by a
    value head wv [H] | bv [1] (float32)."""
    rng = np.random.default_rng(seed + 1)
    head = np.concatenate([rng.standard_normal(H) * (scale / np.sqrt(H)), [10.0 * scale]])
    return np.concatenate([policy_weights(D, H, N, seed, scale), head]).astype(np.float32)


def a2c_params_gauss(D: int, H: int, d: int, seed: int = SEED, log_std: float = -0.5) -> np.ndarray:
    """NEXT-N2 continuous actor-critic parameters (R35): W1 | b1 | W2 [H][d] | b2 [d] |
    log_std [d] | wv [H] | bv, float32 (Glorot-like normal draws)."""
    rng = np.random.default_rng(seed + 3)
    parts = [rng.standard_normal(D * H) / np.sqrt(D), rng.standard_normal(H) * 0.1,
             rng.standard_normal(H * d) / np.sqrt(H), np.zeros(d), np.full(d, log_std),
             rng.standard_normal(H) / np.sqrt(H), [-100.0]]
    return np.concatenate(parts).astype(np.float32)


def a2c_batch(rows: int, D: int, N: int, seed: int = SEED, invalid_frac: float = 0.0):
    """NEXT-N2 given inputs of one update: obs [rows, D] (CartPole-scale N(0, 0.5^2)),
    actions [rows] int32 (a fraction set to -1, the R13 invalid-row marker), advantages
    (N(0.5, 2^2)) and returns (N(10, 5^2)) float32."""
    rng = np.random.default_rng(seed + 2)
    obs = (0.5 * rng.standard_normal((rows, D))).astype(np.float32)
    act = rng.integers(0, N, rows).astype(np.int32)
    if invalid_frac > 0:
        act[rng.random(rows) < invalid_frac] = -1
    adv = (0.5 + 2.0 * rng.standard_normal(rows)).astype(np.float32)
    ret = (10.0 + 5.0 * rng.standard_normal(rows)).astype(np.float32)
    return obs, act, adv, ret
