"""User environments for the NEXT-N4 composer (include/ws.h ws_register_env): C source that
a user of the engine writes.  They are INPUTS to the composer -- compiled by NVRTC into the
GPU roll-out template, and by g++ into the oracle -- like the probability tables of the other
workloads; the engine semantics around them (sampling, store, resets, statistics) are
implemented separately on each side.

* CARTPOLE_SRC   gym CartPole-v1 in gym's operation order (the built-in env, rewritten as a
                 user env: its trajectories must equal the built-in ones bit for bit).
* MOUNTAINCAR_SRC gym MountainCar-v0 (force 0.001, gravity 0.0025, |v| <= 0.07,
                 x in [-1.2, 0.6], inelastic left wall, goal x >= 0.5; start U(-0.6, -0.4)).
* POINTMASS_SRC  a damped point mass with per-replica parameters (prm[0] force gain, prm[1]
                 damping: parameter jitter) and a shared read-only reward map of 64 cells over
                 [-1, 1] (a grid in global memory, Fig 1).
"""

CARTPOLE = dict(state_dim=4, obs_dim=4, n_actions=2, n_reset_draws=4, max_steps=500, n_params=0)
CARTPOLE_SRC = r"""
WS_FN void ws_env_init(float *s, const float *u, const float *prm, const float *shared) {
  for (int i = 0; i < 4; ++i) s[i] = -0.05f + 0.1f * u[i];
}
WS_FN void ws_env_obs(const float *s, float *o, const float *prm, const float *shared) {
  for (int i = 0; i < 4; ++i) o[i] = s[i];
}
WS_FN int ws_env_step(float *s, int a, float *r, const float *prm, const float *shared) {
  const float total_mass = 0.1f + 1.0f, polemass_length = 0.1f * 0.5f;
  const float theta_threshold = (float)(12 * 2 * 3.14159265358979323846 / 360);
  const float x = s[0], x_dot = s[1], theta = s[2], theta_dot = s[3];
  const float force = (a == 1) ? 10.0f : -10.0f;
  const float costheta = ws_cos(theta), sintheta = ws_sin(theta);
  const float temp = (force + polemass_length * (theta_dot * theta_dot) * sintheta) / total_mass;
  const float thetaacc = (9.8f * sintheta - costheta * temp) /
                         (0.5f * ((float)(4.0 / 3.0) - 0.1f * (costheta * costheta) / total_mass));
  const float xacc = temp - polemass_length * thetaacc * costheta / total_mass;
  s[0] = x + 0.02f * x_dot;
  s[1] = x_dot + 0.02f * xacc;
  s[2] = theta + 0.02f * theta_dot;
  s[3] = theta_dot + 0.02f * thetaacc;
  *r = 1.0f;
  return (s[0] < -2.4f || s[0] > 2.4f || s[2] < -theta_threshold || s[2] > theta_threshold) ? 1 : 0;
}
"""

MOUNTAINCAR = dict(state_dim=2, obs_dim=2, n_actions=3, n_reset_draws=1, max_steps=200, n_params=0)
MOUNTAINCAR_SRC = r"""
WS_FN void ws_env_init(float *s, const float *u, const float *prm, const float *shared) {
  s[0] = -0.6f + 0.2f * u[0];
  s[1] = 0.0f;
}
WS_FN void ws_env_obs(const float *s, float *o, const float *prm, const float *shared) {
  o[0] = s[0];
  o[1] = s[1];
}
WS_FN int ws_env_step(float *s, int a, float *r, const float *prm, const float *shared) {
  float v = s[1] + (float)(a - 1) * 0.001f + ws_cos(3.0f * s[0]) * (-0.0025f);
  v = ws_clip(v, -0.07f, 0.07f);
  float x = ws_clip(s[0] + v, -1.2f, 0.6f);
  if (x == -1.2f && v < 0.0f) v = 0.0f;
  s[0] = x;
  s[1] = v;
  *r = -1.0f;
  return (x >= 0.5f && v >= 0.0f) ? 1 : 0;
}
"""

POINTMASS = dict(state_dim=2, obs_dim=3, n_actions=3, n_reset_draws=1, max_steps=100, n_params=2)
POINTMASS_SRC = r"""
WS_FN void ws_env_init(float *s, const float *u, const float *prm, const float *shared) {
  s[0] = -0.5f + u[0];
  s[1] = 0.0f;
}
WS_FN void ws_env_obs(const float *s, float *o, const float *prm, const float *shared) {
  o[0] = s[0];
  o[1] = s[1];
  o[2] = prm[0];
}
WS_FN int ws_env_step(float *s, int a, float *r, const float *prm, const float *shared) {
  const float f = (float)(a - 1) * prm[0];
  const float v = s[1] + 0.05f * (f - prm[1] * s[1]);
  const float x = s[0] + 0.05f * v;
  s[0] = x;
  s[1] = v;
  int cell = (int)ws_floor((x + 1.0f) * 32.0f);
  cell = cell < 0 ? 0 : (cell > 63 ? 63 : cell);
  *r = shared[cell];
  return (x < -1.0f || x > 1.0f) ? 1 : 0;
}
"""


def pointmass_data(E: int, seed: int = 0x24080930):
    """Per-replica parameters [E, 2] (force gain U(0.5, 2), damping U(0, 0.5): jitter) and the
    shared 64-cell reward map (N(0, 1)), float32."""
    import numpy as np
    rng = np.random.default_rng(seed + 7)
    prm = np.stack([rng.uniform(0.5, 2.0, E), rng.uniform(0.0, 0.5, E)], axis=1).astype(np.float32)
    grid = rng.standard_normal(64).astype(np.float32)
    return prm, grid


ENVS = {"u_cartpole": (CARTPOLE_SRC, CARTPOLE), "u_mountaincar": (MOUNTAINCAR_SRC, MOUNTAINCAR),
        "u_pointmass": (POINTMASS_SRC, POINTMASS)}
