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
* MBGRID_SRC     a discrete walker on a NOISY Mueller-Brown potential-energy surface (the
                 catalysis-style PES of the paper's reaction env, SURVEY 8(f) N4 "noisy PES"):
                 the MB energy (fp32 terms, exponentials via ws_exp) plus a shared 32 x 32 noise
                 grid over the box; per-replica step size prm[0]; start near minimum B, goal =
                 within 0.1 of minimum A; reward -0.01 dE - 0.1.
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
  float costheta, sintheta;
  ws_sincos(theta, &sintheta, &costheta);
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


MBGRID = dict(state_dim=2, obs_dim=3, n_actions=5, n_reset_draws=2, max_steps=200, n_params=1)
MBGRID_SRC = r"""
WS_FN float mb_energy(float x, float y, const float *shared) {
  const float A[4] = {-200.0f, -100.0f, -170.0f, 15.0f};
  const float a[4] = {-1.0f, -1.0f, -6.5f, 0.7f};
  const float b[4] = {0.0f, 0.0f, 11.0f, 0.6f};
  const float c[4] = {-10.0f, -10.0f, -6.5f, 0.7f};
  const float x0[4] = {1.0f, 0.0f, -0.5f, -1.0f};
  const float y0[4] = {0.0f, 0.5f, 1.5f, 1.0f};
  float E = 0.0f;
  for (int k = 0; k < 4; ++k) {
    const float dx = x - x0[k], dy = y - y0[k];
    E = E + A[k] * ws_exp(a[k] * dx * dx + b[k] * dx * dy + c[k] * dy * dy);
  }
  int ix = (int)ws_floor((x + 1.5f) * (32.0f / 2.7f));
  int iy = (int)ws_floor((y + 0.5f) * (32.0f / 2.5f));
  ix = ix < 0 ? 0 : (ix > 31 ? 31 : ix);
  iy = iy < 0 ? 0 : (iy > 31 ? 31 : iy);
  return E + shared[iy * 32 + ix];
}
WS_FN void ws_env_init(float *s, const float *u, const float *prm, const float *shared) {
  s[0] = 0.623f + 0.1f * (u[0] - 0.5f);
  s[1] = 0.028f + 0.1f * (u[1] - 0.5f);
}
WS_FN void ws_env_obs(const float *s, float *o, const float *prm, const float *shared) {
  o[0] = s[0];
  o[1] = s[1];
  o[2] = mb_energy(s[0], s[1], shared);
}
WS_FN int ws_env_step(float *s, int a, float *r, const float *prm, const float *shared) {
  const float e0 = mb_energy(s[0], s[1], shared);
  const float h = prm[0];
  float x = s[0] + (a == 1 ? h : (a == 2 ? -h : 0.0f));
  float y = s[1] + (a == 3 ? h : (a == 4 ? -h : 0.0f));
  x = ws_clip(x, -1.5f, 1.2f);
  y = ws_clip(y, -0.5f, 2.0f);
  s[0] = x;
  s[1] = y;
  *r = -0.01f * (mb_energy(x, y, shared) - e0) - 0.1f;
  return (ws_abs(x + 0.558f) < 0.1f && ws_abs(y - 1.442f) < 0.1f) ? 1 : 0;
}
"""


def mbgrid_data(E: int, seed: int = 0x24080930, noise: float = 5.0):
    """Per-replica step sizes U(0.02, 0.06) (jitter) and the shared 32 x 32 noise grid
    N(0, noise^2) (0 = the clean surface), float32."""
    import numpy as np
    rng = np.random.default_rng(seed + 11)
    prm = rng.uniform(0.02, 0.06, (E, 1)).astype(np.float32)
    grid = (noise * rng.standard_normal(32 * 32)).astype(np.float32)
    return prm, grid


PENDULUM = dict(state_dim=2, obs_dim=3, n_actions=0, n_reset_draws=2, max_steps=200, n_params=0, act_dim=1)
PENDULUM_SRC = r"""
/* gymnasium Pendulum-v1 in the built-in env's operation order: a continuous-action user env */
WS_FN void ws_env_init(float *s, const float *u, const float *prm, const float *shared) {
  s[0] = -(float)3.14159265358979323846 + (float)(2 * 3.14159265358979323846) * u[0];
  s[1] = -1.0f + 2.0f * u[1];
}
WS_FN void ws_env_obs(const float *s, float *o, const float *prm, const float *shared) {
  o[0] = ws_cos(s[0]);
  o[1] = ws_sin(s[0]);
  o[2] = s[1];
}
WS_FN int ws_env_step(float *s, const float *a, float *r, const float *prm, const float *shared) {
  const float pi = (float)3.14159265358979323846, two_pi = (float)(2 * 3.14159265358979323846);
  const float th = s[0], thdot = s[1];
  const float u = ws_clip(a[0], -2.0f, 2.0f);
  float an = ws_fmod(th + pi, two_pi);
  if (an != 0.0f && an < 0.0f) an = an + two_pi;
  an = an - pi;
  const float costs = an * an + 0.1f * (thdot * thdot) + 0.001f * (u * u);
  float newthdot = thdot + (3.0f * 10.0f / (2.0f * 1.0f) * ws_sin(th) + 3.0f / (1.0f * (1.0f * 1.0f)) * u) * 0.05f;
  newthdot = ws_clip(newthdot, -8.0f, 8.0f);
  s[0] = th + newthdot * 0.05f;
  s[1] = newthdot;
  *r = -costs;
  return 0;
}
"""

ENVS = {"u_cartpole": (CARTPOLE_SRC, CARTPOLE), "u_mountaincar": (MOUNTAINCAR_SRC, MOUNTAINCAR),
        "u_pointmass": (POINTMASS_SRC, POINTMASS), "u_mbgrid": (MBGRID_SRC, MBGRID),
        "u_pendulum": (PENDULUM_SRC, PENDULUM)}
