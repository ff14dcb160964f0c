/*
 * oracle/wso.cpp -- the CPU ORACLE of the WarpSci roll-out hot path.
 *
 *   *** TEST INFRASTRUCTURE ONLY. ***
 *   Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and its
 *   `--impl reference` arm) may load this library.  The product path
 *   (paper_2408_00930_b200/) never imports, links or executes anything under oracle/.
 *   This file shares no code, header, table or constant generator with the CUDA path.
 *
 * What it is: a plain, slow, scalar C++17 simulation of the batched roll-out step the
 * paper describes -- "each thread is responsible for operating an agent that samples
 * actions and computes rewards", reset on device, in-place
 * roll-out store -- with the environments and sampler that SPEC.md
 * defines and the readings Q1..Q27 of SURVEY.md section 8(c),
 * restated in DESIGN.md section 3.  One environment at a time, one agent at a time, in
 * the order the paper / SPEC state: for t: sample, log, step_all,
 * auto_reset.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * BJ:5 = BASELINE.json north_star; Qk = SURVEY.md 8(c) reading k.
 *
 * Arithmetic (readings R2-R4): environment state is fp32 (BJ:5
 * "fp32 states"); every transcendental is evaluated in fp64 and rounded once to fp32
 * (Tr<float>); no FMA contraction (built with -ffp-contract=off); division and sqrt are
 * IEEE.  Each environment step is a template on the real type R so the same text also
 * runs in fp64 ("gym mode") for the closed-form and physics pins in tests/.
 *
 * NEXT-N2 (first stage): generalised advantage estimation over the store (SPEC compute_gae
 * S:389-397, reading R30), the step that consumes the roll-out store in place for training.
 *
 * Pins: every exported function is pinned by tests/test_oracle_*.py against values the
 * mathematics fixes (Random123 known answers, exact rational steps, Lagrangian
 * mechanics, published Mueller-Brown stationary points, exhaustive multinomial counts,
 * SPEC rule examples).  Nothing here is "parity unpinned".
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <map>
#include <limits>
#include <string>
#include <thread>
#include <vector>

namespace {

/* ------------------------------------------------------------------------------------
 * A1. Philox4x32-10 counter-based RNG (S:120-124 RngStream; BJ:5 "driven by a
 * counter-based Philox RNG").  Algorithm of Salmon et al., SC'11 ("Random123"): ten
 * rounds of  (hi0,lo0)=mulhilo(0xD2511F53,c0), (hi1,lo1)=mulhilo(0xCD9E8D57,c2),
 * c=(hi1^c1^k0, lo1, hi0^c3^k1, lo0), key bumped by the Weyl constants between rounds.
 * ---------------------------------------------------------------------------------- */
void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint32_t k[2] = {key_in[0], key_in[1]};
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k[0] += 0x9E3779B9u;
      k[1] += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
  }
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* Stream layout, reading Q15: draw j of stream (env_global, agent, purpose) is word
 * (j & 3) of Philox(ctr = (j >> 2, env_global, agent, purpose), key = (seed_lo, seed_hi)). */
enum Purpose : uint32_t { ACTION = 1, RESET = 2, GAUSS = 3 };

uint32_t draw(uint64_t seed, uint64_t env_global, uint32_t agent, uint32_t purpose, uint64_t j) {
  uint32_t ctr[4] = {(uint32_t)(j >> 2), (uint32_t)env_global, agent, purpose};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t w[4];
  philox4x32_10(ctr, key, w);
  return w[j & 3];
}

/* Reading Q14: u = (w >> 8) * 2^-24, exact in fp32, in [0, 1). */
float u01(uint32_t w) { return (float)(w >> 8) * (1.0f / 16777216.0f); }

/* Transcendental contract (reading Q3 / DESIGN R3): fp64 evaluation, one rounding. */
template <class R> struct Tr;
template <> struct Tr<float> {
  static float sin(float x) { return (float)std::sin((double)x); }
  static float cos(float x) { return (float)std::cos((double)x); }
};
template <> struct Tr<double> {
  static double sin(double x) { return std::sin(x); }
  static double cos(double x) { return std::cos(x); }
};

constexpr double kPi = 3.14159265358979323846;

/* ------------------------------------------------------------------------------------
 * A3/A4. CartPole-v1 (constants S:229).  The standard gym
 * cart-pole equations with explicit Euler, written in gym's operation order.
 * ---------------------------------------------------------------------------------- */
template <class R> struct CartPole {
  static constexpr R gravity = R(9.8), masscart = R(1.0), masspole = R(0.1);
  static constexpr R total_mass = masspole + masscart;
  static constexpr R length = R(0.5);  // half the pole length ("half-length 0.5")
  static constexpr R polemass_length = masspole * length;
  static constexpr R force_mag = R(10.0), tau = R(0.02);
  static constexpr R theta_threshold = R(12 * 2 * kPi / 360);  // S:211 "12 pi/180"
  static constexpr R x_threshold = R(2.4);

  /* returns 1 on InvalidAction, else 0; reward 1.0 every step */
  static int step(const R s[4], int a, R out[4], R* reward, int* terminated) {
    if (a != 0 && a != 1) return 1;
    R x = s[0], x_dot = s[1], theta = s[2], theta_dot = s[3];
    R force = (a == 1) ? force_mag : -force_mag;
    R costheta = Tr<R>::cos(theta);
    R sintheta = Tr<R>::sin(theta);
    R temp = (force + polemass_length * (theta_dot * theta_dot) * sintheta) / total_mass;
    R thetaacc = (gravity * sintheta - costheta * temp) /
                 (length * (R(4.0 / 3.0) - masspole * (costheta * costheta) / total_mass));
    R xacc = temp - polemass_length * thetaacc * costheta / total_mass;
    out[0] = x + tau * x_dot;
    out[1] = x_dot + tau * xacc;
    out[2] = theta + tau * theta_dot;
    out[3] = theta_dot + tau * thetaacc;
    *terminated = (out[0] < -x_threshold || out[0] > x_threshold ||
                   out[2] < -theta_threshold || out[2] > theta_threshold);
    *reward = R(1.0);
    return 0;
  }
};

/* ------------------------------------------------------------------------------------
 * Acrobot-v1: the "book" two-link dynamics (reading Q9),
 * classical RK4 over dt = 0.2, torque in {-1, 0, +1}; cos(x - pi/2) written as
 * sin(x) (reading Q7); wrap / bound as gym (reading Q8).
 * ---------------------------------------------------------------------------------- */
template <class R> struct Acrobot {
  static constexpr R m1 = R(1), m2 = R(1), l1 = R(1), lc1 = R(0.5), lc2 = R(0.5);
  static constexpr R I1 = R(1), I2 = R(1), g = R(9.8), dt = R(0.2);
  static constexpr R pi = R(kPi);
  static constexpr R max_vel_1 = R(4 * kPi), max_vel_2 = R(9 * kPi);

  static void dsdt(const R s[4], R torque, R d[4]) {
    R theta1 = s[0], theta2 = s[1], dtheta1 = s[2], dtheta2 = s[3];
    R c2 = Tr<R>::cos(theta2);
    R s2 = Tr<R>::sin(theta2);
    R d1 = m1 * (lc1 * lc1) + m2 * (l1 * l1 + lc2 * lc2 + R(2) * l1 * lc2 * c2) + I1 + I2;
    R d2 = m2 * (lc2 * lc2 + l1 * lc2 * c2) + I2;
    R phi2 = m2 * lc2 * g * Tr<R>::sin(theta1 + theta2);
    R phi1 = -m2 * l1 * lc2 * (dtheta2 * dtheta2) * s2 -
             R(2) * m2 * l1 * lc2 * dtheta2 * dtheta1 * s2 +
             (m1 * lc1 + m2 * l1) * g * Tr<R>::sin(theta1) + phi2;
    R ddtheta2 = (torque + d2 / d1 * phi1 - m2 * l1 * lc2 * (dtheta1 * dtheta1) * s2 - phi2) /
                 (m2 * (lc2 * lc2) + I2 - (d2 * d2) / d1);
    R ddtheta1 = -(d2 * ddtheta2 + phi1) / d1;
    d[0] = dtheta1; d[1] = dtheta2; d[2] = ddtheta1; d[3] = ddtheta2;
  }
  static R wrap(R x) {  // gym wrap(x, -pi, pi)
    R diff = pi - (-pi);
    while (x > pi) x = x - diff;
    while (x < -pi) x = x + diff;
    return x;
  }
  static R bound(R x, R lo, R hi) { return std::min(std::max(x, lo), hi); }
  static int terminal(const R s[4]) {
    return (-Tr<R>::cos(s[0]) - Tr<R>::cos(s[1] + s[0])) > R(1.0);
  }
  static int step(const R s[4], int a, R out[4], R* reward, int* terminated) {
    if (a < 0 || a > 2) return 1;
    const R torque = (a == 0) ? R(-1) : (a == 1 ? R(0) : R(1));
    R k1[4], k2[4], k3[4], k4[4], y[4];
    const R dt2 = dt / R(2);
    dsdt(s, torque, k1);
    for (int i = 0; i < 4; ++i) y[i] = s[i] + dt2 * k1[i];
    dsdt(y, torque, k2);
    for (int i = 0; i < 4; ++i) y[i] = s[i] + dt2 * k2[i];
    dsdt(y, torque, k3);
    for (int i = 0; i < 4; ++i) y[i] = s[i] + dt * k3[i];
    dsdt(y, torque, k4);
    const R dt6 = dt / R(6);
    for (int i = 0; i < 4; ++i)
      out[i] = s[i] + dt6 * (k1[i] + R(2) * k2[i] + R(2) * k3[i] + k4[i]);
    out[0] = wrap(out[0]);
    out[1] = wrap(out[1]);
    out[2] = bound(out[2], -max_vel_1, max_vel_1);
    out[3] = bound(out[3], -max_vel_2, max_vel_2);
    *terminated = terminal(out);
    *reward = *terminated ? R(0) : R(-1);
    return 0;
  }
};

/* ------------------------------------------------------------------------------------
 * Pendulum-v1 (BJ:9 only; reading Q24, gymnasium Pendulum-v1): g = 10, m = l = 1,
 * dt = 0.05, |u| <= 2, |thdot| <= 8; cost from the pre-step state and clipped u.
 * ---------------------------------------------------------------------------------- */
template <class R> struct Pendulum {
  static constexpr R g = R(10), m = R(1), l = R(1), dt = R(0.05);
  static constexpr R max_torque = R(2), max_speed = R(8);
  static constexpr R pi = R(kPi), two_pi = R(2 * kPi);
  static R angle_normalize(R x) {  // ((x + pi) % (2 pi)) - pi, Python floored modulo
    R r = std::fmod(x + pi, two_pi);
    if (r != R(0) && r < R(0)) r = r + two_pi;
    return r - pi;
  }
  static int step(const R s[2], R u_in, R out[2], R* reward) {
    if (!std::isfinite(u_in)) return 1;
    R th = s[0], thdot = s[1];
    R u = std::min(std::max(u_in, -max_torque), max_torque);
    R an = angle_normalize(th);
    R costs = an * an + R(0.1) * (thdot * thdot) + R(0.001) * (u * u);
    R newthdot = thdot + (R(3) * g / (R(2) * l) * Tr<R>::sin(th) + R(3) / (m * (l * l)) * u) * dt;
    newthdot = std::min(std::max(newthdot, -max_speed), max_speed);
    R newth = th + newthdot * dt;
    out[0] = newth; out[1] = newthdot;
    *reward = -costs;
    return 0;
  }
};

/* ------------------------------------------------------------------------------------
 * Mueller-Brown surface (standard published constants S:257) and the D-dim
 * extension "surface-D" (reading Q23): E_D(q) = MB(q0,q1) + 1/2 kappa sum_{i>=2} q_i^2.
 * ---------------------------------------------------------------------------------- */
constexpr double MB_A[4] = {-200, -100, -170, 15};
constexpr double MB_a[4] = {-1, -1, -6.5, 0.7};
constexpr double MB_b[4] = {0, 0, 11, 0.6};
constexpr double MB_c[4] = {-10, -10, -6.5, 0.7};
constexpr double MB_x0[4] = {1, 0, -0.5, -1};
constexpr double MB_y0[4] = {0, 0.5, 1.5, 1};

/* Pairwise (binary-tree) sum of w[0..n), n a power of two: sum(w, n) = sum(w, n/2) +
 * sum(w + n/2, n/2) (reading R23: the fixed summation order of the energy's two sums). */
double pairwise_sum(const double* w, int n) {
  if (n == 1) return w[0];
  return pairwise_sum(w, n / 2) + pairwise_sum(w + n / 2, n / 2);
}

/* Mueller-Brown potential: sum of the four terms t_k = A_k exp(a_k dx^2 + b_k dx dy +
 * c_k dy^2), added as the pairwise tree (t0 + t1) + (t2 + t3) (R23).  The gradient (S:262,
 * used by the pins only) is summed left to right. */
double mb_energy(double x, double y, double* gx, double* gy) {
  double t[4], Gx = 0, Gy = 0;
  for (int k = 0; k < 4; ++k) {
    double dx = x - MB_x0[k], dy = y - MB_y0[k];
    double ex = MB_A[k] * std::exp(MB_a[k] * dx * dx + MB_b[k] * dx * dy + MB_c[k] * dy * dy);
    t[k] = ex;
    Gx += ex * (2 * MB_a[k] * dx + MB_b[k] * dy);
    Gy += ex * (MB_b[k] * dx + 2 * MB_c[k] * dy);
  }
  if (gx) *gx = Gx;
  if (gy) *gy = Gy;
  return pairwise_sum(t, 4);
}

struct SurfaceParams {
  static constexpr double kappa = 100.0;
  static constexpr float delta = 0.05f, w_E = 0.01f, c_step = 0.1f, bonus = 10.0f;
  static constexpr double r_goal = 0.1;
  static constexpr double start0 = 0.623499, start1 = 0.028038;   // minimum B (Q23)
  static constexpr double goal0 = -0.558224, goal1 = 1.441726;    // minimum A (Q23)
  static float lo(int i) { return i == 0 ? -1.8f : (i == 1 ? -0.5f : -1.0f); }
  static float hi(int i) { return i == 0 ? 1.2f : (i == 1 ? 2.2f : 1.0f); }
  static double goal(int i) { return i == 0 ? goal0 : (i == 1 ? goal1 : 0.0); }
  static float start(int i) { return i == 0 ? (float)start0 : (i == 1 ? (float)start1 : 0.0f); }
};

/* spring sum of q_i^2, i = 2..D-1, as the pairwise tree over P = the smallest power of two
 * >= max(D, 4) leaves w_i = q_i^2 (2 <= i < D), +0 otherwise (R23) */
double surface_spring(const float* q, int D) {
  int P = 4;
  while (P < D) P *= 2;
  std::vector<double> w(P, 0.0);
  for (int i = 2; i < D; ++i) w[i] = (double)q[i] * (double)q[i];
  return pairwise_sum(w.data(), P);
}

/* energy in fp64 from the fp32 state, rounded once (DESIGN R3, R23) */
float surface_energy(const float* q, int D) {
  double E = mb_energy((double)q[0], (double)q[1], nullptr, nullptr);
  return (float)(E + 0.5 * SurfaceParams::kappa * surface_spring(q, D));
}

int surface_step(const float* q, const float* a, int D, float* out, float* reward, int* terminated) {
  for (int i = 0; i < D; ++i)
    if (!std::isfinite(a[i])) return 1;  // S:267 InvalidAction (non-finite)
  for (int i = 0; i < D; ++i) {
    float ai = std::min(std::max(a[i], -SurfaceParams::delta), SurfaceParams::delta);
    float qi = q[i] + ai;
    out[i] = std::min(std::max(qi, SurfaceParams::lo(i)), SurfaceParams::hi(i));
  }
  float E0 = surface_energy(q, D), E1 = surface_energy(out, D);
  double d2 = 0;
  for (int i = 0; i < D; ++i) {
    double di = (double)out[i] - SurfaceParams::goal(i);
    d2 += di * di;
  }
  *terminated = d2 < SurfaceParams::r_goal * SurfaceParams::r_goal;
  float r = -(SurfaceParams::w_E * (E1 - E0)) - SurfaceParams::c_step;
  if (*terminated) r = r + SurfaceParams::bonus;
  *reward = r;
  return 0;
}

/* ------------------------------------------------------------------------------------
 * Tag gridworld (parameters reading Q22).
 * ---------------------------------------------------------------------------------- */
int tag_step(int A, int G, int n_taggers, int32_t* x, int32_t* y, uint8_t* active,
             const int32_t* act, float* rew, int* terminated) {
  for (int a = 0; a < A; ++a)
    if (act[a] < 0 || act[a] > 4) return 1;
  /* simultaneous moves, clipped to the grid; tagged runners frozen */
  for (int a = 0; a < A; ++a) {
    bool tagger = a < n_taggers;
    if (!tagger && !active[a]) continue;
    int nx = x[a], ny = y[a];
    switch (act[a]) {
      case 1: ny = y[a] + 1; break;  // N
      case 2: ny = y[a] - 1; break;  // S
      case 3: nx = x[a] + 1; break;  // E
      case 4: nx = x[a] - 1; break;  // W
      default: break;                // stay
    }
    x[a] = std::min(std::max(nx, 0), G - 1);
    y[a] = std::min(std::max(ny, 0), G - 1);
  }
  std::vector<int> taggers_on(G * G, 0), tagged_on(G * G, 0);
  for (int a = 0; a < n_taggers && a < A; ++a) taggers_on[y[a] * G + x[a]] += 1;
  int runners = 0, still_active = 0;
  for (int a = n_taggers; a < A; ++a) {
    ++runners;
    rew[a] = 0.0f;
    if (!active[a]) continue;
    int cell = y[a] * G + x[a];
    if (taggers_on[cell] >= 1) {  // S:248 "a runner sharing a cell with >=1 tagger is tagged"
      rew[a] = -1.0f;
      active[a] = 0;
      tagged_on[cell] += 1;
    } else {
      rew[a] = 0.01f;  // S:248 "+0.01 per surviving step"
      ++still_active;
    }
  }
  for (int a = 0; a < n_taggers && a < A; ++a) {  // "+1 split equally among co-located taggers"
    int cell = y[a] * G + x[a];
    rew[a] = (float)tagged_on[cell] / (float)taggers_on[cell];
  }
  *terminated = (runners > 0 && still_active == 0);
  return 0;
}

/* ------------------------------------------------------------------------------------
 * A2. Sampling from given probabilities ("inverse-CDF"; readings Q13, Q16).
 * The CDF is accumulated sequentially in fp64 in action-index order.
 * ---------------------------------------------------------------------------------- */
int sample_discrete(const float* p, int n, float u, int32_t* act, float* logp, int* ambiguous) {
  double S = 0;
  int last_nz = -1;
  for (int i = 0; i < n; ++i) {
    if (!(p[i] >= 0.0f) || !std::isfinite(p[i])) {  // negative or NaN or inf
      *act = -1; *logp = std::numeric_limits<float>::quiet_NaN(); *ambiguous = 0;
      return 1;
    }
    S += (double)p[i];
    if (p[i] > 0.0f) last_nz = i;
  }
  if (!(S > 0.0) || !std::isfinite(S)) {
    *act = -1; *logp = std::numeric_limits<float>::quiet_NaN(); *ambiguous = 0;
    return 1;
  }
  const double target = (double)u * S;
  int chosen = -1;
  double C = 0;
  int amb = 0;
  for (int i = 0; i < n; ++i) {
    C += (double)p[i];
    if (chosen < 0 && p[i] > 0.0f && target < C) chosen = i;
    if (i < last_nz && std::fabs(target - C) < 1e-6 * S) amb = 1;  // Q16 interior boundary
  }
  if (chosen < 0) chosen = last_nz;  // Q13 fallback
  *act = chosen;
  *logp = (float)(std::log((double)p[chosen]) - std::log(S));
  *ambiguous = amb;
  return 0;
}

/* Box-Muller on one word pair (reading Q14): u1 = ((wa >> 8) + 1) 2^-24 in (0, 1] (so the log is
 * finite), u2 = (wb >> 8) 2^-24 in [0, 1); z = sqrt(-2 ln u1) cos(2 pi u2) for the even draw of the
 * pair, sqrt(-2 ln u1) sin(2 pi u2) for the odd one; fp64, rounded once (reading Q3).
 * Pinned by SURVEY App. A.8's worked value (tests/golden/box_muller.txt). */
float box_muller(uint32_t wa, uint32_t wb, int odd) {
  double u1 = (double)((wa >> 8) + 1) * (1.0 / 16777216.0);  // (0, 1]
  double u2 = (double)(wb >> 8) * (1.0 / 16777216.0);        // [0, 1)
  double r = std::sqrt(-2.0 * std::log(u1));
  double ang = 2.0 * kPi * u2;
  return (float)(odd ? r * std::sin(ang) : r * std::cos(ang));
}

/* Gaussian draw k of agent a at step t (reading Q14/Q15): j = t*d + k, Box-Muller on the
 * word pair (2p, 2p+1), p = (j & 3) >> 1; even j -> cos branch, odd j -> sin branch. */
float gauss(uint64_t seed, uint64_t e_g, uint32_t agent, uint64_t t, int d, int k) {
  uint64_t j = t * (uint64_t)d + (uint64_t)k;
  uint32_t ctr[4] = {(uint32_t)(j >> 2), (uint32_t)e_g, agent, GAUSS};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t w[4];
  philox4x32_10(ctr, key, w);
  int p = (int)((j & 3) >> 1);
  return box_muller(w[2 * p], w[2 * p + 1], (int)(j & 1));
}

/* ------------------------------------------------------------------------------------
 * The batch: make_batch, step_all, auto_reset, run_rollout
 * (S:158), log_step -- with the time-major store of S:40-45.
 * ---------------------------------------------------------------------------------- */
enum Kind { K_CARTPOLE = 0, K_ACROBOT = 1, K_PENDULUM = 2, K_TAG = 3, K_SURFACE = 4, K_DUMMY = 5, K_USER = 6 };

/* NEXT-N4: an environment given as C source (the composer's input, include/ws.h contract),
 * compiled by g++ into a shared object and called through these pointers; the engine
 * semantics around it (sampling, store, truncation, reset draws, statistics) are the
 * oracle's own, exactly as for the built-in envs. */
struct UserEnv {
  int state_dim, obs_dim, n_actions, n_reset, max_steps, n_params;
  void (*init)(float*, const float*, const float*, const float*);
  void (*obs)(const float*, float*, const float*, const float*);
  int (*step)(float*, int, float*, const float*, const float*);
  int act_dim;  // 0: discrete; > 0: continuous actions (step_c)
  int (*step_c)(float*, const float*, float*, const float*, const float*);
};
std::map<std::string, UserEnv>& user_envs() {
  static std::map<std::string, UserEnv> m;
  return m;
}
enum Err { E_OK = 0, E_INVALID_ARGUMENT = 1, E_UNKNOWN_ENV = 2, E_INVALID_ACTION = 3,
           E_INVALID_PROBS = 4, E_OUT_OF_RANGE = 5, E_BAD_STATE = 6 };
const int ERRBIT_ACTION = 1, ERRBIT_PROBS = 2;

/* ---------------------------------------------------------------------------------------
 * NEXT-N1 ("action inference with deep policy models resident in global
 * memory", "roll-outs, action inference, reset and training"): a two-layer MLP policy
 * obs[D] -> ReLU(W1^T obs + b1)[H] -> logits W2^T h + b2 [N] -> softmax -> probabilities.
 * Reading R29 (DESIGN): fp32 with fused multiply-adds in a fixed order -- h_j = b1_j, then
 * h_j = fma(W1[k][j], obs_k, h_j) for k = 0..D-1, h_j = h_j > 0 ? h_j : 0; every output i
 * of the second layer (R29', DESIGN): the hidden units are split into four quarters
 * Q_q = [q H/4, (q+1) H/4), P_q = 0, then P_q = fma(W2[j][i], h_j, P_q) for j in Q_q ascending,
 * and l_i = b2_i + ((P_0 + P_1) + (P_2 + P_3)); m = max_i l_i (first wins); e_i = (float)
 * exp((double)(l_i - m)) (R3); S = e_0 + e_1 + ... in fp32; p_i = e_i / S.  Packed weights:
 * W1 [D][H] | b1 [H] | W2 [H][N] | b2 [N], row-major fp32.
 * ------------------------------------------------------------------------------------- */
/* R29' second-layer output: b + ((P_0 + P_1) + (P_2 + P_3)) over the four quarters of the
 * hidden units (W2 column i with row stride `stride`) */
static float quarter_dot(const float* W2col, int stride, const float* h, int H, float b) {
  float P[4];
  const int Hq = H / 4;
  for (int q = 0; q < 4; ++q) {
    float acc = 0.0f;
    for (int j = q * Hq; j < (q + 1) * Hq; ++j) acc = std::fma(W2col[(size_t)j * stride], h[j], acc);
    P[q] = acc;
  }
  return b + ((P[0] + P[1]) + (P[2] + P[3]));
}

static void policy_hidden(const float* w, int D, int H, const float* obs, float* h) {
  const float* W1 = w;
  const float* b1 = W1 + (size_t)D * H;
  for (int j = 0; j < H; ++j) {
    float acc = b1[j];
    for (int k = 0; k < D; ++k) acc = std::fma(W1[(size_t)k * H + j], obs[k], acc);
    h[j] = acc > 0.0f ? acc : 0.0f;
  }
}

static void policy_logits(const float* w, int D, int H, int N, const float* obs, float* l) {
  const float* W2 = w + (size_t)D * H + H;
  const float* b2 = W2 + (size_t)H * N;
  std::vector<float> h((size_t)H);
  policy_hidden(w, D, H, obs, h.data());
  for (int i = 0; i < N; ++i) l[i] = quarter_dot(W2 + i, N, h.data(), H, b2[i]);
}

static void policy_probs(const float* w, int D, int H, int N, const float* obs, float* p) {
  std::vector<float> l((size_t)N);
  policy_logits(w, D, H, N, obs, l.data());
  float m = l[0];
  for (int i = 1; i < N; ++i) m = l[i] > m ? l[i] : m;
  float S = 0.0f;
  for (int i = 0; i < N; ++i) {
    p[i] = (float)std::exp((double)(l[i] - m));
    S = S + p[i];
  }
  for (int i = 0; i < N; ++i) p[i] = p[i] / S;
}

struct Batch {
  Kind kind;
  const UserEnv* user = nullptr;       // K_USER
  std::vector<float> prm, shared;      // K_USER per-replica parameters [E, n_params] / shared data
  const float* prm_row(int64_t e) const { return user && user->n_params ? &prm[(size_t)e * user->n_params] : nullptr; }
  const float* shared_ptr() const { return shared.empty() ? nullptr : shared.data(); }
  int64_t E, E_global, offset;
  int A;
  uint64_t seed;
  int T_max;
  int tag_G = 20, tag_taggers = 1, D = 20;
  /* derived */
  int obs_dim, n_actions /* discrete n, 0 if continuous */, act_dim /* d if continuous */;
  int state_dim;  /* fp32 state words per env (tag uses the int arrays below) */
  int n_reset_draws; /* RESET stream draws per reset per agent */
  /* live state */
  std::vector<float> state;          // [E, state_dim]
  std::vector<int32_t> tx, ty;       // tag [E, A]
  std::vector<uint8_t> tactive;      // tag [E, A]
  std::vector<float> obs_live;       // [E, A, obs_dim]
  std::vector<int32_t> ep_step;      // [E]
  std::vector<uint32_t> reset_count; // [E]
  std::vector<float> ep_ret;         // [E, A]
  /* store (time-major) */
  int T_cap = 0;
  std::vector<float> obs;      // [T, E, A, obs_dim]
  std::vector<int32_t> act_i;  // [T, E, A]          (discrete)
  std::vector<float> act_f;    // [T, E, A, act_dim] (continuous)
  std::vector<float> logp;     // [T, E, A]
  std::vector<float> rew;      // [T, E, A]
  std::vector<uint8_t> done;   // [T, E]  bit0 terminated, bit1 truncated
  std::vector<double> stats;   // [T, 4]  n_done, sum_ret, sum_len, sum_rew
  int cursor = 0;
  uint64_t t = 0;
  int sampled_slot = -1;
  int err = 0;

  int64_t EA() const { return E * (int64_t)A; }

  void alloc_store(int T) {
    T_cap = T;
    obs.assign((size_t)T * EA() * obs_dim, 0.0f);
    if (n_actions) act_i.assign((size_t)T * EA(), 0); else act_f.assign((size_t)T * EA() * act_dim, 0.0f);
    logp.assign((size_t)T * EA(), 0.0f);
    rew.assign((size_t)T * EA(), 0.0f);
    done.assign((size_t)T * E, 0);
    stats.assign((size_t)T * 4, 0.0);
  }

  uint64_t eg(int64_t e) const { return (uint64_t)(offset + e); }

  /* init(e, r): reading Q11 distributions, draws j = r * n_s + i of the RESET stream */
  void init_env(int64_t e) {
    uint32_t r = reset_count[e];
    auto U = [&](uint32_t agent, int i) {
      return u01(draw(seed, eg(e), agent, RESET, (uint64_t)r * n_reset_draws + i));
    };
    float* s = &state[e * state_dim];
    switch (kind) {
      case K_CARTPOLE:
        for (int i = 0; i < 4; ++i) s[i] = -0.05f + 0.1f * U(0, i);
        break;
      case K_ACROBOT:
        for (int i = 0; i < 4; ++i) s[i] = -0.1f + 0.2f * U(0, i);
        break;
      case K_PENDULUM: {
        const float pi = (float)kPi;
        s[0] = -pi + (float)(2 * kPi) * U(0, 0);
        s[1] = -1.0f + 2.0f * U(0, 1);
        break;
      }
      case K_SURFACE:
        for (int i = 0; i < D; ++i) s[i] = SurfaceParams::start(i) + (-0.05f + 0.1f * U(0, i));
        break;
      case K_TAG:
        for (int a = 0; a < A; ++a) {
          for (int d = 0; d < 2; ++d) {
            uint32_t w = draw(seed, eg(e), (uint32_t)a, RESET, (uint64_t)r * 2 + d);
            int32_t c = (int32_t)(((uint64_t)w * (uint64_t)tag_G) >> 32);
            (d == 0 ? tx : ty)[e * A + a] = c;
          }
          tactive[e * A + a] = 1;
        }
        break;
      case K_DUMMY:
        break;
      case K_USER: {
        std::vector<float> u(std::max(1, user->n_reset));
        for (int i = 0; i < user->n_reset; ++i) u[i] = U(0, i);
        user->init(s, u.data(), prm_row(e), shared_ptr());
        break;
      }
    }
  }

  void write_obs_live(int64_t e) {
    float* o = &obs_live[e * A * obs_dim];
    const float* s = &state[e * state_dim];
    switch (kind) {
      case K_CARTPOLE:
        for (int i = 0; i < 4; ++i) o[i] = s[i];
        break;
      case K_ACROBOT:
        o[0] = Tr<float>::cos(s[0]); o[1] = Tr<float>::sin(s[0]);
        o[2] = Tr<float>::cos(s[1]); o[3] = Tr<float>::sin(s[1]);
        o[4] = s[2]; o[5] = s[3];
        break;
      case K_PENDULUM:
        o[0] = Tr<float>::cos(s[0]); o[1] = Tr<float>::sin(s[0]); o[2] = s[1];
        break;
      case K_SURFACE:
        for (int i = 0; i < D; ++i) o[i] = s[i];
        o[D] = surface_energy(s, D);
        break;
      case K_TAG:
        for (int a = 0; a < A; ++a) {
          float* oa = o + a * obs_dim;
          oa[0] = (float)tx[e * A + a] / (float)(tag_G - 1);
          oa[1] = (float)ty[e * A + a] / (float)(tag_G - 1);
          oa[2] = a < tag_taggers ? 1.0f : 0.0f;
          oa[3] = tactive[e * A + a] ? 1.0f : 0.0f;
        }
        break;
      case K_DUMMY:
        for (int i = 0; i < obs_dim; ++i) o[i] = 0.0f;
        break;
      case K_USER:
        user->obs(s, o, prm_row(e), shared_ptr());
        break;
    }
  }

  void reset_all() {  // S:131-139 make_batch: all replicas to initial states
    for (int64_t e = 0; e < E; ++e) {
      reset_count[e] = 0;
      init_env(e);
      ep_step[e] = 0;
      for (int a = 0; a < A; ++a) ep_ret[e * A + a] = 0.0f;
      write_obs_live(e);
    }
    t = 0; cursor = 0; sampled_slot = -1; err = 0;
    std::fill(stats.begin(), stats.end(), 0.0);
  }

  /* sample into slot c for envs [e0, e1) using probs rows (e*A + a)*row_stride */
  void sample_range(int c, uint64_t tt, const float* probs, int64_t row_stride,
                    const int32_t* override_act, uint8_t* ambiguous, int64_t e0, int64_t e1,
                    int* err_out) {
    for (int64_t e = e0; e < e1; ++e) {
      for (int a = 0; a < A; ++a) {
        int64_t ea = e * A + a;
        const float* row = probs + ea * row_stride;
        if (n_actions) {
          float u = u01(draw(seed, eg(e), (uint32_t)a, ACTION, tt));
          int32_t act; float lp; int amb;
          if (sample_discrete(row, n_actions, u, &act, &lp, &amb)) *err_out |= ERRBIT_PROBS;
          if (override_act && override_act[ea] >= 0) act = override_act[ea];  // Q16 adoption
          act_i[(size_t)c * EA() + ea] = act;
          logp[(size_t)c * EA() + ea] = (override_act && override_act[ea] >= 0)
              ? (float)(std::log((double)row[act]) - std::log(row_sum(row)))
              : lp;
          if (ambiguous) ambiguous[ea] = (uint8_t)amb;
        } else {
          /* Gaussian head ("mean + std * gaussian"), probs row = mean[d] | log_std[d] */
          const float* mean = row;
          const float* log_std = row + act_dim;
          bool ok = true;
          for (int k = 0; k < act_dim; ++k)
            if (!std::isfinite(mean[k]) || !std::isfinite(log_std[k])) ok = false;
          double lp = 0;
          for (int k = 0; k < act_dim; ++k) {
            float z = gauss(seed, eg(e), (uint32_t)a, tt, act_dim, k);
            float sd = (float)std::exp((double)log_std[k]);
            act_f[((size_t)c * EA() + ea) * act_dim + k] =
                ok ? mean[k] + sd * z : std::numeric_limits<float>::quiet_NaN();
            lp += -0.5 * (double)z * (double)z - (double)log_std[k] - 0.5 * std::log(2 * kPi);
          }
          logp[(size_t)c * EA() + ea] = ok ? (float)lp : std::numeric_limits<float>::quiet_NaN();
          if (!ok) *err_out |= ERRBIT_PROBS;
          if (ambiguous) ambiguous[ea] = 0;
        }
      }
    }
  }
  double row_sum(const float* row) const {
    double S = 0;
    for (int i = 0; i < n_actions; ++i) S += (double)row[i];
    return S;
  }

  /* step_all on envs [e0, e1) using the actions in slot c, writing the
   * per-step statistics contribution into st[4] */
  void step_range(int c, int64_t e0, int64_t e1, double st[4], int* err_out) {
    for (int64_t e = e0; e < e1; ++e) {
      const size_t base = (size_t)c * EA() + (size_t)e * A;
      /* log_step: pre-step observation (reading Q12) */
      for (int i = 0; i < A * obs_dim; ++i)
        obs[base * obs_dim + i] = obs_live[(size_t)e * A * obs_dim + i];
      float* s = &state[e * state_dim];
      std::vector<float> r(A, 0.0f);
      int term = 0, bad = 0;
      switch (kind) {
        case K_CARTPOLE: {
          float out[4];
          bad = CartPole<float>::step(s, act_i[base], out, &r[0], &term);
          if (!bad) std::memcpy(s, out, sizeof out);
          break;
        }
        case K_ACROBOT: {
          float out[4];
          bad = Acrobot<float>::step(s, act_i[base], out, &r[0], &term);
          if (!bad) std::memcpy(s, out, sizeof out);
          break;
        }
        case K_PENDULUM: {
          float out[2];
          bad = Pendulum<float>::step(s, act_f[base], out, &r[0]);
          if (!bad) std::memcpy(s, out, sizeof out);
          break;
        }
        case K_SURFACE: {
          std::vector<float> out(D);
          bad = surface_step(s, &act_f[base * D], D, out.data(), &r[0], &term);
          if (!bad) std::memcpy(s, out.data(), sizeof(float) * D);
          break;
        }
        case K_TAG: {
          std::vector<int32_t> x(&tx[e * A], &tx[e * A] + A), y(&ty[e * A], &ty[e * A] + A);
          std::vector<uint8_t> act(&tactive[e * A], &tactive[e * A] + A);
          bad = tag_step(A, tag_G, tag_taggers, x.data(), y.data(), act.data(), &act_i[base], r.data(), &term);
          if (!bad) {
            std::copy(x.begin(), x.end(), &tx[e * A]);
            std::copy(y.begin(), y.end(), &ty[e * A]);
            std::copy(act.begin(), act.end(), &tactive[e * A]);
          }
          break;
        }
        case K_DUMMY: {
          int a = act_i[base];
          bad = (a < 0 || a > 1);
          r[0] = 1.0f;
          break;
        }
        case K_USER: {
          if (user->act_dim > 0) {  // continuous: a non-finite action is invalid (R19)
            const float* ac = &act_f[base * user->act_dim];
            bad = false;
            for (int k = 0; k < user->act_dim; ++k) bad = bad || !std::isfinite(ac[k]);
            if (!bad) term = user->step_c(s, ac, &r[0], prm_row(e), shared_ptr());
          } else {
            int a = act_i[base];
            bad = (a < 0 || a >= n_actions);
            if (!bad) term = user->step(s, a, &r[0], prm_row(e), shared_ptr());
          }
          break;
        }
      }
      if (bad) {  // reading Q19: sticky error, env not advanced, rew = 0, done = 0
        *err_out |= ERRBIT_ACTION;
        for (int a = 0; a < A; ++a) rew[base + a] = 0.0f;
        done[(size_t)c * E + e] = 0;
        continue;
      }
      ep_step[e] += 1;
      int trunc = ep_step[e] >= T_max;  // S:185 truncation flagged
      uint8_t d = (uint8_t)((term ? 1 : 0) | (trunc ? 2 : 0));
      double rsum = 0, retsum = 0;
      for (int a = 0; a < A; ++a) {
        rew[base + a] = r[a];
        ep_ret[e * A + a] += r[a];
        rsum += (double)r[a];
      }
      done[(size_t)c * E + e] = d;
      st[3] += rsum;
      if (d) {  // auto_reset; statistics of completed episodes
        for (int a = 0; a < A; ++a) retsum += (double)ep_ret[e * A + a];
        st[0] += 1; st[1] += retsum; st[2] += ep_step[e];
        reset_count[e] += 1;
        init_env(e);
        ep_step[e] = 0;
        for (int a = 0; a < A; ++a) ep_ret[e * A + a] = 0.0f;
      }
      write_obs_live(e);
    }
  }
};

/* ------------------------------------------------------------------------------------
 * NEXT-N2 (first stage): generalised advantage estimation over the time-major store,
 * SPEC compute_gae, "standard actor-critic machinery the paper presumes"
 * ("supports actor-critic algorithms"), reading R30 of DESIGN.md:
 *   columns c = e*A + a; d = done[t][e]; v_T = bootstrap[c]; A_T = 0; for t = T-1 .. 0:
 *     terminated, or truncated without a terminal value:  delta = r_t - v_t;  A_t = delta
 *     truncated with v_trunc given:       delta = (r_t + g*vtr_t) - v_t; A_t = delta
 *     otherwise:  delta = (r_t + g*v_{t+1}) - v_t;  A_t = delta + (g*l)*A_{t+1}
 *     returns_t = A_t + v_t
 * The recursion of S:392 written out with the done mask applied by dropping the masked
 * terms; every operation rounds to R (fp32 parity mode, fp64 for the brute-force pins).
 * ---------------------------------------------------------------------------------- */
template <class R>
void gae(int T, int64_t E, int A, const R* rew, const uint8_t* done, const R* values,
         const R* bootstrap, const R* v_trunc, R gamma, R lambda, R* adv, R* ret) {
  const int64_t C = E * A;
  const R gl = gamma * lambda;
  for (int64_t c = 0; c < C; ++c) {
    R a_next = (R)0;
    for (int t = T - 1; t >= 0; --t) {
      const size_t i = (size_t)t * C + c;
      const uint8_t d = done[(size_t)t * E + c / A];
      const R r = rew[i], v = values[i];
      R delta, a;
      if ((d & 1) || ((d & 2) && !v_trunc)) {
        delta = r - v;
        a = delta;
      } else if (d & 2) {
        delta = (r + gamma * v_trunc[i]) - v;
        a = delta;
      } else {
        const R v_next = (t == T - 1) ? bootstrap[c] : values[i + C];
        delta = (r + gamma * v_next) - v;
        a = delta + gl * a_next;
      }
      adv[i] = a;
      ret[i] = a + v;
      a_next = a;
    }
  }
}

Kind parse_kind(const char* s, bool* ok) {
  *ok = true;
  std::string n(s ? s : "");
  if (n == "cartpole") return K_CARTPOLE;
  if (n == "acrobot") return K_ACROBOT;
  if (n == "pendulum") return K_PENDULUM;
  if (n == "tag") return K_TAG;
  if (n == "surface") return K_SURFACE;
  if (n == "dummy") return K_DUMMY;
  if (user_envs().count(n)) return K_USER;
  *ok = false;
  return K_DUMMY;
}

int status_from_err(int err) {
  if (err & ERRBIT_PROBS) return E_INVALID_PROBS;
  if (err & ERRBIT_ACTION) return E_INVALID_ACTION;
  return E_OK;
}

}  // namespace

/* =====================================================================================
 * C API (ctypes) -- mirrors the product ABI in spirit, not in code.
 * ===================================================================================== */
extern "C" {

void wso_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  philox4x32_10(ctr, key, out);
}
uint32_t wso_draw(uint64_t seed, uint64_t env_global, uint32_t agent, uint32_t purpose, uint64_t j) {
  return draw(seed, env_global, agent, purpose, j);
}
float wso_u01(uint32_t w) { return u01(w); }
float wso_box_muller(uint32_t wa, uint32_t wb, int odd) { return box_muller(wa, wb, odd); }
float wso_gauss(uint64_t seed, uint64_t e_g, uint32_t agent, uint64_t t, int d, int k) {
  return gauss(seed, e_g, agent, t, d, k);
}
int wso_sample_discrete(const float* p, int n, float u, int32_t* act, float* logp, int* ambiguous) {
  return sample_discrete(p, n, u, act, logp, ambiguous);
}
/* exhaustive u grid (SURVEY 8(c) "brute force over the whole u grid"): counts[n] and the
 * number of grid points flagged ambiguous */
int64_t wso_sample_grid(const float* p, int n, int64_t* counts) {
  int64_t amb_total = 0;
  for (int i = 0; i < n; ++i) counts[i] = 0;
  for (uint32_t k = 0; k < (1u << 24); ++k) {
    int32_t a; float lp; int amb;
    if (sample_discrete(p, n, (float)k * (1.0f / 16777216.0f), &a, &lp, &amb)) return -1;
    counts[a] += 1;
    amb_total += amb;
  }
  return amb_total;
}

/* the transcendental contract (Tr<float>, reading Q3) on n inputs */
void wso_sincos_f32(const float* x, int64_t n, float* s, float* c) {
  for (int64_t i = 0; i < n; ++i) {
    s[i] = Tr<float>::sin(x[i]);
    c[i] = Tr<float>::cos(x[i]);
  }
}

int wso_cartpole_step_f32(const float* s, int a, float* out, float* r, int* term) {
  return CartPole<float>::step(s, a, out, r, term);
}
int wso_cartpole_step_f64(const double* s, int a, double* out, double* r, int* term) {
  return CartPole<double>::step(s, a, out, r, term);
}
int wso_acrobot_step_f32(const float* s, int a, float* out, float* r, int* term) {
  return Acrobot<float>::step(s, a, out, r, term);
}
int wso_acrobot_step_f64(const double* s, int a, double* out, double* r, int* term) {
  return Acrobot<double>::step(s, a, out, r, term);
}
void wso_acrobot_dsdt_f64(const double* s, double torque, double* d) { Acrobot<double>::dsdt(s, torque, d); }
int wso_acrobot_terminal_f32(const float* s) { return Acrobot<float>::terminal(s); }
int wso_pendulum_step_f32(const float* s, float u, float* out, float* r) {
  return Pendulum<float>::step(s, u, out, r);
}
int wso_pendulum_step_f64(const double* s, double u, double* out, double* r) {
  return Pendulum<double>::step(s, u, out, r);
}
double wso_mb_energy(double x, double y, double* gx, double* gy) { return mb_energy(x, y, gx, gy); }
float wso_surface_energy(const float* q, int D) { return surface_energy(q, D); }
double wso_surface_spring(const float* q, int D) { return surface_spring(q, D); }
int wso_surface_step(const float* q, const float* a, int D, float* out, float* r, int* term) {
  return surface_step(q, a, D, out, r, term);
}
int wso_tag_step(int A, int G, int n_taggers, int32_t* x, int32_t* y, uint8_t* active,
                 const int32_t* act, float* rew, int* term) {
  return tag_step(A, G, n_taggers, x, y, active, act, rew, term);
}

/* ---- batch ---- */
void* wso_create(const char* env, int64_t E, int A, uint64_t seed, int64_t env_offset,
                 int64_t E_global, int max_steps, int p0, int p1, int* status) {
  bool ok;
  Kind kind = parse_kind(env, &ok);
  if (!ok) { *status = E_UNKNOWN_ENV; return nullptr; }
  if (E <= 0 || A <= 0 || env_offset < 0) { *status = E_INVALID_ARGUMENT; return nullptr; }
  if (E_global <= 0) E_global = env_offset + E;
  if (env_offset + E > E_global) { *status = E_INVALID_ARGUMENT; return nullptr; }
  if (kind != K_TAG && A != 1) { *status = E_INVALID_ARGUMENT; return nullptr; }
  Batch* b = new Batch();
  b->kind = kind; b->E = E; b->A = A; b->seed = seed; b->offset = env_offset; b->E_global = E_global;
  switch (kind) {
    case K_CARTPOLE: b->obs_dim = 4; b->n_actions = 2; b->act_dim = 1; b->state_dim = 4; b->n_reset_draws = 4; b->T_max = 500; break;
    case K_ACROBOT: b->obs_dim = 6; b->n_actions = 3; b->act_dim = 1; b->state_dim = 4; b->n_reset_draws = 4; b->T_max = 500; break;
    case K_PENDULUM: b->obs_dim = 3; b->n_actions = 0; b->act_dim = 1; b->state_dim = 2; b->n_reset_draws = 2; b->T_max = 200; break;
    case K_TAG:
      b->tag_G = p0 > 0 ? p0 : 20;
      b->tag_taggers = p1 > 0 ? p1 : std::max(1, A / 10);
      if (b->tag_G < 2 || b->tag_taggers > A) { delete b; *status = E_INVALID_ARGUMENT; return nullptr; }
      b->obs_dim = 4; b->n_actions = 5; b->act_dim = 1; b->state_dim = 0; b->n_reset_draws = 2; b->T_max = 200;
      break;
    case K_SURFACE:
      b->D = p0 > 0 ? p0 : 20;
      if (b->D < 2) { delete b; *status = E_INVALID_ARGUMENT; return nullptr; }
      b->obs_dim = b->D + 1; b->n_actions = 0; b->act_dim = b->D; b->state_dim = b->D; b->n_reset_draws = b->D; b->T_max = 200;
      break;
    case K_DUMMY: b->obs_dim = 4; b->n_actions = 2; b->act_dim = 1; b->state_dim = 0; b->n_reset_draws = 0; b->T_max = 100; break;
    case K_USER: {
      const UserEnv& u = user_envs()[env];
      b->user = &u;
      b->obs_dim = u.obs_dim; b->n_actions = u.n_actions; b->act_dim = u.act_dim > 0 ? u.act_dim : 1;
      b->state_dim = u.state_dim;
      b->n_reset_draws = u.n_reset; b->T_max = u.max_steps;
      break;
    }
  }
  if (max_steps > 0) b->T_max = max_steps;
  b->state.assign((size_t)E * b->state_dim, 0.0f);
  if (kind == K_TAG) {
    b->tx.assign((size_t)E * A, 0); b->ty.assign((size_t)E * A, 0); b->tactive.assign((size_t)E * A, 0);
  }
  b->obs_live.assign((size_t)E * A * b->obs_dim, 0.0f);
  b->ep_step.assign(E, 0);
  b->reset_count.assign(E, 0);
  b->ep_ret.assign((size_t)E * A, 0.0f);
  if (kind != K_USER) b->reset_all();  // registered envs: wso_set_env_data, then wso_reset
  *status = E_OK;
  return b;
}

/* NEXT-N4: register the env compiled (by oracle/__init__.py) into so_path */
int wso_register_user(const char* name, const char* so_path, int state_dim, int obs_dim, int n_actions, int n_reset,
                      int max_steps, int n_params, int act_dim) {
  void* lib = dlopen(so_path, RTLD_NOW | RTLD_LOCAL);
  if (!lib) return E_INVALID_ARGUMENT;
  UserEnv u{state_dim, obs_dim, n_actions, n_reset, max_steps, n_params,
            reinterpret_cast<void (*)(float*, const float*, const float*, const float*)>(dlsym(lib, "wsu_init")),
            reinterpret_cast<void (*)(const float*, float*, const float*, const float*)>(dlsym(lib, "wsu_obs")),
            nullptr, act_dim, nullptr};
  if (act_dim > 0)
    u.step_c = reinterpret_cast<int (*)(float*, const float*, float*, const float*, const float*)>(dlsym(lib, "wsu_step"));
  else
    u.step = reinterpret_cast<int (*)(float*, int, float*, const float*, const float*)>(dlsym(lib, "wsu_step"));
  if (!u.init || !u.obs || !(u.step || u.step_c)) return E_INVALID_ARGUMENT;
  user_envs()[name] = u;
  return E_OK;
}

int wso_set_env_data(void* h, const float* prm, int64_t n_prm, const float* shared, int64_t n_shared) {
  Batch* b = (Batch*)h;
  if (b->kind != K_USER) return E_INVALID_ARGUMENT;
  b->prm.assign(prm, prm + n_prm);
  b->shared.assign(shared, shared + n_shared);
  return E_OK;
}

void wso_destroy(void* h) { delete (Batch*)h; }

int wso_set_capacity(void* h, int T) {
  Batch* b = (Batch*)h;
  if (T < 1) return E_INVALID_ARGUMENT;
  b->alloc_store(T);
  b->cursor = 0;
  return E_OK;
}

int wso_reset(void* h) {
  Batch* b = (Batch*)h;
  b->reset_all();
  return E_OK;
}

/* sample for slot `cursor` */
int wso_sample(void* h, const float* probs, int64_t row_stride, const int32_t* override_act,
               uint8_t* ambiguous) {
  Batch* b = (Batch*)h;
  if (b->cursor >= b->T_cap) return E_OUT_OF_RANGE;  // S:79 SlotOutOfRange
  int err = 0;
  b->sample_range(b->cursor, b->t, probs, row_stride, override_act, ambiguous, 0, b->E, &err);
  b->err |= err;
  b->sampled_slot = b->cursor;
  return E_OK;
}

/* step_all + auto_reset for slot `cursor`; actions == NULL uses the sampled
 * ones; else int32 [E, A] (discrete) / float [E, A, d] (continuous); logp = NaN (Q27) */
int wso_step(void* h, const void* actions) {
  Batch* b = (Batch*)h;
  if (b->cursor >= b->T_cap) return E_OUT_OF_RANGE;
  const int c = b->cursor;
  if (actions == nullptr) {
    if (b->sampled_slot != c) return E_BAD_STATE;
  } else {
    const size_t n = (size_t)b->EA();
    for (size_t i = 0; i < n; ++i) {
      if (b->n_actions) b->act_i[(size_t)c * n + i] = ((const int32_t*)actions)[i];
      else for (int k = 0; k < b->act_dim; ++k)
        b->act_f[((size_t)c * n + i) * b->act_dim + k] = ((const float*)actions)[i * b->act_dim + k];
      b->logp[(size_t)c * n + i] = std::numeric_limits<float>::quiet_NaN();
    }
  }
  double st[4] = {0, 0, 0, 0};
  int err = 0;
  b->step_range(c, 0, b->E, st, &err);
  for (int i = 0; i < 4; ++i) b->stats[(size_t)c * 4 + i] = st[i];
  b->err |= err;
  b->cursor += 1;
  b->t += 1;
  b->sampled_slot = -1;
  return E_OK;
}

/* run_rollout with given probabilities: slots [0, T); probs element
 * (t, e, a, i) at probs[t*step_stride + (e*A + a)*row_stride + i]; n_threads contiguous
 * env ranges, results independent of n_threads.
 * override_act [T, E, A] (>= 0 replaces the sampled action: Q16 adoption), ambiguous_out
 * [T, E, A] (may be NULL). */
int wso_rollout(void* h, int T, const float* probs, int64_t row_stride, int64_t step_stride,
                const int32_t* override_act, uint8_t* ambiguous_out, int n_threads) {
  Batch* b = (Batch*)h;
  if (T < 1) return E_INVALID_ARGUMENT;
  if (T > b->T_cap) return E_OUT_OF_RANGE;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > b->E) n_threads = (int)b->E;
  const uint64_t t0 = b->t;
  b->cursor = 0;
  std::vector<std::vector<double>> st(n_threads, std::vector<double>((size_t)T * 4, 0.0));
  std::vector<int> errs(n_threads, 0);
  auto worker = [&](int w) {
    int64_t e0 = b->E * w / n_threads, e1 = b->E * (w + 1) / n_threads;  // S:170 balanced
    for (int c = 0; c < T; ++c) {
      /* each worker sees the same global step index t0 + c */
      const float* pr = probs + (int64_t)c * step_stride;
      const int32_t* ov = override_act ? override_act + (size_t)c * b->EA() : nullptr;
      uint8_t* amb = ambiguous_out ? ambiguous_out + (size_t)c * b->EA() : nullptr;
      b->sample_range(c, t0 + c, pr, row_stride, ov, amb, e0, e1, &errs[w]);
      b->step_range(c, e0, e1, &st[w][(size_t)c * 4], &errs[w]);
    }
  };
  if (n_threads == 1) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (int w = 0; w < n_threads; ++w) th.emplace_back(worker, w);
    for (auto& x : th) x.join();
  }
  for (int c = 0; c < T; ++c)
    for (int i = 0; i < 4; ++i) {
      double s = 0;
      for (int w = 0; w < n_threads; ++w) s += st[w][(size_t)c * 4 + i];
      b->stats[(size_t)c * 4 + i] = s;
    }
  for (int w = 0; w < n_threads; ++w) b->err |= errs[w];
  b->t = t0 + T;
  b->cursor = T;
  b->sampled_slot = -1;
  return E_OK;
}

/* NEXT-N2: GAE (R30) over time-major arrays; v_trunc may be NULL. */
int wso_gae_f32(int T, int64_t E, int A, const float* rew, const uint8_t* done, const float* values,
                const float* bootstrap, const float* v_trunc, float gamma, float lambda, float* adv,
                float* ret) {
  if (T < 1 || E < 1 || A < 1 || !rew || !done || !values || !bootstrap || !adv || !ret)
    return E_INVALID_ARGUMENT;
  gae<float>(T, E, A, rew, done, values, bootstrap, v_trunc, gamma, lambda, adv, ret);
  return E_OK;
}
int wso_gae_f64(int T, int64_t E, int A, const double* rew, const uint8_t* done, const double* values,
                const double* bootstrap, const double* v_trunc, double gamma, double lambda, double* adv,
                double* ret) {
  if (T < 1 || E < 1 || A < 1 || !rew || !done || !values || !bootstrap || !adv || !ret)
    return E_INVALID_ARGUMENT;
  gae<double>(T, E, A, rew, done, values, bootstrap, v_trunc, gamma, lambda, adv, ret);
  return E_OK;
}

/* NEXT-N1: probabilities of the MLP policy for n observations [n][D] -> out [n][N] */
int wso_policy_logits(const float* weights, int D, int H, int N, const float* obs, int64_t n, float* out) {
  if (!weights || !obs || !out || D < 1 || H < 4 || H % 4 || N < 1 || n < 0) return E_INVALID_ARGUMENT;
  for (int64_t r = 0; r < n; ++r) policy_logits(weights, D, H, N, obs + r * D, out + r * N);
  return 0;
}
int wso_policy_probs(const float* weights, int D, int H, int N, const float* obs, int64_t n, float* out) {
  if (!weights || !obs || !out || D < 1 || H < 4 || H % 4 || N < 1) return E_INVALID_ARGUMENT;
  for (int64_t r = 0; r < n; ++r) policy_probs(weights, D, H, N, obs + r * D, out + r * N);
  return E_OK;
}

/* NEXT-N1: roll-out whose probabilities come from the MLP policy applied to each replica's
 * pre-step observation obs_live (single-agent discrete envs); otherwise as wso_rollout. */
int wso_rollout_policy(void* h, int T, const float* weights, int H, int n_threads) {
  Batch* b = (Batch*)h;
  if (T < 1 || !weights || H < 4 || H % 4 || b->n_actions < 1) return E_INVALID_ARGUMENT;  // R29' quarters
  if (T > b->T_cap) return E_OUT_OF_RANGE;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > b->E) n_threads = (int)b->E;
  const uint64_t t0 = b->t;
  const int D = b->obs_dim, N = b->n_actions;
  b->cursor = 0;
  const int A = b->A;  // multi-agent (tag): every agent evaluates the policy on its own row (R36)
  std::vector<float> probs((size_t)b->E * A * N);
  std::vector<std::vector<double>> st(n_threads, std::vector<double>((size_t)T * 4, 0.0));
  std::vector<int> errs(n_threads, 0);
  auto worker = [&](int w) {
    int64_t e0 = b->E * w / n_threads, e1 = b->E * (w + 1) / n_threads;
    for (int c = 0; c < T; ++c) {
      for (int64_t e = e0; e < e1; ++e)
        for (int ag = 0; ag < A; ++ag)
          policy_probs(weights, D, H, N, &b->obs_live[((size_t)e * A + ag) * D], &probs[((size_t)e * A + ag) * N]);
      b->sample_range(c, t0 + c, probs.data(), N, nullptr, nullptr, e0, e1, &errs[w]);
      b->step_range(c, e0, e1, &st[w][(size_t)c * 4], &errs[w]);
    }
  };
  if (n_threads == 1) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (int w = 0; w < n_threads; ++w) th.emplace_back(worker, w);
    for (auto& x : th) x.join();
  }
  for (int c = 0; c < T; ++c)
    for (int i = 0; i < 4; ++i) {
      double s = 0;
      for (int w = 0; w < n_threads; ++w) s += st[w][(size_t)c * 4 + i];
      b->stats[(size_t)c * 4 + i] = s;
    }
  for (int w = 0; w < n_threads; ++w) b->err |= errs[w];
  b->t = t0 + T;
  b->cursor = T;
  b->sampled_slot = -1;
  return E_OK;
}

/* NEXT-N1 for continuous actions (reading R34): a Gaussian policy -- the R29 network with d
 * linear outputs as the mean (mean_i = b2_i + ((P_0 + P_1) + (P_2 + P_3)), the R29' quarter
 * sums of fma(W2[j][i], h_j, .)) and a learned, state-independent log standard deviation vector;
 * packed weights
 * W1 [D][H] | b1 [H] | W2 [H][d] | b2 [d] | log_std [d].  Each step the replica's head row
 * (mean | log_std) is sampled by the R14 Gaussian head exactly as a given row would be. */
static void policy_gauss_row(const float* w, int D, int H, int d, const float* obs, float* row) {
  const float* W1 = w;
  const float* b1 = W1 + (size_t)D * H;
  const float* W2 = b1 + H;
  const float* b2 = W2 + (size_t)H * d;
  const float* log_std = b2 + d;
  (void)b1;
  std::vector<float> h((size_t)H);
  policy_hidden(w, D, H, obs, h.data());
  for (int i = 0; i < d; ++i) {
    row[i] = quarter_dot(W2 + i, d, h.data(), H, b2[i]);
    row[d + i] = log_std[i];
  }
}

int wso_policy_gauss_rows(const float* weights, int D, int H, int d, const float* obs, int64_t n, float* out) {
  for (int64_t r = 0; r < n; ++r) policy_gauss_row(weights, D, H, d, obs + r * D, out + r * 2 * d);
  return E_OK;
}

int wso_rollout_policy_gauss(void* h, int T, const float* weights, int H, int n_threads) {
  Batch* b = (Batch*)h;
  if (T < 1 || !weights || H < 4 || H % 4 || b->A != 1 || b->n_actions != 0) return E_INVALID_ARGUMENT;
  if (T > b->T_cap) return E_OUT_OF_RANGE;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > b->E) n_threads = (int)b->E;
  const uint64_t t0 = b->t;
  const int D = b->obs_dim, d = b->act_dim;
  b->cursor = 0;
  std::vector<float> rows((size_t)b->E * 2 * d);
  std::vector<std::vector<double>> st(n_threads, std::vector<double>((size_t)T * 4, 0.0));
  std::vector<int> errs(n_threads, 0);
  auto worker = [&](int w) {
    int64_t e0 = b->E * w / n_threads, e1 = b->E * (w + 1) / n_threads;
    for (int c = 0; c < T; ++c) {
      for (int64_t e = e0; e < e1; ++e)
        policy_gauss_row(weights, D, H, d, &b->obs_live[(size_t)e * D], &rows[(size_t)e * 2 * d]);
      b->sample_range(c, t0 + c, rows.data(), 2 * d, nullptr, nullptr, e0, e1, &errs[w]);
      b->step_range(c, e0, e1, &st[w][(size_t)c * 4], &errs[w]);
    }
  };
  if (n_threads == 1) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (int w = 0; w < n_threads; ++w) th.emplace_back(worker, w);
    for (auto& x : th) x.join();
  }
  for (int c = 0; c < T; ++c)
    for (int i = 0; i < 4; ++i) {
      double s = 0;
      for (int w = 0; w < n_threads; ++w) s += st[w][(size_t)c * 4 + i];
      b->stats[(size_t)c * 4 + i] = s;
    }
  for (int w = 0; w < n_threads; ++w) b->err |= errs[w];
  b->t = t0 + T;
  b->cursor = T;
  b->sampled_slot = -1;
  return E_OK;
}

int wso_synchronize(void* h) { return status_from_err(((Batch*)h)->err); }

/* introspection: info[0..9] = obs_dim, n_actions, act_dim, state_dim, T_max, T_cap,
 * cursor, t, A, E */
void wso_info(void* h, int64_t* info) {
  Batch* b = (Batch*)h;
  info[0] = b->obs_dim; info[1] = b->n_actions; info[2] = b->act_dim; info[3] = b->state_dim;
  info[4] = b->T_max; info[5] = b->T_cap; info[6] = b->cursor; info[7] = (int64_t)b->t;
  info[8] = b->A; info[9] = b->E;
}

void* wso_get(void* h, const char* name) {
  Batch* b = (Batch*)h;
  std::string n(name);
  if (n == "obs") return b->obs.data();
  if (n == "act") return b->n_actions ? (void*)b->act_i.data() : (void*)b->act_f.data();
  if (n == "logp") return b->logp.data();
  if (n == "rew") return b->rew.data();
  if (n == "done") return b->done.data();
  if (n == "stats") return b->stats.data();
  if (n == "state") return b->state.data();
  if (n == "obs_live") return b->obs_live.data();
  if (n == "ep_step") return b->ep_step.data();
  if (n == "reset_count") return b->reset_count.data();
  if (n == "ep_ret") return b->ep_ret.data();
  if (n == "tag_x") return b->tx.data();
  if (n == "tag_y") return b->ty.data();
  if (n == "tag_active") return b->tactive.data();
  return nullptr;
}

}  // extern "C"
