// composer.cu -- NEXT-N4: runtime environment composer.  A user environment is plain C
// source (three functions, include/ws.h "NEXT-N4"), compiled at registration time by NVRTC
// for sm_100a into a fused roll-out template (the analogue of the paper's Numba / CUDA C
// environment path: "environments ... written in CUDA C or Numba", P:65 / P:71 one
// replica per GPU thread, "domain agnostic"), loaded per device with
// cudaLibraryLoadData and launched through the same handle API as the built-in envs.
//
// The template implements the engine's semantics exactly as the built-in lane kernels do
// (DESIGN R11-R15, R19-R21): Philox4x32-10 streams keyed by the global replica index, the
// R13 inverse-CDF sampler on the given probabilities (fp64 prefix sums), the pre-step
// observation in obs[t] (R12), truncation at T_max (R10), auto-reset from the RESET stream
// (draw j = reset_count * n_reset + i), sticky device errors (R19), exact fixed-point
// per-slot statistics (R20).  The user functions receive a per-replica parameter row
// (parameter jitter) and a shared read-only array in global memory (e.g. a 3-D grid, Fig 1).
// NVRTC is loaded with dlopen at the first registration, so libws has no link-time
// dependency on it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ws.h"
#include "kernels.h"

namespace {

// ------------------------------------------------------------------------------ NVRTC
struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
  nvrtcResult (*log_size)(nvrtcProgram, size_t*);
  nvrtcResult (*log)(nvrtcProgram, char*);
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*);
  nvrtcResult (*cubin)(nvrtcProgram, char*);
  nvrtcResult (*destroy)(nvrtcProgram*);
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                             "/usr/local/cuda/lib64/libnvrtc.so"}) {
      if ((lib = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
    }
    if (!lib) {
      n.why = "libnvrtc.so.12 not found";
      return;
    }
    bool good = true;
    auto sym = [&](const char* s) {
      void* p = dlsym(lib, s);
      good = good && p;
      return p;
    };
    n.create = reinterpret_cast<decltype(n.create)>(sym("nvrtcCreateProgram"));
    n.compile = reinterpret_cast<decltype(n.compile)>(sym("nvrtcCompileProgram"));
    n.log_size = reinterpret_cast<decltype(n.log_size)>(sym("nvrtcGetProgramLogSize"));
    n.log = reinterpret_cast<decltype(n.log)>(sym("nvrtcGetProgramLog"));
    n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(sym("nvrtcGetCUBINSize"));
    n.cubin = reinterpret_cast<decltype(n.cubin)>(sym("nvrtcGetCUBIN"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("nvrtcDestroyProgram"));
    n.ok = good;
    if (!good) n.why = "libnvrtc: missing symbols";
  });
  return n;
}

// ------------------------------------------------------------------------------ template
// Kernel arguments: the same struct is spelled in the template source below (by value).
struct UserArgs {
  float* obs;
  int32_t* act;
  float* logp;
  float* rew;
  uint8_t* done;
  unsigned long long* stats;
  float* state;
  float* obs_live;
  int32_t* ep_step;
  uint32_t* reset_count;
  float* ep_ret;
  uint32_t* err;
  const float* prm;
  const float* shared;
  int64_t E;
  int64_t offset;
  int32_t max_steps;
  int32_t write_logp;
  uint32_t k0, k1;
};

const char* kPrelude = R"WS(
typedef unsigned int ws_u32; typedef unsigned long long ws_u64; typedef long long ws_i64;
typedef unsigned char ws_u8; typedef int ws_i32;
#define WS_FN __device__ __forceinline__
/* transcendental contract (DESIGN R3): fp64 evaluation, one rounding to fp32.  sin / cos use
   the library's branch-free fp64 evaluation (Cody-Waite reduction by pi/2 with the fdlibm
   three-part constant, Taylor polynomials through r^17 / r^18 on |r| <= pi/4 -- pinned against
   the host libm by the device tests); |x| >= 2^20 falls back to libdevice */
WS_FN void ws_sincos64(double x, double* s, double* c) {
  const double kd = fma(x, 6.36619772367581382433e-01, 6755399441055744.0);
  const double k = kd - 6755399441055744.0;
  const int q = __double2loint(kd);
  double r = fma(-k, 1.57079632673412561417e+00, x);
  r = fma(-k, 6.07710050630396597660e-11, r);
  r = fma(-k, 2.02226624871116645580e-21, r);
  r = fma(-k, 8.47842766036889956997e-32, r);
  const double z = r * r, z2 = z * z, z4 = z2 * z2;
  const double s_a = fma(z, 1.0 / 120.0, -1.0 / 6.0);
  const double s_b = fma(z, 1.0 / 362880.0, -1.0 / 5040.0);
  const double s_c = fma(z, 1.0 / 6227020800.0, -1.0 / 39916800.0);
  const double s_d = fma(z, 1.0 / 355687428096000.0, -1.0 / 1307674368000.0);
  const double ps = fma(z4, fma(z2, s_d, s_c), fma(z2, s_b, s_a));
  const double c_a = fma(z, 1.0 / 24.0, -0.5);
  const double c_b = fma(z, 1.0 / 40320.0, -1.0 / 720.0);
  const double c_c = fma(z, 1.0 / 479001600.0, -1.0 / 3628800.0);
  const double c_d = fma(z, 1.0 / 20922789888000.0, -1.0 / 87178291200.0);
  const double pc = fma(z4, fma(z4, -1.0 / 6402373705728000.0, fma(z2, c_d, c_c)), fma(z2, c_b, c_a));
  const double sr = fma(r * z, ps, r);
  const double cr = fma(z, pc, 1.0);
  const double s0 = (q & 1) ? cr : sr;
  const double c0 = (q & 1) ? sr : cr;
  *s = (q & 2) ? -s0 : s0;
  *c = ((q + 1) & 2) ? -c0 : c0;
  if (!(fabs(x) < 1048576.0)) sincos(x, s, c);
}
WS_FN float ws_sin(float x) { double s, c; ws_sincos64((double)x, &s, &c); return (float)s; }
WS_FN float ws_cos(float x) { double s, c; ws_sincos64((double)x, &s, &c); return (float)c; }
WS_FN float ws_exp(float x) { return (float)exp((double)x); }
WS_FN float ws_log(float x) { return (float)log((double)x); }
WS_FN float ws_tanh(float x) { return (float)tanh((double)x); }
WS_FN float ws_sqrt(float x) { return __fsqrt_rn(x); }
WS_FN float ws_min(float a, float b) { return b < a ? b : a; }
WS_FN float ws_max(float a, float b) { return a < b ? b : a; }
WS_FN float ws_clip(float x, float lo, float hi) { return x < lo ? lo : (hi < x ? hi : x); }
WS_FN float ws_abs(float x) { return fabsf(x); }
WS_FN float ws_floor(float x) { return floorf(x); }
WS_FN float ws_fmod(float x, float y) { return fmodf(x, y); }
/* both with one fp64 range reduction, each rounded once (R3) */
WS_FN void ws_sincos(float x, float *s, float *c) {
  double sd, cd;
  ws_sincos64((double)x, &sd, &cd);
  *s = (float)sd;
  *c = (float)cd;
}
#line 1 "user_env.c"
)WS";

const char* kEngine = R"WS(
#line 1 "ws_composer_engine"
struct WsUserArgs {
  float* obs; ws_i32* act; float* logp; float* rew; ws_u8* done; ws_u64* stats;
  float* state; float* obs_live; ws_i32* ep_step; ws_u32* reset_count; float* ep_ret; ws_u32* err;
  const float* prm; const float* shared;
  ws_i64 E; ws_i64 offset; ws_i32 max_steps; ws_i32 write_logp; ws_u32 k0, k1;
};

/* Philox4x32-10; draw j of stream (env_global, agent, purpose) = word j & 3 of
   Philox(ctr = (j >> 2, env_global, agent, purpose), key) (DESIGN R15) */
WS_FN void ws_philox(ws_u32 c0, ws_u32 c1, ws_u32 c2, ws_u32 c3, ws_u32 k0, ws_u32 k1, ws_u32* w) {
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const ws_u32 lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const ws_u32 lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const ws_u32 n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  w[0] = c0; w[1] = c1; w[2] = c2; w[3] = c3;
}
WS_FN ws_u32 ws_draw(const WsUserArgs& a, ws_u32 eg, ws_u32 purpose, ws_u64 j) {
  ws_u32 w[4];
  ws_philox((ws_u32)(j >> 2), eg, 0u, purpose, a.k0, a.k1, w);
  return w[j & 3];
}
WS_FN float ws_u01(ws_u32 w) { return (float)(w >> 8) * (1.0f / 16777216.0f); }
/* R14: Gaussian draw j of the GAUSS stream: Box-Muller on the word pair (2p, 2p+1),
   p = (j & 3) >> 1, u1 in (0, 1], u2 in [0, 1), fp64, one rounding */
WS_FN float ws_gauss(const WsUserArgs& a, ws_u32 eg, ws_u64 j) {
  ws_u32 w[4];
  ws_philox((ws_u32)(j >> 2), eg, 0u, 3u, a.k0, a.k1, w);
  const int p = (int)((j & 3) >> 1);
  const double u1 = (double)((w[2 * p] >> 8) + 1) * (1.0 / 16777216.0);
  const double u2 = (double)(w[2 * p + 1] >> 8) * (1.0 / 16777216.0);
  const double r = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.14159265358979323846 * u2;
  return (float)((j & 1) ? r * sin(ang) : r * cos(ang));
}

WS_FN void ws_init(const WsUserArgs& a, ws_u32 eg, ws_u32 rc, float* s, const float* prm) {
  float u[WS_R > 0 ? WS_R : 1];
  for (int i = 0; i < WS_R; ++i) u[i] = ws_u01(ws_draw(a, eg, 2u, (ws_u64)rc * WS_R + i));
  ws_env_init(s, u, prm, a.shared);
}

/* R13: inverse CDF in index order on u * S (fp64), strict <, zero-probability actions never
   drawn, fallback = last nonzero; invalid row -> -1 */
WS_FN int ws_sample(const float* p, float u, float* lp) {
  double S = 0.0;
  int last = -1;
  bool bad = false;
  for (int i = 0; i < WS_N; ++i) {
    const float x = p[i];
    bad = bad || !(x >= 0.0f) || !isfinite(x);
    S += (double)x;
    if (x > 0.0f) last = i;
  }
  if (bad || !(S > 0.0) || !isfinite(S)) { *lp = __int_as_float(0x7fc00000); return -1; }
  const double target = (double)u * S;
  double C = 0.0;
  int chosen = -1;
  for (int i = 0; i < WS_N; ++i) {
    C += (double)p[i];
    if (chosen < 0 && p[i] > 0.0f && target < C) chosen = i;
  }
  if (chosen < 0) chosen = last;
  *lp = (float)(log((double)p[chosen]) - log(S));
  return chosen;
}

WS_FN ws_i64 ws_fx(float v) { return __float2ll_rn(v * 4294967296.0f); }
/* exact warp sum of 64-bit values (two's complement, mod 2^64): four 16-bit chunks, one
   REDUX each (32 x (2^16 - 1) < 2^32), recombined */
WS_FN ws_i64 ws_wsum(ws_i64 v) {
  const ws_u64 u = (ws_u64)v;
  ws_u64 t = 0;
  for (int k = 0; k < 4; ++k) t += (ws_u64)__reduce_add_sync(0xffffffffu, (ws_u32)((u >> (16 * k)) & 0xffffu)) << (16 * k);
  return (ws_i64)t;
}

/* R13 sampler state for a probability row that is constant over the roll-out (step_stride
   0): prefix sums, total and log-probabilities computed once per replica */
struct WsRow {
  double C[WS_N];
  double S;
  float lp[WS_N];
  int last;
  bool bad;
};
WS_FN void ws_row_init(const float* p, WsRow& r) {
  r.S = 0.0; r.last = -1; r.bad = false;
  for (int i = 0; i < WS_N; ++i) {
    const float x = p[i];
    r.bad = r.bad || !(x >= 0.0f) || !isfinite(x);
    r.S += (double)x;
    r.C[i] = r.S;
    if (x > 0.0f) r.last = i;
  }
  r.bad = r.bad || !(r.S > 0.0) || !isfinite(r.S);
  const double lS = r.bad ? 0.0 : log(r.S);
  for (int i = 0; i < WS_N; ++i) r.lp[i] = (!r.bad && p[i] > 0.0f) ? (float)(log((double)p[i]) - lS) : 0.0f;
}
WS_FN int ws_row_draw(const WsRow& r, const float* p, float u, float* lp) {
  if (r.bad) { *lp = __int_as_float(0x7fc00000); return -1; }
  const double target = (double)u * r.S;
  int chosen = -1;
  for (int i = 0; i < WS_N; ++i)
    if (chosen < 0 && p[i] > 0.0f && target < r.C[i]) chosen = i;
  if (chosen < 0) chosen = r.last;
  *lp = r.lp[chosen];
  return chosen;
}

extern "C" __global__ void k_user_reset(const WsUserArgs a) {
  const ws_i64 e = (ws_i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.E) return;
  const float* prm = a.prm ? a.prm + e * (WS_P > 0 ? WS_P : 1) : 0;
  float s[WS_S];
  ws_init(a, (ws_u32)(a.offset + e), 0u, s, prm);
  for (int i = 0; i < WS_S; ++i) a.state[e * WS_S + i] = s[i];
  float o[WS_D];
  ws_env_obs(s, o, prm, a.shared);
  for (int i = 0; i < WS_D; ++i) a.obs_live[e * WS_D + i] = o[i];
  a.ep_step[e] = 0;
  a.reset_count[e] = 0u;
  a.ep_ret[e] = 0.0f;
}

/* fused roll-out of T steps, one replica per thread (P:65, P:71) */
/* The fused loop.  kH == 0: actions from the given probabilities (R13); kH > 0: from the
   R29 MLP policy (hidden kH, weights in shared memory `sw`) on the pre-step observation,
   evaluated in R29's order, with the R31 critic written to values / bootstrap if kCritic. */
template <int kH, bool kCritic>
WS_FN void ws_run(const WsUserArgs& a, int T, ws_u64 t0, const float* probs, ws_i64 row_stride,
                  ws_i64 step_stride, const float* sw, float* values, float* bootstrap) {
  const ws_i64 e0 = (ws_i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e0 - (threadIdx.x & 31) >= a.E) return;          /* whole warp past the end */
  const bool live = e0 < a.E;
  const ws_i64 e = live ? e0 : a.E - 1;                /* tail lanes shadow E-1, store nothing */
  const ws_u32 eg = (ws_u32)(a.offset + e);
  const float* prm = a.prm ? a.prm + e * (WS_P > 0 ? WS_P : 1) : 0;
  float s[WS_S], o[WS_D];
  for (int i = 0; i < WS_S; ++i) s[i] = a.state[e * WS_S + i];
  for (int i = 0; i < WS_D; ++i) o[i] = a.obs_live[e * WS_D + i];
  ws_i32 ep_step = a.ep_step[e];
  ws_u32 rc = a.reset_count[e];
  float ep_ret = a.ep_ret[e];
  ws_u32 err = 0;
  const bool hoist = kH == 0 && step_stride == 0 && WS_C == 0;  /* same row every step: CDF and logs once */
  float p0[WS_N];
  WsRow row;
  if (hoist) {
    for (int i = 0; i < WS_N; ++i) p0[i] = probs[e * row_stride + i];
    ws_row_init(p0, row);
  }
  const int kHH = kH > 0 ? kH : 1;
  const int kHQ = kHH >= 4 ? kHH / 4 : 1;  /* R29' quarter size */
  const float* W1 = sw;                       /* [D][H] */
  const float* b1 = W1 + WS_D * kHH;          /* [H] */
  const float* W2 = b1 + kHH;                 /* [H][N] */
  const float* b2 = W2 + kHH * WS_N;          /* [N] */
  const float* wv = b2 + WS_N;                /* [H] | bv (critic) */
  ws_u32 w4[4] = {0u, 0u, 0u, 0u};
  for (int c = 0; c < T; ++c) {
    const ws_u64 t = t0 + (ws_u64)c;
    const ws_i64 idx = (ws_i64)c * a.E + e;
    if (live) for (int i = 0; i < WS_D; ++i) __stcs(a.obs + idx * WS_D + i, o[i]);   /* R12 */
    /* ACTION stream: one Philox block serves 4 consecutive steps (draw j = t, R15) */
    if (c == 0 || (t & 3) == 0) ws_philox((ws_u32)(t >> 2), eg, 0u, 1u, a.k0, a.k1, w4);
    const float u = ws_u01(w4[t & 3]);
    float lp;
    int act;
#if WS_C > 0
    /* continuous actions (R14): row = mean [WS_C] | log_std [WS_C] */
    float cact[WS_C];
    {
      const float* row = probs + (ws_i64)c * step_stride + e * row_stride;
      bool okr = true;
      for (int k = 0; k < WS_C; ++k) okr = okr && isfinite(row[k]) && isfinite(row[WS_C + k]);
      double lpd = 0.0;
      for (int k = 0; k < WS_C; ++k) {
        const float z = ws_gauss(a, eg, t * (ws_u64)WS_C + (ws_u64)k);
        const float sd = (float)exp((double)row[WS_C + k]);
        cact[k] = okr ? row[k] + sd * z : __int_as_float(0x7fc00000);
        lpd = lpd + (((-0.5 * (double)z) * (double)z - (double)row[WS_C + k]) - 0.9189385332046727);
        if (live) __stcs(reinterpret_cast<float*>(a.act) + idx * WS_C + k, cact[k]);
      }
      lp = okr ? (float)lpd : __int_as_float(0x7fc00000);
      bool fin = true;
      for (int k = 0; k < WS_C; ++k) fin = fin && isfinite(cact[k]);
      act = fin ? 0 : -1;
      if (live && !okr) err |= 2u;
    }
    if (true) {
    } else if (kH > 0) {
#else
    if (kH > 0) {
#endif
      /* R29': second layer as four quarter chains P_q from +0, l = b2 + ((P0 + P1) + (P2 + P3)) */
      float lg[WS_N], Pq[4][WS_N], Pv[4];
      for (int qq = 0; qq < 4; ++qq) {
        Pv[qq] = 0.0f;
        for (int i = 0; i < WS_N; ++i) Pq[qq][i] = 0.0f;
      }
      for (int j = 0; j < kHH; ++j) {
        float acc = b1[j];
        for (int k = 0; k < WS_D; ++k) acc = __fmaf_rn(W1[k * kHH + j], o[k], acc);
        const float hj = acc > 0.0f ? acc : 0.0f;
        const int qq = j / kHQ;
        for (int i = 0; i < WS_N; ++i) Pq[qq][i] = __fmaf_rn(W2[j * WS_N + i], hj, Pq[qq][i]);
        if (kCritic) Pv[qq] = __fmaf_rn(wv[j], hj, Pv[qq]);
      }
      for (int i = 0; i < WS_N; ++i)
        lg[i] = __fadd_rn(b2[i], __fadd_rn(__fadd_rn(Pq[0][i], Pq[1][i]), __fadd_rn(Pq[2][i], Pq[3][i])));
      const float v = kCritic ? __fadd_rn(wv[kHH], __fadd_rn(__fadd_rn(Pv[0], Pv[1]), __fadd_rn(Pv[2], Pv[3]))) : 0.0f;
      if (kCritic && live) __stcs(values + idx, v);
      float m = lg[0];
      for (int i = 1; i < WS_N; ++i) m = lg[i] > m ? lg[i] : m;
      float p[WS_N], S = 0.0f;
      for (int i = 0; i < WS_N; ++i) {
        p[i] = (float)exp((double)__fsub_rn(lg[i], m));
        S = __fadd_rn(S, p[i]);
      }
      for (int i = 0; i < WS_N; ++i) p[i] = __fdiv_rn(p[i], S);
      act = ws_sample(p, u, &lp);
    } else {
      act = hoist ? ws_row_draw(row, p0, u, &lp)
                  : ws_sample(probs + (ws_i64)c * step_stride + e * row_stride, u, &lp);
    }
    if (live) {
#if WS_C == 0
      __stcs(a.act + idx, act);
#endif
      if (a.write_logp) __stcs(a.logp + idx, lp);
    }
    float r = 0.0f;
    ws_u32 d = 0u;
    float ret = 0.0f;
    ws_i32 es = 0;
    if (act < 0) {                                   /* R19: not advanced, rew 0, done 0 */
      if (live) err |= (WS_C > 0 ? 1u : 3u);
    } else {
#if WS_C > 0
      const int term = ws_env_step(s, cact, &r, prm, a.shared);
#else
      const int term = ws_env_step(s, act, &r, prm, a.shared);
#endif
      es = ep_step + 1;
      d = (term ? 1u : 0u) | (es >= a.max_steps ? 2u : 0u);
      ret = ep_ret + r;
      ep_step = es;
      ep_ret = ret;
      if (d) {                                       /* auto-reset (R11) */
        rc += 1u;
        ws_init(a, eg, rc, s, prm);
        ep_step = 0;
        ep_ret = 0.0f;
      }
      ws_env_obs(s, o, prm, a.shared);
    }
    if (live) {
      __stcs(a.rew + idx, r);
      a.done[idx] = (ws_u8)d;
    }
    /* exact fixed-point per-slot statistics (R20), warp-reduced then one atomic per field */
    const bool dl = live && d;
    const ws_i64 f3 = ws_wsum(live ? ws_fx(r) : 0);
    const unsigned any = __ballot_sync(0xffffffffu, dl);
    ws_i64 f0 = 0, f1 = 0, f2 = 0;
    if (any) {
      f0 = ws_wsum(dl ? 1 : 0);
      f1 = ws_wsum(dl ? ws_fx(ret) : 0);
      f2 = ws_wsum(dl ? (ws_i64)es : 0);
    }
    if ((threadIdx.x & 31) == 0) {
      ws_u64* st = a.stats + (ws_i64)c * 4;
      if (f3) atomicAdd(st + 3, (ws_u64)f3);
      if (any) {
        atomicAdd(st + 0, (ws_u64)f0);
        atomicAdd(st + 1, (ws_u64)f1);
        atomicAdd(st + 2, (ws_u64)f2);
      }
    }
  }
  if (kCritic) {  /* bootstrap value of the observation after the last step (R29' quarters) */
    float Pv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int j = 0; j < kHH; ++j) {
      float acc = b1[j];
      for (int k = 0; k < WS_D; ++k) acc = __fmaf_rn(W1[k * kHH + j], o[k], acc);
      Pv[j / kHQ] = __fmaf_rn(wv[j], acc > 0.0f ? acc : 0.0f, Pv[j / kHQ]);
    }
    if (live) bootstrap[e] = __fadd_rn(wv[kHH], __fadd_rn(__fadd_rn(Pv[0], Pv[1]), __fadd_rn(Pv[2], Pv[3])));
  }
  if (live) {
    for (int i = 0; i < WS_S; ++i) a.state[e * WS_S + i] = s[i];
    for (int i = 0; i < WS_D; ++i) a.obs_live[e * WS_D + i] = o[i];
    a.ep_step[e] = ep_step;
    a.reset_count[e] = rc;
    a.ep_ret[e] = ep_ret;
    if (err) atomicOr(a.err, err);
  }
}

extern "C" __global__ void k_user_rollout(const WsUserArgs a, int T, ws_u64 t0, const float* probs,
                                          ws_i64 row_stride, ws_i64 step_stride) {
  ws_run<0, false>(a, T, t0, probs, row_stride, step_stride, 0, 0, 0);
}

#if WS_C == 0
/* Roll-out with GIVEN constant probabilities (step stride 0): the library's plan kernel has
   already drawn every action (R28: act / logp slabs and the packed plan, four 8-bit actions per
   word, 0xFF = invalid row), so the loop only runs the user's dynamics -- the hand-written lane
   kernel's structure: actions prefetched one 4-step group ahead, the reset state init(e, rc + 1)
   kept ready in registers and selected on done (refilled once per group; a second reset inside a
   group recomputes it, warp-uniformly), per-warp statistics window in shared memory reduced every
   16 slots to exact fixed point (one atomic per field, slot and warp; R20). */
#define WS_WR 16
extern "C" __global__ void __launch_bounds__(128) k_user_rollout_plan(const WsUserArgs a, int T, const ws_u32* plan) {
  __shared__ float win[4][3][WS_WR][33];  /* per warp: [len | ret | rew][slot row][lane] */
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const ws_i64 e0 = (ws_i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e0 - lane >= a.E) return;                         /* whole warp past the end */
  const bool live = e0 < a.E;
  const ws_i64 e = live ? e0 : a.E - 1;                 /* tail lanes shadow E-1 (identical stores) */
  const ws_u32 eg = (ws_u32)(a.offset + e);
  const float* prm = a.prm ? a.prm + e * (WS_P > 0 ? WS_P : 1) : 0;
  float s[WS_S], nx[WS_S], o[WS_D];
  for (int i = 0; i < WS_S; ++i) s[i] = a.state[e * WS_S + i];
  for (int i = 0; i < WS_D; ++i) o[i] = a.obs_live[e * WS_D + i];
  ws_i32 ep_step = a.ep_step[e];
  ws_u32 rc = a.reset_count[e];
  float ep_ret = a.ep_ret[e];
  ws_u32 err = 0;
  bool stale = true;
  const int ng = (T + 3) / 4;
  ws_u32 pk_next = plan[e];
  for (int j = 0; j < ng; ++j) {
    const ws_u32 pk = pk_next;
    if (j + 1 < ng) pk_next = plan[(ws_i64)(j + 1) * a.E + e];
    if (__any_sync(0xffffffffu, stale)) { ws_init(a, eg, rc + 1u, nx, prm); stale = false; }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = 4 * j + k;
      if (c >= T) break;
      const ws_i64 idx = (ws_i64)c * a.E + e;
#if WS_D % 4 == 0                                    /* R12, vector stores: a warp writes whole lines */
      for (int i = 0; i < WS_D; i += 4) __stcs(reinterpret_cast<float4*>(a.obs + idx * WS_D + i), make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]));
#elif WS_D % 2 == 0
      for (int i = 0; i < WS_D; i += 2) __stcs(reinterpret_cast<float2*>(a.obs + idx * WS_D + i), make_float2(o[i], o[i + 1]));
#else
      for (int i = 0; i < WS_D; ++i) __stcs(a.obs + idx * WS_D + i, o[i]);
#endif
      const int act = (int)(signed char)(unsigned char)(pk >> (8 * k));
      float r = 0.0f;
      ws_u32 d = 0u;
      float ret = 0.0f;
      ws_i32 es = 0;
      if (act < 0) {                                 /* R19: not advanced, rew 0, done 0 */
        if (live) err |= 3u;
      } else {
        const int term = ws_env_step(s, act, &r, prm, a.shared);
        es = ep_step + 1;
        d = (term ? 1u : 0u) | (es >= a.max_steps ? 2u : 0u);
        ret = ep_ret + r;
        ep_step = d ? 0 : es;
        ep_ret = d ? 0.0f : ret;
      }
      if (__any_sync(0xffffffffu, d != 0u && stale)) {  /* second reset inside this group */
        if (d != 0u && stale) ws_init(a, eg, rc + 1u, nx, prm);
      }
      if (d) {                                       /* auto-reset (R11) from the look-ahead state */
        rc += 1u;
        for (int i = 0; i < WS_S; ++i) s[i] = nx[i];
        stale = true;
      }
      ws_env_obs(s, o, prm, a.shared);
      __stcs(a.rew + idx, r);
      a.done[idx] = (ws_u8)d;
      const int row = c & (WS_WR - 1);
      win[wp][0][row][lane] = (live && d) ? __int_as_float(es) : 0.0f;
      win[wp][1][row][lane] = (live && d) ? ret : 0.0f;
      win[wp][2][row][lane] = live ? r : 0.0f;
      if (row == WS_WR - 1 || c == T - 1) {          /* lane i reduces slot row i (R20, exact) */
        __syncwarp();
        if (lane <= row) {
          ws_u64 nd = 0, ln = 0;
          ws_i64 rt = 0, rs = 0;
          for (int q = 0; q < 32; ++q) {
            const int l = __float_as_int(win[wp][0][lane][q]);
            nd += l != 0 ? 1u : 0u;
            ln += (ws_u64)l;
            rt += ws_fx(win[wp][1][lane][q]);
            rs += ws_fx(win[wp][2][lane][q]);
          }
          ws_u64* st = a.stats + (ws_i64)(c - row + lane) * 4;
          if (nd) { atomicAdd(st + 0, nd); atomicAdd(st + 1, (ws_u64)rt); atomicAdd(st + 2, ln); }
          if (rs) atomicAdd(st + 3, (ws_u64)rs);
        }
        __syncwarp();
      }
    }
  }
  if (live) {
    for (int i = 0; i < WS_S; ++i) a.state[e * WS_S + i] = s[i];
    for (int i = 0; i < WS_D; ++i) a.obs_live[e * WS_D + i] = o[i];
    a.ep_step[e] = ep_step;
    a.reset_count[e] = rc;
    a.ep_ret[e] = ep_ret;
    if (err) atomicOr(a.err, err);
  }
}

/* policy roll-outs: weights (R29, + R31 value head for the critic variants) staged in shared
   memory once per CTA */
template <int kH, bool kCritic>
WS_FN void ws_policy(const WsUserArgs& a, int T, ws_u64 t0, const float* w, float* values, float* bootstrap) {
  __shared__ float sw[WS_D * kH + kH + kH * WS_N + WS_N + kH + 1];
  const int nw = WS_D * kH + kH + kH * WS_N + WS_N + (kCritic ? kH + 1 : 0);
  for (int i = threadIdx.x; i < nw; i += blockDim.x) sw[i] = w[i];
  __syncthreads();
  ws_run<kH, kCritic>(a, T, t0, 0, 0, 0, sw, values, bootstrap);
}
extern "C" __global__ void k_user_policy_32(const WsUserArgs a, int T, ws_u64 t0, const float* w) {
  ws_policy<32, false>(a, T, t0, w, 0, 0);
}
extern "C" __global__ void k_user_policy_64(const WsUserArgs a, int T, ws_u64 t0, const float* w) {
  ws_policy<64, false>(a, T, t0, w, 0, 0);
}
extern "C" __global__ void k_user_ac_32(const WsUserArgs a, int T, ws_u64 t0, const float* w, float* v, float* b) {
  ws_policy<32, true>(a, T, t0, w, v, b);
}
extern "C" __global__ void k_user_ac_64(const WsUserArgs a, int T, ws_u64 t0, const float* w, float* v, float* b) {
  ws_policy<64, true>(a, T, t0, w, v, b);
}
#endif
)WS";

// ------------------------------------------------------------------------------ registry
struct UserEnv {
  ws_env_def def{};
  std::string name, source, log;
  std::vector<char> cubin;
  struct Kernels {
    cudaLibrary_t lib;
    cudaKernel_t reset, rollout, policy32, policy64, ac32, ac64, rollout_plan;
  };
  std::map<int, Kernels> per_dev;
};

std::mutex g_mu;
std::map<std::string, std::unique_ptr<UserEnv>>& registry() {
  static std::map<std::string, std::unique_ptr<UserEnv>> r;
  return r;
}

bool builtin(const std::string& n) {
  for (const char* b : {"cartpole", "acrobot", "pendulum", "tag", "surface", "dummy"})
    if (n == b) return true;
  return false;
}

void copy_log(const std::string& s, char* log, size_t n) {
  if (!log || !n) return;
  const size_t k = std::min(n - 1, s.size());
  std::memcpy(log, s.data(), k);
  log[k] = '\0';
}

cudaError_t kernels_for(UserEnv* u, const UserEnv::Kernels** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  std::lock_guard<std::mutex> g(g_mu);
  auto it = u->per_dev.find(dev);
  if (it == u->per_dev.end()) {
    UserEnv::Kernels k{};
    if ((e = cudaLibraryLoadData(&k.lib, u->cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0))) return e;
    const std::pair<cudaKernel_t*, const char*> names[] = {
        {&k.reset, "k_user_reset"},       {&k.rollout, "k_user_rollout"}, {&k.policy32, "k_user_policy_32"},
        {&k.policy64, "k_user_policy_64"}, {&k.ac32, "k_user_ac_32"},      {&k.ac64, "k_user_ac_64"},
        {&k.rollout_plan, "k_user_rollout_plan"}};
    const int n_req = u->def.act_dim > 0 ? 2 : 7;  // continuous envs carry no policy / plan kernels
    for (int i = 0; i < n_req; ++i)
      if ((e = cudaLibraryGetKernel(names[i].first, k.lib, names[i].second))) return e;
    it = u->per_dev.emplace(dev, k).first;
  }
  *out = &it->second;
  return cudaSuccess;
}

UserArgs user_args(const ws::UserLaunch& l) {
  const ws::KArgs& k = l.k;
  return UserArgs{k.obs, static_cast<int32_t*>(k.act), k.logp, k.rew, k.done, k.stats, k.state, k.obs_live,
                  k.ep_step, k.reset_count, k.ep_ret, k.err, l.prm, l.shared, k.E, k.offset, k.max_steps,
                  k.write_logp, k.k0, k.k1};
}

}  // namespace

namespace ws {

bool user_env_spec(const char* name, UserSpec* out) {
  if (!name) return false;
  std::lock_guard<std::mutex> g(g_mu);
  auto it = registry().find(name);
  if (it == registry().end()) return false;
  const ws_env_def& d = it->second->def;
  out->handle = it->second.get();
  out->obs_dim = d.obs_dim;
  out->n_actions = d.n_actions;
  out->state_dim = d.state_dim;
  out->max_steps = d.max_steps;
  out->n_params = d.n_params;
  out->act_dim = d.act_dim;
  return true;
}

cudaError_t launch_user_reset(const UserLaunch& l) {
  const UserEnv::Kernels* k = nullptr;
  cudaError_t e = kernels_for(static_cast<UserEnv*>(l.handle), &k);
  if (e) return e;
  UserArgs a = user_args(l);
  void* args[] = {&a};
  const unsigned grid = (unsigned)((l.k.E + 127) / 128);
  return cudaLaunchKernel(reinterpret_cast<const void*>(k->reset), dim3(grid), dim3(128), args, 0, l.stream);
}

cudaError_t launch_user_rollout(const UserLaunch& l, int T, uint64_t t0, const float* probs, int64_t row_stride,
                                int64_t step_stride) {
  const UserEnv::Kernels* k = nullptr;
  cudaError_t e = kernels_for(static_cast<UserEnv*>(l.handle), &k);
  if (e) return e;
  UserArgs a = user_args(l);
  const unsigned grid = (unsigned)((l.k.E + 127) / 128);
  const UserEnv* u = static_cast<const UserEnv*>(l.handle);
  if (step_stride == 0 && u->def.act_dim == 0 && u->def.n_actions <= 8 && l.k.plan) {
    // constant probabilities: the library's plan kernel draws every action up front (R28), the
    // composed kernel runs only the dynamics
    if ((e = launch_plan(l.k, u->def.n_actions, T, t0, probs, row_stride, l.stream))) return e;
    const uint32_t* plan = l.k.plan;
    void* args[] = {&a, &T, &plan};
    return cudaLaunchKernel(reinterpret_cast<const void*>(k->rollout_plan), dim3(grid), dim3(128), args, 0,
                            l.stream);
  }
  void* args[] = {&a, &T, &t0, &probs, &row_stride, &step_stride};
  return cudaLaunchKernel(reinterpret_cast<const void*>(k->rollout), dim3(grid), dim3(128), args, 0, l.stream);
}

cudaError_t launch_user_policy(const UserLaunch& l, int T, uint64_t t0, const float* weights, int hidden,
                               float* values, float* bootstrap) {
  const UserEnv::Kernels* k = nullptr;
  cudaError_t e = kernels_for(static_cast<UserEnv*>(l.handle), &k);
  if (e) return e;
  UserArgs a = user_args(l);
  const unsigned grid = (unsigned)((l.k.E + 127) / 128);
  cudaKernel_t f = values ? (hidden == 32 ? k->ac32 : k->ac64) : (hidden == 32 ? k->policy32 : k->policy64);
  if (values) {
    void* args[] = {&a, &T, &t0, &weights, &values, &bootstrap};
    return cudaLaunchKernel(reinterpret_cast<const void*>(f), dim3(grid), dim3(128), args, 0, l.stream);
  }
  void* args[] = {&a, &T, &t0, &weights};
  return cudaLaunchKernel(reinterpret_cast<const void*>(f), dim3(grid), dim3(128), args, 0, l.stream);
}

}  // namespace ws

extern "C" {

ws_status ws_register_env(const ws_env_def* def, char* log, size_t log_size) {
  copy_log("", log, log_size);
  const bool cont = def && def->act_dim != 0;
  if (!def || !def->name || !def->source || !*def->name || builtin(def->name) || def->state_dim < 1 ||
      def->state_dim > 32 || def->obs_dim < 1 || def->obs_dim > 32 ||
      (cont ? (def->act_dim < 1 || def->act_dim > 8 || def->n_actions != 0)
            : (def->n_actions < 2 || def->n_actions > 16)) ||
      def->n_reset_draws < 0 || def->n_reset_draws > 64 || def->max_steps < 1 || def->n_params < 0 ||
      def->n_params > 64) {
    copy_log("ws_register_env: name (not a built-in), source, state_dim 1..32, obs_dim 1..32, n_actions 2..16, "
             "n_reset_draws 0..64, max_steps >= 1, n_params 0..64", log, log_size);
    return WS_ERR_INVALID_ARGUMENT;
  }
  {
    std::lock_guard<std::mutex> g(g_mu);
    if (registry().count(def->name)) {
      copy_log("ws_register_env: name already registered", log, log_size);
      return WS_ERR_INVALID_ARGUMENT;
    }
  }
  Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    copy_log("ws_register_env: " + nv.why, log, log_size);
    return WS_ERR_CUDA;
  }
  auto u = std::make_unique<UserEnv>();
  u->def = *def;
  u->name = def->name;
  u->source = def->source;
  u->def.name = u->name.c_str();
  u->def.source = u->source.c_str();
  const std::string defs = "#define WS_S " + std::to_string(def->state_dim) + "\n#define WS_D " +
                           std::to_string(def->obs_dim) + "\n#define WS_N " +
                           std::to_string(def->act_dim > 0 ? 1 : def->n_actions) + "\n#define WS_R " +
                           std::to_string(def->n_reset_draws) + "\n#define WS_P " + std::to_string(def->n_params) +
                           "\n#define WS_C " + std::to_string(def->act_dim) + "\n";
  const std::string src = defs + kPrelude + u->source + "\n" + kEngine;
  nvrtcProgram prog;
  if (nv.create(&prog, src.c_str(), "ws_user_env.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    copy_log("ws_register_env: nvrtcCreateProgram failed", log, log_size);
    return WS_ERR_CUDA;
  }
  // --fmad=false: no FMA contraction of the user's fp32 arithmetic (DESIGN R4), IEEE div/sqrt
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17", "-lineinfo",
                        "--prec-div=true", "--prec-sqrt=true", "-default-device"};
  const nvrtcResult rc = nv.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t n = 0;
  nv.log_size(prog, &n);
  std::string lg(n, '\0');
  if (n) nv.log(prog, &lg[0]);
  while (!lg.empty() && lg.back() == '\0') lg.pop_back();
  u->log = lg;
  if (rc != NVRTC_SUCCESS) {
    copy_log(lg, log, log_size);
    nv.destroy(&prog);
    return WS_ERR_INVALID_ARGUMENT;
  }
  nv.cubin_size(prog, &n);
  u->cubin.resize(n);
  nv.cubin(prog, u->cubin.data());
  nv.destroy(&prog);
  copy_log(lg, log, log_size);
  std::lock_guard<std::mutex> g(g_mu);
  registry()[u->name] = std::move(u);
  return WS_OK;
}

int32_t ws_registered_env(const char* name) {
  if (!name) return 0;
  std::lock_guard<std::mutex> g(g_mu);
  return registry().count(name) ? 1 : 0;
}

}  // extern "C"
