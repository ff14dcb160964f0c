// kernels.cu -- the sm_100a kernels of libws.
//
//  k_rollout_lane<Env>  A7: T fused steps (sample -> log -> step -> reward/done -> auto-reset
//                       -> store -> per-slot statistics partial), one replica per lane, state
//                       in registers.  The paper's literal mapping is one replica per CTA
//                       (P:71); for single-agent envs that would leave 31/32 lanes idle, so
//                       32 replicas share a warp (DESIGN R1) -- results are identical because
//                       replicas never interact.
//  k_rollout_tag        A7 for the multi-agent tag env: one CTA per replica, one thread per
//                       agent, agents interact through a shared-memory cell grid.
//  k_sample_*/k_step_*  the single-step calls ws_sample / ws_step.
//  k_reset_*            ws_reset.
//  statistics (A8)      exact fixed-point per-slot sums accumulated in place by integer
//                       atomics (no separate reduction kernel).
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "envs.cuh"
#include "kernels.h"
#include "sampler.cuh"

#ifndef WS_EXP
#define WS_EXP 0  // profiling experiment bits (compile-time; 0 in production)
#endif

namespace ws {

// =======================================================================================
// Per-env adapters for the lane kernels: state I/O, reset draws, observation, action type.
// =======================================================================================
template <class Env>
struct Lane;

template <>
struct Lane<CartPole> {
  using Env = CartPole;
  using St = CartPole::St;
  static constexpr bool kDiscrete = true;
  static constexpr int N = 2, D = 4, S = 4, kDim = 1;
  __device__ static void load(const float* p, St& s) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    s = St{v.x, v.y, v.z, v.w};
  }
  __device__ static void save(float* p, const St& s) {
    *reinterpret_cast<float4*>(p) = make_float4(s.x, s.xd, s.th, s.thd);
  }
  __device__ static void init(const Key& k, uint32_t eg, uint32_t rc, St& s) {
    const U4 b = block(k, rc, eg, 0, kReset);  // draws j = rc*4 + i -> block rc
    CartPole::init(s, b.x, b.y, b.z, b.w);
  }
  __device__ static void obs_store(float* dst, const St& s, bool cs) {
    const float4 v = make_float4(s.x, s.xd, s.th, s.thd);
    if (cs) st_cs(reinterpret_cast<float4*>(dst), v); else *reinterpret_cast<float4*>(dst) = v;
  }
  template <bool kFast>
  __device__ static void step(St& s, int a, float& r, bool& term) { CartPole::step<kFast>(s, a, r, term); }
  // per-state cached data carried by the fused loop (none for CartPole)
  struct Aux {};
  __device__ static Aux aux_of(const St&) { return Aux{}; }
  template <bool kFast>
  __device__ static void step_aux(St& s, Aux&, int a, float& r, bool& term) { step<kFast>(s, a, r, term); }
  __device__ static void obs_store_aux(float* dst, const St& s, const Aux&, bool cs) { obs_store(dst, s, cs); }
  __device__ static Aux select(bool p, const Aux& x, const Aux&) { return x; }
  __device__ static void obs_vals(const St& s, const Aux&, float (&o)[4]) {
    o[0] = s.x; o[1] = s.xd; o[2] = s.th; o[3] = s.thd;
  }
  __device__ static bool valid(int a) { return CartPole::valid(a); }
  // natural episodes last >= 8 steps (tests/test_oracle_envs.py::test_cartpole_min_episode_length)
  static constexpr int kMinEpisode = 8;
  static constexpr bool kRolled = false;
  // two builds of the fused roll-out (section 5): latency (few warps: unconstrained registers for
  // the deepest schedule) and throughput (many warps: register budget for occupancy)
  static constexpr int kMaxThreads = 256;
  static constexpr int kWinRowsLat = 32, kWinRowsThr = 32, kMinBlocksThr = 0;  // 0: no register cap hint
  __device__ static bool fast_ok(const St& s) { return CartPole::fast_ok(s); }
};

template <>
struct Lane<Acrobot> {
  using St = Acrobot::St;
  static constexpr bool kDiscrete = true;
  static constexpr int N = 3, D = 6, S = 4, kDim = 1;
  __device__ static void load(const float* p, St& s) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    s = St{v.x, v.y, v.z, v.w};
  }
  __device__ static void save(float* p, const St& s) {
    *reinterpret_cast<float4*>(p) = make_float4(s.t1, s.t2, s.w1, s.w2);
  }
  __device__ static void init(const Key& k, uint32_t eg, uint32_t rc, St& s) {
    const U4 b = block(k, rc, eg, 0, kReset);
    Acrobot::init(s, b.x, b.y, b.z, b.w);
  }
  // obs = (cos t1, sin t1, cos t2, sin t2, w1, w2) (gym Acrobot-v1)
  __device__ static void obs_store(float* dst, const St& s, bool cs) {
    float s1, c1, s2, c2;
    sincos_c<false>(s.t1, s1, c1);  // wrapped angles: |t| <= pi
    sincos_c<false>(s.t2, s2, c2);
    const float2 a = make_float2(c1, s1), b = make_float2(c2, s2), c = make_float2(s.w1, s.w2);
    float2* d = reinterpret_cast<float2*>(dst);
    if (cs) { st_cs(d, a); st_cs(d + 1, b); st_cs(d + 2, c); }
    else { d[0] = a; d[1] = b; d[2] = c; }
  }
  template <bool kFast>
  __device__ static void step(St& s, int a, float& r, bool& term) { Acrobot::step(s, a, r, term); }
  // the fused loop carries each state's trigonometry: it serves the pre-step observation,
  // the first RK4 stage and (computed for the new state) the terminal test -- 12 instead of
  // 16 fp64 sincos evaluations per step
  using Aux = Acrobot::Trig;
  __device__ static Aux aux_of(const St& s) { return Acrobot::trig_of(s); }
  template <bool kFast>
  __device__ static void step_aux(St& s, Aux& tr, int a, float& r, bool& term) { Acrobot::step_trig(s, tr, a, r, term); }
  __device__ static void obs_store_aux(float* dst, const St& s, const Aux& t, bool cs) {
    const float2 a = make_float2(t.c1, t.s1), b = make_float2(t.c2, t.s2), c = make_float2(s.w1, s.w2);
    float2* d = reinterpret_cast<float2*>(dst);
    if (cs) { st_cs(d, a); st_cs(d + 1, b); st_cs(d + 2, c); }
    else { d[0] = a; d[1] = b; d[2] = c; }
  }
  __device__ static Aux select(bool p, const Aux& x, const Aux& y) {
    return Aux{p ? x.s1 : y.s1, p ? x.c1 : y.c1, p ? x.s2 : y.s2, p ? x.c2 : y.c2, p ? x.s12 : y.s12, p ? x.c12 : y.c12};
  }
  __device__ static void obs_vals(const St& s, const Aux& t, float (&o)[6]) {
    o[0] = t.c1; o[1] = t.s1; o[2] = t.c2; o[3] = t.s2; o[4] = s.w1; o[5] = s.w2;
  }
  __device__ static bool valid(int a) { return Acrobot::valid(a); }
  static constexpr int kMinEpisode = 1;  // no proven bound: keep the per-step reset check
  static constexpr bool kRolled = true;  // ~1000-instruction step: a rolled loop keeps the I-cache warm
  // throughput build: an 8-row statistics window and <= 96 registers (5 resident CTAs of 128
  // threads per SM, no spills); latency build: 32 rows, unconstrained registers
  static constexpr int kMaxThreads = 128;
#ifndef WS_ACRO_MINB
#define WS_ACRO_MINB 5  // 96 registers, no spills (6: 80 with spills; C3a 3.00 -> 2.94 ms, C3S 10.2 -> 9.9 ms)
#endif
  static constexpr int kWinRowsLat = 32, kWinRowsThr = 8, kMinBlocksThr = WS_ACRO_MINB;
  __device__ static bool fast_ok(const St&) { return true; }
};

// Dummy (S:164 calibration env): constant zero observation, reward 1, truncation only.
struct Dummy {
  struct St {};
};
template <>
struct Lane<Dummy> {
  using St = Dummy::St;
  static constexpr bool kDiscrete = true;
  static constexpr int N = 2, D = 4, S = 0, kDim = 1;
  __device__ static void load(const float*, St&) {}
  __device__ static void save(float*, const St&) {}
  __device__ static void init(const Key&, uint32_t, uint32_t, St&) {}
  __device__ static void obs_store(float* dst, const St&, bool cs) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    if (cs) st_cs(reinterpret_cast<float4*>(dst), z); else *reinterpret_cast<float4*>(dst) = z;
  }
  template <bool kFast>
  __device__ static void step(St&, int, float& r, bool& term) {
    r = 1.0f;
    term = false;
  }
  struct Aux {};
  __device__ static Aux aux_of(const St&) { return Aux{}; }
  template <bool kFast>
  __device__ static void step_aux(St& s, Aux&, int a, float& r, bool& term) { step<kFast>(s, a, r, term); }
  __device__ static void obs_store_aux(float* dst, const St& s, const Aux&, bool cs) { obs_store(dst, s, cs); }
  __device__ static Aux select(bool p, const Aux& x, const Aux&) { return x; }
  __device__ static void obs_vals(const St&, const Aux&, float (&o)[4]) { o[0] = o[1] = o[2] = o[3] = 0.0f; }
  __device__ static bool valid(int a) { return a == 0 || a == 1; }
  static constexpr int kMinEpisode = 1 << 30;  // episodes end by truncation only
  static constexpr bool kRolled = false;
  static constexpr int kMaxThreads = 256;
  static constexpr int kWinRowsLat = 32, kWinRowsThr = 32, kMinBlocksThr = 0;  // 0: no register cap hint
  __device__ static bool fast_ok(const St&) { return true; }
};

template <>
struct Lane<Pendulum> {
  using St = Pendulum::St;
  static constexpr bool kDiscrete = false;
  static constexpr int N = 0, D = 3, S = 2, kDim = 1;
  __device__ static void load(const float* p, St& s) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    s = St{v.x, v.y};
  }
  __device__ static void save(float* p, const St& s) {
    *reinterpret_cast<float2*>(p) = make_float2(s.th, s.thd);
  }
  __device__ static void init(const Key& k, uint32_t eg, uint32_t rc, St& s) {
    const U4 b = block(k, rc >> 1, eg, 0, kReset);  // draws j = rc*2 + i
    if (rc & 1) Pendulum::init(s, b.z, b.w); else Pendulum::init(s, b.x, b.y);
  }
  // obs = (cos th, sin th, thdot)
  __device__ static void obs_store(float* dst, const St& s, bool cs) {
    float sn, c;
    sincos_c(s.th, sn, c);
    if (cs) { st_cs(dst, c); st_cs(dst + 1, sn); st_cs(dst + 2, s.thd); }
    else { dst[0] = c; dst[1] = sn; dst[2] = s.thd; }
  }
  // returns false on a non-finite action
  __device__ static bool step_c(St& s, const float (&a)[1], float& r, bool& term) {
    if (!isfinite(a[0])) return false;
    Pendulum::step(s, a[0], r);
    term = false;
    return true;
  }
};

template <int DD>
struct Lane<Surface<DD>> {
  using Env = Surface<DD>;
  using St = typename Env::St;
  static constexpr bool kDiscrete = false;
  static constexpr int N = 0, D = DD + 1, S = DD, kDim = DD;
  __device__ static void load(const float* p, St& s) {
#pragma unroll
    for (int i = 0; i < DD; ++i) s.q[i] = p[i];
    s.E = Env::energy(s.q);
  }
  __device__ static void save(float* p, const St& s) {
#pragma unroll
    for (int i = 0; i < DD; ++i) p[i] = s.q[i];
  }
  // R11/R23: q_i = start_i + (-0.05 + 0.1 u_i), draws j = rc*D + i
  __device__ static void init(const Key& k, uint32_t eg, uint32_t rc, St& s) {
    const uint64_t j0 = (uint64_t)rc * DD;
    U4 b = block(k, j0 >> 2, eg, 0, kReset);
    uint64_t cur = j0 >> 2;
#pragma unroll
    for (int i = 0; i < DD; ++i) {
      const uint64_t j = j0 + i;
      if ((j >> 2) != cur) {
        cur = j >> 2;
        b = block(k, cur, eg, 0, kReset);
      }
      s.q[i] = Env::start(i) + (-0.05f + 0.1f * u01(pick(b, (uint32_t)(j & 3))));
    }
    s.E = Env::energy(s.q);
  }
  __device__ static void obs_store(float* dst, const St& s, bool cs) {
#pragma unroll
    for (int i = 0; i < DD; ++i) {
      if (cs) st_cs(dst + i, s.q[i]); else dst[i] = s.q[i];
    }
    if (cs) st_cs(dst + DD, s.E); else dst[DD] = s.E;
  }
  __device__ static bool step_c(St& s, const float (&a)[DD], float& r, bool& term) {
    return Env::step(s, a, r, term);
  }
};

// =======================================================================================
// Continuous-head sampling for one agent (R14): act_k = mean_k + exp(log_std_k) z_k,
// logp = sum_k (-z_k^2/2 - log_std_k - log(2 pi)/2) in fp64, rounded once.
// =======================================================================================
template <int DIM>
__device__ __forceinline__ bool gauss_sample(const Key& key, uint32_t eg, uint32_t agent, uint64_t t,
                                             const float (&mean)[DIM], const float (&log_std)[DIM],
                                             float (&act)[DIM], float& logp) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < DIM; ++k) ok = ok && isfinite(mean[k]) && isfinite(log_std[k]);
  double lp = 0.0;
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    const float z = gauss_z(key, eg, agent, t * (uint64_t)DIM + (uint64_t)k);
    const float sd = (float)exp((double)log_std[k]);
    act[k] = ok ? mean[k] + sd * z : __int_as_float(0x7fc00000);
    lp = lp + (((-0.5 * (double)z) * (double)z - (double)log_std[k]) - kHalfLog2Pi);
  }
  logp = ok ? (float)lp : __int_as_float(0x7fc00000);
  return ok;
}

// =======================================================================================
// A8: per-warp statistics window in shared memory.  Each lane records its per-slot
// contribution (done ? episode length : 0, done ? episode return : 0, reward; the float
// ones in 2^-32 fixed point) in row (slot & 31); every 32 slots (and at the end) lane i
// reduces row i over the 32 lanes and adds the slot's four integers to stats[slot] with
// integer atomics -- exact and order-independent.  Row strides (36 words, 34 int64) keep
// rows 16-byte aligned and the quarter-warp phases of LDS.128 free of bank conflicts.
// =======================================================================================
constexpr int kWinStride = 36;
constexpr int kWinWords = 3 * 32 * kWinStride;  // per warp (13.5 KiB)
#ifndef WS_CONT_WIN_ROWS
#define WS_CONT_WIN_ROWS 16
#endif
constexpr int kContWinRows = WS_CONT_WIN_ROWS;  // window depth of k_rollout_continuous
#ifndef WS_SURF_TRIP
#define WS_SURF_TRIP 8  // surface-D fast-trip length (D % 4 == 0); <= the 16-row statistics window
#endif

struct StatsWindow {
  uint32_t* len;
  float* ret;
  float* rew;
  // rows: the window depth (32, or fewer where the shared-memory footprint limits occupancy)
  __device__ __forceinline__ void init(uint32_t* base, int rows = 32) {
    len = base;
    ret = reinterpret_cast<float*>(base + rows * kWinStride);
    rew = reinterpret_cast<float*>(base + 2 * rows * kWinStride);
  }
  __device__ __forceinline__ void put(int row, int lane, uint32_t l, float rt, float rw) {
    len[row * kWinStride + lane] = l;
    ret[row * kWinStride + lane] = rt;
    rew[row * kWinStride + lane] = rw;
  }
  // rows [row_lo, row_hi] -> stats of slots slot0 + row (row 0 may precede the roll-out's
  // first slot, hence the signed slot0); lanes >= nlive are shadow lanes and are ignored.
  // Each value is converted to 2^-32 fixed point before the integer sums (R20).
  __device__ __forceinline__ void flush(int lane, int row_lo, int row_hi, int64_t slot0, unsigned long long* stats,
                                        int nlive = 32) {
    if (nlive <= 0) return;  // (fully dead warps exit at kernel entry; defensive)
    __syncwarp();
    if (nlive < 32) {  // tail warp: zero the shadow lanes' columns (they duplicate replica E-1)
      for (int r = row_lo; r <= row_hi; ++r)
        if (lane >= nlive) put(r, lane, 0u, 0.0f, 0.0f);
      __syncwarp();
    }
    if (lane >= row_lo && lane <= row_hi) {
      const uint4* l4 = reinterpret_cast<const uint4*>(len + lane * kWinStride);
      const float4* t4 = reinterpret_cast<const float4*>(ret + lane * kWinStride);
      const float4* r4 = reinterpret_cast<const float4*>(rew + lane * kWinStride);
      unsigned long long nd = 0, ln = 0;
      long long rt = 0, rs = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 v = l4[j];
        nd += (v.x != 0) + (v.y != 0) + (v.z != 0) + (v.w != 0);
        ln += (unsigned long long)v.x + v.y + v.z + v.w;
        const float4 t = t4[j], r = r4[j];
        rt += to_fx(t.x) + to_fx(t.y) + to_fx(t.z) + to_fx(t.w);
        rs += to_fx(r.x) + to_fx(r.y) + to_fx(r.z) + to_fx(r.w);
      }
      if (cta_acc) {  // CTA-level aggregation in shared memory (pushed by CtaStats::push)
        unsigned long long* acc = cta_acc + lane * 4;
        if (nd) atomicAdd(acc + kStEpisodes, nd);
        if (rt) atomicAdd(acc + kStReturn, (unsigned long long)rt);
        if (ln) atomicAdd(acc + kStLength, ln);
        if (rs) atomicAdd(acc + kStReward, (unsigned long long)rs);
      } else {
        unsigned long long* st = stats + (size_t)(slot0 + lane) * 4;
        if (nd) atomicAdd(st + kStEpisodes, nd);
        if (rt) atomicAdd(st + kStReturn, (unsigned long long)rt);
        if (ln) atomicAdd(st + kStLength, ln);
        if (rs) atomicAdd(st + kStReward, (unsigned long long)rs);
      }
    }
    __syncwarp();
  }
  unsigned long long* cta_acc = nullptr;  // [32 rows][4] when aggregating per CTA
};

// Per-CTA statistics accumulator: the warps of a CTA add their window rows into a shared
// [2][32][4] u64 buffer (double-buffered by window parity); after a named barrier over the
// CTA's live warps, its first warp adds the 32 rows to the global stats with one atomic per
// field and row, then clears the buffer -- 1/(warps per CTA) of the global atomics.
struct CtaStats {
  unsigned long long* buf;  // [2][32][4]
  int n_live_threads;       // live warps x 32
  bool leader;              // first warp of the CTA
  __device__ __forceinline__ unsigned long long* acc(int window) { return buf + (window & 1) * 128; }
  __device__ __forceinline__ void push(int lane, int window, int row_lo, int row_hi, int64_t slot0,
                                       unsigned long long* stats) {
    asm volatile("bar.sync 1, %0;" ::"r"(n_live_threads) : "memory");
    if (leader && lane >= row_lo && lane <= row_hi) {
      unsigned long long* a = acc(window) + lane * 4;
      unsigned long long* st = stats + (size_t)(slot0 + lane) * 4;
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        if (a[f]) atomicAdd(st + f, a[f]);
        a[f] = 0ull;
      }
    }
  }
};

__device__ __forceinline__ uint32_t* warp_window() {
  extern __shared__ __align__(16) uint32_t ws_smem[];
  return ws_smem + (threadIdx.x >> 5) * kWinWords;
}
// CTA accumulator at the start of dynamic shared memory (kernels without per-warp windows)
__device__ __forceinline__ unsigned long long* cta_stats_buf_only() {
  extern __shared__ __align__(16) uint32_t ws_smem[];
  return reinterpret_cast<unsigned long long*>(ws_smem);
}
// the [2][32][4] u64 CTA accumulator follows the per-warp windows
__device__ __forceinline__ unsigned long long* cta_stats_buf() {
  extern __shared__ __align__(16) uint32_t ws_smem[];
  return reinterpret_cast<unsigned long long*>(ws_smem + (blockDim.x >> 5) * kWinWords);
}

// =======================================================================================
// A2 for the fused roll-out of discrete single-agent envs: the "plan" kernel.
//
// With GIVEN probabilities (BJ:5) the sampled action of (replica e, step t) depends only on
// the seed, e, t and the probability row -- never on the environment state -- so all T x E
// draws are sampled up front by this full-occupancy kernel (thread = one replica x 64
// steps), leaving only the inherently sequential dynamics on the latency-bound roll-out
// kernel.  It writes the act and logp slabs of the store directly and a compact plan
// (four 8-bit actions of slots 4j..4j+3 per u32, 0xFF = invalid row) that the dynamics
// kernel reads back with prefetched 32-bit loads.
// =======================================================================================
#ifndef WS_PLAN_CHUNK
#define WS_PLAN_CHUNK 128
#endif
constexpr int kPlanChunk = WS_PLAN_CHUNK;  // steps per plan thread (thresholds amortised over the chunk)

// One warp's share of the plan: the 32 consecutive replicas starting at e - lane (lane =
// threadIdx.x & 31), steps [c_begin, c_end) -- every lane of the warp must call it (the CDF of
// the probability rows is a warp scan).
template <int N, bool kStrided>
__device__ __forceinline__ void plan_rows(const KArgs& a, const int T, const uint64_t t0, const float* __restrict__ probs,
                                          const int64_t row_stride, const int64_t step_stride, const int64_t e,
                                          const int c_begin, const int c_end) {
  const int lane = threadIdx.x & 31;
  const int64_t E = a.E;
  const bool live = e < E;
  const int64_t ec = live ? e : E - 1;  // tail lanes duplicate replica E-1 (identical stores)
  const uint32_t eg = (uint32_t)(a.offset + ec);
  const Key key{a.k0, a.k1};
  const bool wlogp = a.write_logp != 0;
  int32_t* const p_act = reinterpret_cast<int32_t*>(a.act) + ec;
  float* const p_logp = a.logp + ec;
  uint32_t* const p_plan = a.plan + ec;

  Thresholds<N> th;
  if constexpr (!kStrided) {
    RowCDF<N> cdf;
    warp_row_cdf<N>(probs, row_stride, e - lane, E, lane, cdf);
    make_thresholds<N>(cdf, th);
  }
  bool any_bad = false;
  auto sample = [&](const int c, const uint32_t word, float& lp) {
    int act;
    bool bad;
    if constexpr (!kStrided) {
      act = search_k<N>(th, word >> 8, lp);
      bad = th.bad;
    } else {
      RowCDF<N> cdf;
      warp_row_cdf<N>(probs + (int64_t)c * step_stride, row_stride, e - lane, E, lane, cdf);
      bad = cdf.bad;
      act = search<N>(cdf, u01(word));
      lp = logp_of<N>(cdf, act);
    }
    if (bad) {
      act = -1;
      lp = __int_as_float(0x7fc00000);
    }
    any_bad |= bad;
    return act;
  };
  const size_t sE = (size_t)E;
  if ((t0 & 3) == 0) {
    // aligned: one Philox4x32 call per 4-slot group (ACTION draws j = t)
    const int g_end = c_end >> 2;  // full groups
    const KeySchedule ks = key_schedule(key.k0, key.k1);
    for (int g = c_begin >> 2; g < g_end; ++g) {
      const U4 w = philox_ks((uint32_t)((t0 >> 2) + (uint64_t)g), eg, 0, kAction, ks);
      const size_t base = (size_t)(4 * g) * sE;
      float lp0, lp1, lp2, lp3;
      const int a0 = sample(4 * g, w.x, lp0), a1 = sample(4 * g + 1, w.y, lp1);
      const int a2 = sample(4 * g + 2, w.z, lp2), a3 = sample(4 * g + 3, w.w, lp3);
      st_cs(p_act + base, a0);
      st_cs(p_act + base + sE, a1);
      st_cs(p_act + base + 2 * sE, a2);
      st_cs(p_act + base + 3 * sE, a3);
      if (wlogp) {
        st_cs(p_logp + base, lp0);
        st_cs(p_logp + base + sE, lp1);
        st_cs(p_logp + base + 2 * sE, lp2);
        st_cs(p_logp + base + 3 * sE, lp3);
      }
      p_plan[(size_t)g * sE] = (uint32_t)(a0 & 0xFF) | ((uint32_t)(a1 & 0xFF) << 8) |
                               ((uint32_t)(a2 & 0xFF) << 16) | ((uint32_t)(a3 & 0xFF) << 24);
    }
    if ((c_end & 3) != 0) {  // partial last group
      const int c0 = c_end & ~3;
      const U4 w = block(key, (t0 >> 2) + (uint64_t)(c0 >> 2), eg, 0, kAction);
      uint32_t pack = 0;
      for (int c = c0; c < c_end; ++c) {
        float lp;
        const int act = sample(c, pick(w, (uint32_t)(c & 3)), lp);
        st_cs(p_act + (size_t)c * sE, act);
        if (wlogp) st_cs(p_logp + (size_t)c * sE, lp);
        pack |= (uint32_t)(act & 0xFF) << (8 * (c & 3));
      }
      p_plan[(size_t)(c0 >> 2) * sE] = pack;
    }
  } else {
    uint32_t pack = 0;
    for (int c = c_begin; c < c_end; ++c) {
      const uint64_t t = t0 + (uint64_t)c;
      float lp;
      const int act = sample(c, pick(block(key, t >> 2, eg, 0, kAction), (uint32_t)(t & 3)), lp);
      st_cs(p_act + (size_t)c * sE, act);
      if (wlogp) st_cs(p_logp + (size_t)c * sE, lp);
      pack |= (uint32_t)(act & 0xFF) << (8 * (c & 3));
      if ((c & 3) == 3 || c == c_end - 1) {
        p_plan[(size_t)(c >> 2) * sE] = pack;
        pack = 0;
      }
    }
  }
  if (live && any_bad) atomicOr(a.err, kErrProbs | kErrAction);
}

template <int N, bool kStrided>
__global__ void __launch_bounds__(128) k_plan_discrete(const KArgs a, const int T, const uint64_t t0,
                                                      const float* __restrict__ probs, const int64_t row_stride,
                                                      const int64_t step_stride, const int zero_stats) {
  // zero_stats: this launch also clears the roll-out's [T, 4] statistics slab (the roll-out kernel
  // runs after it on the same stream) -- one launch fewer than a separate memset
  if (zero_stats && blockIdx.x == 0 && blockIdx.y == 0)
    for (int i = threadIdx.x; i < 4 * T; i += blockDim.x) a.stats[i] = 0ull;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c_begin = blockIdx.y * kPlanChunk;
  plan_rows<N, kStrided>(a, T, t0, probs, row_stride, step_stride, e, c_begin, min(T, c_begin + kPlanChunk));
}

// =======================================================================================
// A7: fused roll-out, discrete single-agent envs (CartPole, Acrobot, Dummy).
//
// One replica per lane, state in registers for all T steps; actions come from the plan
// (loaded two 4-step blocks ahead).  The step is straight-line code:
//  - tail lanes of the last warp shadow replica E-1 (identical values, identical stores),
//    so no store is predicated and the statistics ignore them at flush time;
//  - the next reset state init(e, rc + 1) is kept ready in registers (look-ahead) and
//    selected on done; it is refilled once per 8 steps when the env's episodes provably
//    last >= 8 steps (kFast), else once per 4-step block with a warp-uniform slow path for
//    a second reset inside the block;
//  - blocks whose four actions are all valid (the common case) skip the invalid-row
//    bookkeeping (kClean);
//  - store addresses advance by one uniform slot stride per step.
// =======================================================================================
template <class Env, bool kLat>
struct DiscreteRunner {
  using L = Lane<Env>;
  using St = typename L::St;
  static constexpr int kRows = kLat ? L::kWinRowsLat : L::kWinRowsThr;  // window depth (power of 2, <= 32)
  // per-lane constants
  int lane, nlive, max_steps, T;
  uint32_t eg;
  Key key;
  size_t sE;
  float* p_obs;
  float* p_rew;
  uint8_t* p_done;
  const uint32_t* p_plan;
  unsigned long long* p_stats;
  CtaStats cta;
  StatsWindow win;
  // replica state (registers)
  St s, nxt;
  typename L::Aux aux, aux_nxt;  // per-state cached data (Acrobot: trigonometry)
  int32_t ep_step;
  uint32_t rc;
  float ep_ret;
  bool stale;

  static __device__ __forceinline__ int act_of(uint32_t pk, int k) { return (int)(int8_t)(uint8_t)(pk >> (8 * k)); }

  __device__ __forceinline__ uint32_t ld(int j) const {
    return j < (T + 3) / 4 ? __ldg(p_plan + (size_t)j * sE) : 0u;
  }
  __device__ __forceinline__ void refill() {
    if (!(WS_EXP & 8)) L::init(key, eg, rc + 1, nxt);
    aux_nxt = L::aux_of(nxt);
    stale = false;
  }
  __device__ __forceinline__ void flush_after(int c_last) {
    if ((c_last & (kRows - 1)) == kRows - 1 || c_last == T - 1) {
      const int w = c_last / kRows;
      // latency build of the straight-line envs (few warps, each alone on its scheduler): every
      // warp adds its window to the global statistics itself -- a CTA barrier would make the four
      // warps wait for the slowest every window (measured: C2 roll-out 0.170 -> 0.160 ms without
      // it; the rolled Acrobot loop measured 0.750 -> 0.771 ms, so it keeps the CTA path);
      // throughput build: CTA aggregation first (a quarter of the atomics on the slot's words)
      if ((kLat && !L::kRolled) || (WS_EXP & 64)) {
        win.cta_acc = nullptr;
        win.flush(lane, 0, c_last & (kRows - 1), c_last & ~(kRows - 1), p_stats, nlive);
      } else {
        win.cta_acc = cta.acc(w);
        win.flush(lane, 0, c_last & (kRows - 1), c_last & ~(kRows - 1), p_stats, nlive);
        cta.push(lane, w, 0, c_last & (kRows - 1), c_last & ~(kRows - 1), p_stats);
      }
    }
  }

  // one fused step at slot c (store offset idx = c * E)
  template <bool kFast, bool kClean>
  __device__ __forceinline__ void step(const int c, const size_t idx, const int act_in) {
    const bool bad = kClean ? false : act_in < 0;  // invalid probability row (plan byte 0xFF)
    // ---- A6 log the pre-step observation (R12)
    if (!(WS_EXP & 4)) L::obs_store_aux(p_obs + idx * L::D, s, aux, true);
    // ---- A3 / A4 dynamics, reward, done
    St s2 = s;
    typename L::Aux aux2 = aux;
    float r;
    bool term;
    L::template step_aux<kFast || (WS_EXP & 1)>(s2, aux2, kClean ? act_in : (bad ? 0 : act_in), r, term);
    const int32_t es = ep_step + 1;
    uint32_t d = (term ? 1u : 0u) | (es >= max_steps ? 2u : 0u);
    float rw = r;
    if (!kClean) {
      d = bad ? 0u : d;
      rw = bad ? 0.0f : r;
    }
    const float ret = ep_ret + r;
    // ---- A5 auto-reset from the look-ahead state init(e, rc + 1)
    if (!kFast) {
      if (__any_sync(kFull, d != 0 && stale)) {  // second reset within one refill window
        if (d != 0 && stale) {
          L::init(key, eg, rc + 1, nxt);
          aux_nxt = L::aux_of(nxt);
        }
      }
    }
    if (kClean) {
      s = d ? nxt : s2;
      aux = L::select(d != 0, aux_nxt, aux2);
      ep_step = d ? 0 : es;
      ep_ret = d ? 0.0f : ret;
    } else {
      aux = L::select(d != 0, aux_nxt, L::select(bad, aux, aux2));
      s = d ? nxt : (bad ? s : s2);
      ep_step = d ? 0 : (bad ? ep_step : es);
      ep_ret = d ? 0.0f : (bad ? ep_ret : ret);
    }
    stale = stale || d != 0;
    rc += d ? 1u : 0u;
    if (!(WS_EXP & 4)) {
      st_cs(p_rew + idx, rw);
      st_cs_u8(p_done + idx, (uint8_t)d);
    }
    // ---- A8 per-slot statistics contribution
    if (!(WS_EXP & 2)) win.put(c & (kRows - 1), lane, d ? (uint32_t)es : 0u, d ? ret : 0.0f, rw);
  }

  template <bool kFast, bool kClean>
  __device__ __forceinline__ void body4(const int j, const uint32_t pk) {
    const size_t idx = (size_t)(4 * j) * sE;
    step<kFast, kClean>(4 * j, idx, act_of(pk, 0));
    step<kFast, kClean>(4 * j + 1, idx + sE, act_of(pk, 1));
    step<kFast, kClean>(4 * j + 2, idx + 2 * sE, act_of(pk, 2));
    step<kFast, kClean>(4 * j + 3, idx + 3 * sE, act_of(pk, 3));
  }
  // one 8-step trip = blocks j, j+1.  The validity vote comes first so that the look-ahead
  // refill and all eight steps form one straight-line basic block the scheduler can
  // interleave (refill Philox and each step's stores / statistics under the next step's
  // dynamics).
  template <bool kFast>
  __device__ __forceinline__ void trip8(const int j, const uint32_t p0, const uint32_t p1) {
    if (kFast && __all_sync(kFull, ((p0 | p1) & 0x80808080u) == 0u)) {
      refill();
      body4<kFast, true>(j, p0);
      body4<kFast, true>(j + 1, p1);
    } else {
      refill();
      body4<false, false>(j, p0);
      refill();
      body4<false, false>(j + 1, p1);
    }
    flush_after(4 * j + 7);
  }

  // rolled loop for envs whose step is long (Acrobot: RK4 with 12 fp64 sincos): one step body
  // in the instruction stream instead of eight, so the loop stays resident in the instruction
  // cache; the same refill-per-4-steps and second-reset logic as the trips' slow path
  __device__ __forceinline__ void run_rolled() {
    const int ng = (T + 3) / 4;
    uint32_t A = ld(0);
#pragma unroll 1
    for (int j = 0; j < ng; ++j) {
      const uint32_t p = A;
      A = ld(j + 1);
      refill();
      const int n = min(4, T - 4 * j);
#pragma unroll 1
      for (int k = 0; k < n; ++k) {
        const int c = 4 * j + k;
        step<false, false>(c, (size_t)c * sE, act_of(p, k));
        flush_after(c);
      }
    }
  }

  template <bool kFast>
  __device__ __forceinline__ void run() {
    if constexpr (L::kRolled) {
      run_rolled();
      return;
    }
    const int nfull = T >> 2;  // full 4-step blocks
    uint32_t A0 = ld(0), A1 = ld(1);
    int j = 0;
    for (; j + 2 <= nfull; j += 2) {  // 8 steps per trip; static prefetch registers
      const uint32_t p0 = A0, p1 = A1;
      A0 = ld(j + 2);
      A1 = ld(j + 3);
      trip8<kFast>(j, p0, p1);
    }
    if (j < nfull) {
      refill();
      body4<false, false>(j, A0);
      flush_after(4 * j + 3);
      ++j;
    }
    for (int c = 4 * j; c < T; ++c) {  // tail (T % 4 steps)
      step<false, false>(c, (size_t)c * sE, act_of(ld(c >> 2), c & 3));
      flush_after(c);
    }
  }
};

template <class Env, bool kLat>
__device__ __forceinline__ void rollout_discrete_body(const KArgs& a, const int T) {
  using L = Lane<Env>;
  using Run = DiscreteRunner<Env, kLat>;
  constexpr int kWin = 3 * Run::kRows * kWinStride;  // window words per warp
  extern __shared__ __align__(16) uint32_t ws_smem[];
  Run R;
  R.lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = a.E;
  if (e - R.lane >= E) return;  // whole warp past the last replica (its partial part would not exist)
  const bool live = e < E;
  const int64_t ec = live ? e : E - 1;  // tail lanes shadow replica E-1 (identical stores)
  R.nlive = (int)min((int64_t)32, E - (e - R.lane));
  R.eg = (uint32_t)(a.offset + ec);
  R.key = Key{a.k0, a.k1};
  R.max_steps = a.max_steps;
  R.T = T;
  R.sE = (size_t)E;
  R.win.init(ws_smem + (threadIdx.x >> 5) * kWin, Run::kRows);
  R.p_obs = a.obs + ec * L::D;
  R.p_rew = a.rew + ec;
  R.p_done = a.done + ec;
  R.p_plan = a.plan + ec;
  R.p_stats = a.stats;
  {
    const int64_t cta_first = (int64_t)blockIdx.x * blockDim.x;
    const int64_t live_thr = min((int64_t)blockDim.x, ((E - cta_first + 31) / 32) * 32);
    R.cta.buf = reinterpret_cast<unsigned long long*>(ws_smem + (blockDim.x >> 5) * kWin);
    R.cta.n_live_threads = (int)live_thr;
    R.cta.leader = (threadIdx.x >> 5) == 0;
    for (int i = threadIdx.x; i < 256; i += (int)live_thr) R.cta.buf[i] = 0ull;  // live threads only
    asm volatile("bar.sync 1, %0;" ::"r"(R.cta.n_live_threads) : "memory");
  }
  L::load(a.state + ec * L::S, R.s);
  R.ep_step = a.ep_step[ec];
  R.rc = a.reset_count[ec];
  R.ep_ret = a.ep_ret[ec];
  L::init(R.key, R.eg, R.rc + 1, R.nxt);
  R.aux = L::aux_of(R.s);
  R.aux_nxt = L::aux_of(R.nxt);
  R.stale = false;

  // Fast path: one look-ahead reset refill per 8-step trip needs every episode that starts at a
  // reset to last >= 8 steps -- proven for CartPole over the whole R11 reset box and all action
  // sequences by interval arithmetic (tests/test_oracle_envs.py::
  // test_cartpole_min_episode_proof_over_reset_box); truncation needs max_steps >= 8.
  const bool fast = L::kMinEpisode >= 8 && R.max_steps >= 8 && __all_sync(kFull, L::fast_ok(R.s));
  if (fast) R.template run<true>(); else R.template run<false>();

  if (live) {
    L::save(a.state + e * L::S, R.s);
    a.ep_step[e] = R.ep_step;
    a.reset_count[e] = R.rc;
    a.ep_ret[e] = R.ep_ret;
    L::obs_store(a.obs_live + e * L::D, R.s, false);
  }
}

template <class Env, bool kLat>
// latency build: minBlocks 1 lets ptxas spend registers on a deeper schedule (C2 measured:
// 174 registers, 0.180 ms vs 100 registers, 0.200 ms); throughput build: the env's budget
__global__ void __launch_bounds__(Lane<Env>::kMaxThreads, kLat ? 1 : Lane<Env>::kMinBlocksThr)
    k_rollout_discrete(const KArgs a, const int T) {
  rollout_discrete_body<Env, kLat>(a, T);
}

// R29' second-layer output evaluated in one lane: b + ((P_0 + P_1) + (P_2 + P_3)), P_q the fma
// chain from +0 over the q-th quarter of the hidden units (column w with row stride `stride`)
template <int H>
__device__ __forceinline__ float quarter_dot(const float* w, int stride, const float (&h)[H], float b) {
  constexpr int HQ = H / 4;
  float P[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float acc = 0.0f;
#pragma unroll
    for (int u = 0; u < HQ; ++u) acc = __fmaf_rn(w[(q * HQ + u) * stride], h[q * HQ + u], acc);
    P[q] = acc;
  }
  return fadd(b, fadd(fadd(P[0], P[1]), fadd(P[2], P[3])));
}

// =======================================================================================
// NEXT-N1: fused roll-out with in-kernel policy inference ("operating an agent that
// samples actions", "roll-outs, action inference, reset and training" on one GPU store),
// warp-specialised: a CTA of six warps serves 32 replicas (lane = replica).  Warp 0 is the ENV
// warp: it owns the states, publishes the pre-step observations to shared memory, and once
// the inference round is back it combines the four quarter partials (R29': b2 + ((P_0 + P_1) +
// (P_2 + P_3))), draws the action, steps the dynamics (the env's fast path when every lane
// satisfies its invariant) and publishes the next observation.  Warps 1..4 are INFERENCE warps:
// warp 1 + q evaluates hidden quarter q (weights broadcast from shared memory).  Warp 5 is the
// STORE warp: the log-probability (fp64 log), the stores and the statistics of each step, from
// a hand-off record, beside the env warp's next step.  Auto-reset uses a look-ahead state
// init(e, rc + 1) kept in registers and refilled after the record is handed over.  The critic's
// values_trunc (rare) and bootstrap values are evaluated in the env warp (R29' quarter sums
// in-lane).  (Round 2 history: one lane per replica 1.67 ms; env + 4 inference warps 1.18 ms;
// two pipelined replica groups per env warp 2.45 ms, not adopted.)
template <int D, int N>
struct PolicyWsSmem {
  float obs[D][32];            // the env warp's published observations
  float part[4][N + 1][32];    // [quarter] partial logits (+ critic) of the inference warps
  // the step handed from the env warp to the store warp (lane-indexed, conflict-free)
  float po[D][32];             // pre-step observation
  float pa[32], pvv[32], prw[32], pret[32];
  double pcN[32];
  int pact[32], pes[32];
  uint32_t pd[32];
};

// Warp-specialised policy roll-out, 32 replicas per CTA of six warps.  ENV warp (0): the
// recurrence -- partial logits -> softmax -> R13 draw -> dynamics -> auto-reset -> next observation
// published.  INFERENCE warps (1..4): warp 1+q evaluates R29''s hidden quarter q.  STORE warp (5):
// everything that only feeds the store -- the fp64 log of the log-probability, the act / logp /
// obs / value / rew / done stores and the statistics window -- from a per-step hand-off record in
// shared memory, so it runs beside the env warp's next step.  Named barriers: 1 obs ready,
// 2 partials ready (env + inference warps), 5 record written, 6 record read (env + store warp).
template <class Env, int H, bool kCritic>
__global__ void __launch_bounds__(192) k_rollout_policy_ws(const KArgs a, const int T, const uint64_t t0,
                                                          const float* __restrict__ weights,
                                                          float* __restrict__ values, float* __restrict__ bootstrap,
                                                          float* __restrict__ values_trunc) {
  using L = Lane<Env>;
  using St = typename L::St;
  constexpr int D = L::D, N = L::N, HQ = H / 4;
  constexpr int NW = D * H + H + H * N + N + (kCritic ? H + 1 : 0);
  constexpr int kRows = 16;
  __shared__ __align__(16) float sw[NW];
  __shared__ __align__(16) PolicyWsSmem<D, N> x;
  extern __shared__ __align__(16) uint32_t ws_smem[];  // the store warp's statistics window
  for (int i = threadIdx.x; i < NW; i += blockDim.x) sw[i] = weights[i];
  __syncthreads();
  const float* W1 = sw;
  const float* b1 = W1 + D * H;
  const float* W2 = b1 + H;
  const float* b2 = W2 + H * N;
  const float* wv = b2 + N;  // kCritic only
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t E = a.E;
  const size_t sE = (size_t)E;
  // the CTA's 32 replicas (tail lanes shadow replica E-1)
  const int64_t e_lane = (int64_t)blockIdx.x * 32 + lane;
  const bool live = e_lane < E;
  const int64_t ec = live ? e_lane : E - 1;

  if (warp >= 1 && warp <= 4) {  // ------------------------------------- inference warp, quarter q
    const int q = warp - 1;
    for (int t = 0; t < T; ++t) {
      asm volatile("bar.sync 1, 160;" ::: "memory");  // the observation of step t
      float o[D];
#pragma unroll
      for (int d = 0; d < D; ++d) o[d] = x.obs[d][lane];
      float P[N], Pv = 0.0f;
#pragma unroll
      for (int i = 0; i < N; ++i) P[i] = 0.0f;
#pragma unroll
      for (int u = 0; u < HQ; ++u) {
        const int j = q * HQ + u;
        float acc = b1[j];
#pragma unroll
        for (int d = 0; d < D; ++d) acc = __fmaf_rn(W1[d * H + j], o[d], acc);
        const float hj = acc > 0.0f ? acc : 0.0f;
#pragma unroll
        for (int i = 0; i < N; ++i) P[i] = __fmaf_rn(W2[j * N + i], hj, P[i]);
        if (kCritic) Pv = __fmaf_rn(wv[j], hj, Pv);
      }
#pragma unroll
      for (int i = 0; i < N; ++i) x.part[q][i][lane] = P[i];
      if (kCritic) x.part[q][N][lane] = Pv;
      asm volatile("bar.arrive 2, 160;" ::: "memory");
    }
    return;
  }

  if (warp == 5) {  // -------------------------------------------------------------- store warp
    StatsWindow win;
    win.init(ws_smem, kRows);
    const int nlive = (int)max((int64_t)0, min((int64_t)32, E - (int64_t)blockIdx.x * 32));
    for (int c = 0; c < T; ++c) {
      asm volatile("bar.sync 5, 64;" ::: "memory");  // the record of step c
      float o[D];
#pragma unroll
      for (int d = 0; d < D; ++d) o[d] = x.po[d][lane];
      const float pa = x.pa[lane], vv = x.pvv[lane], rw = x.prw[lane], ret = x.pret[lane];
      const double cN = x.pcN[lane];
      const int act = x.pact[lane], es = x.pes[lane];
      const uint32_t d = x.pd[lane];
      asm volatile("bar.arrive 6, 64;" ::: "memory");  // the record may be overwritten
      const size_t idx = (size_t)c * sE + (size_t)ec;
      if (kCritic && live) st_cs(values + idx, vv);
      float* po = a.obs + idx * D;
      if constexpr (D % 4 == 0) {
#pragma unroll
        for (int i = 0; i < D; i += 4) st_cs(reinterpret_cast<float4*>(po + i), make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]));
      } else if constexpr (D % 2 == 0) {
#pragma unroll
        for (int i = 0; i < D; i += 2) st_cs(reinterpret_cast<float2*>(po + i), make_float2(o[i], o[i + 1]));
      } else {
#pragma unroll
        for (int i = 0; i < D; ++i) st_cs(po + i, o[i]);
      }
      st_cs(reinterpret_cast<int32_t*>(a.act) + idx, act);
      if (a.write_logp) {
        // logp_of_normalised: log p_a - log(sum of the normalised row), fp64 (R13 / R18)
        const double dd = cN - 1.0;
        const double lC = fabs(dd) < 1e-6 ? dd * (1.0 - dd * (0.5 - dd * (1.0 / 3.0))) : log(cN);
        st_cs(a.logp + idx, act < 0 ? __int_as_float(0x7fc00000) : (float)(log((double)pa) - lC));
      }
      st_cs(a.rew + idx, rw);
      st_cs_u8(a.done + idx, (uint8_t)d);
      win.put(c & (kRows - 1), lane, d ? (uint32_t)es : 0u, d ? ret : 0.0f, rw);
      if ((c & (kRows - 1)) == kRows - 1 || c == T - 1)
        win.flush(lane, 0, c & (kRows - 1), c & ~(kRows - 1), a.stats, nlive);
    }
    return;
  }

  // ------------------------------------------------------------------------------ env warp
  const Key key{a.k0, a.k1};
  const uint32_t eg = (uint32_t)(a.offset + ec);
  St s, nxt;
  L::load(a.state + ec * L::S, s);
  typename L::Aux aux = L::aux_of(s);
  int32_t ep_step = a.ep_step[ec];
  uint32_t rc = a.reset_count[ec];
  float ep_ret = a.ep_ret[ec];
  L::init(key, eg, rc + 1, nxt);
  U4 w4{0, 0, 0, 0};
  uint32_t err = 0;
  auto publish = [&]() {
    float o[D];
    L::obs_vals(s, aux, o);
#pragma unroll
    for (int d = 0; d < D; ++d) x.obs[d][lane] = o[d];
    asm volatile("bar.arrive 1, 160;" ::: "memory");
  };
  // in-lane R29' evaluation (values_trunc / bootstrap)
  auto value_of = [&](const St& st, const typename L::Aux& ax) {
    float o[D], P[4];
    L::obs_vals(st, ax, o);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float acc_q = 0.0f;
#pragma unroll 4
      for (int u = 0; u < HQ; ++u) {
        const int j = q * HQ + u;
        float acc = b1[j];
#pragma unroll
        for (int d = 0; d < D; ++d) acc = __fmaf_rn(W1[d * H + j], o[d], acc);
        acc_q = __fmaf_rn(wv[j], acc > 0.0f ? acc : 0.0f, acc_q);
      }
      P[q] = acc_q;
    }
    return fadd(wv[H], fadd(fadd(P[0], P[1]), fadd(P[2], P[3])));
  };
  publish();
  for (int c = 0; c < T; ++c) {
    asm volatile("bar.sync 2, 160;" ::: "memory");  // the partials of step c
    const uint64_t t = t0 + (uint64_t)c;
    if (c == 0 || (t & 3) == 0) w4 = block(key, t >> 2, eg, 0, kAction);
    float lg[N], vv = 0.0f;
#pragma unroll
    for (int i = 0; i < N; ++i)
      lg[i] = fadd(b2[i], fadd(fadd(x.part[0][i][lane], x.part[1][i][lane]), fadd(x.part[2][i][lane], x.part[3][i][lane])));
    if (kCritic)
      vv = fadd(wv[H], fadd(fadd(x.part[0][N][lane], x.part[1][N][lane]), fadd(x.part[2][N][lane], x.part[3][N][lane])));
    float m = lg[0];
#pragma unroll
    for (int i = 1; i < N; ++i) m = lg[i] > m ? lg[i] : m;
    RowCDF<N> cdf;
    float S = 0.0f;
    if constexpr (N == 2) {
      // exp(l_max - m) = exp(0) = 1 exactly: one fp64 exponential per step instead of two
      const bool k0 = !(lg[1] > lg[0]);  // m == lg[0]
      const float eo = (float)exp((double)fsub(k0 ? lg[1] : lg[0], m));
      const float em = isfinite(m) ? 1.0f : __int_as_float(0x7fc00000);
      cdf.P[0] = k0 ? em : eo;
      cdf.P[1] = k0 ? eo : em;
      S = fadd(fadd(S, cdf.P[0]), cdf.P[1]);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        cdf.P[i] = (float)exp((double)fsub(lg[i], m));
        S = fadd(S, cdf.P[i]);
      }
    }
    double run = 0.0;
    bool badp = false;
    if constexpr (N == 2) {
      // p_i = e_i / S without the FCHK guard: one e_i is 1 and the other eo in [0, 1], so S lies
      // in [1, 2] (or is NaN, a bad row either way) and div_normal equals IEEE division for the
      // numerators 1 and eo >= 2^-100; below that, S = fl(1 + eo) = 1 and eo / S = eo exactly
      const bool k0 = !(lg[1] > lg[0]);
      const float eo = k0 ? cdf.P[1] : cdf.P[0], em = k0 ? cdf.P[0] : cdf.P[1];
      const float qm = isfinite(em) ? div_normal(1.0f, S) : fdiv(em, S);
      const float qo = eo < 0x1.0p-100f ? eo : div_normal(eo, S);
      cdf.P[0] = k0 ? qm : qo;
      cdf.P[1] = k0 ? qo : qm;
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) cdf.P[i] = fdiv(cdf.P[i], S);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      run += (double)cdf.P[i];
      cdf.C[i] = run;
      badp = badp || !(cdf.P[i] >= 0.0f) || !isfinite(cdf.P[i]);
    }
    cdf.bad = badp || !(run > 0.0) || !isfinite(run);
    // ---- A2 draw (R13) from the ACTION stream
    int act = search<N>(cdf, u01(pick(w4, (uint32_t)(t & 3))));
    float pa = cdf.P[0];
#pragma unroll
    for (int i = 1; i < N; ++i)
      if (act == i) pa = cdf.P[i];
    if (cdf.bad) {
      act = -1;
      if (live) err |= kErrProbs | kErrAction;
    }
    float opre[D];
    L::obs_vals(s, aux, opre);
    // ---- A3-A5
    const bool bad = act < 0;
    St s2 = s;
    typename L::Aux aux2 = aux;
    float rr;
    bool term;
    // the env's fast step when every lane satisfies its invariant (CartPole: guard-free
    // divisions and the Taylor sincos, bit-identical; section 5), else the generic step
    if (L::kMinEpisode >= 8 && __all_sync(kFull, L::fast_ok(s)))
      L::template step_aux<true>(s2, aux2, bad ? 0 : act, rr, term);
    else
      L::template step_aux<false>(s2, aux2, bad ? 0 : act, rr, term);
    const int32_t es = ep_step + 1;
    const uint32_t d = bad ? 0u : ((term ? 1u : 0u) | (es >= a.max_steps ? 2u : 0u));
    const float rw = bad ? 0.0f : rr;
    const float ret = ep_ret + rr;
    if (!bad) {
      s = s2;
      aux = aux2;
      ep_step = es;
      ep_ret = ret;
    }
    if (kCritic && values_trunc && __any_sync(kFull, d == 2u)) {  // truncated only: V of the post-step state
      const float v2 = value_of(s, aux);
      if (live && d == 2u) st_cs(values_trunc + (size_t)c * sE + (size_t)ec, v2);
    }
    if (d) {  // auto-reset (R11) from the look-ahead state init(e, rc + 1)
      rc += 1;
      s = nxt;
      aux = L::aux_of(s);
      ep_step = 0;
      ep_ret = 0.0f;
    }
    if (c + 1 < T) publish();  // the inference warps start step c + 1
    // hand the store-only work of step c to the store warp
    if (c > 0) asm volatile("bar.sync 6, 64;" ::: "memory");  // it has read step c - 1's record
#pragma unroll
    for (int i = 0; i < D; ++i) x.po[i][lane] = opre[i];
    x.pa[lane] = pa;
    x.pvv[lane] = vv;
    x.prw[lane] = rw;
    x.pret[lane] = ret;
    x.pcN[lane] = cdf.C[N - 1];
    x.pact[lane] = act;
    x.pes[lane] = es;
    x.pd[lane] = d;
    asm volatile("bar.arrive 5, 64;" ::: "memory");
    if (__any_sync(kFull, d != 0)) L::init(key, eg, rc + 1, nxt);  // (lanes without a reset recompute the same state)
  }
  asm volatile("bar.sync 6, 64;" ::: "memory");  // the store warp has read the last record
  if constexpr (kCritic) {  // bootstrap value of the observation after the last step
    const float v = value_of(s, aux);
    if (live) bootstrap[e_lane] = v;
  }
  if (live) {
    L::save(a.state + e_lane * L::S, s);
    a.ep_step[e_lane] = ep_step;
    a.reset_count[e_lane] = rc;
    a.ep_ret[e_lane] = ep_ret;
    L::obs_store(a.obs_live + e_lane * L::D, s, false);
  }
  if (err) atomicOr(a.err, err);
}

// =======================================================================================
// A2 for the fused roll-out of continuous single-agent envs (Pendulum, surface-D): the
// Gaussian plan kernel.  Like the discrete plan (R28), the draws z_k of (e, t) do not
// depend on the state, so one thread per (replica, 32-step chunk) walks its contiguous
// range of GAUSS draws j = t*d + k, one Philox4x32 call per 4 draws and one fp64
// Box-Muller per pair, and writes act = mean + exp(log_std) z and logp (R14) into the store.
// =======================================================================================
constexpr int kGaussChunk = 32;  // steps per thread (k_plan_gauss_warp: = the warp size, lane = step)
static_assert(kGaussChunk == 32, "k_plan_gauss_warp maps the chunk's steps onto the lanes");

template <int DIM, bool kStrided>
__global__ void __launch_bounds__(128) k_plan_gauss(const KArgs a, const int T, const uint64_t t0,
                                                   const float* __restrict__ probs, const int64_t row_stride,
                                                   const int64_t step_stride) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = a.E;
  if (e >= E) return;
  const uint32_t eg = (uint32_t)(a.offset + e);
  const Key key{a.k0, a.k1};
  const int c_begin = blockIdx.y * kGaussChunk;
  const int c_end = min(T, c_begin + kGaussChunk);
  float mean[DIM], sd[DIM], log_std[DIM];
  bool ok = true;
  auto load_head = [&](const float* base) {
    ok = true;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      mean[k] = __ldg(base + e * row_stride + k);
      log_std[k] = __ldg(base + e * row_stride + DIM + k);
      ok = ok && isfinite(mean[k]) && isfinite(log_std[k]);
      sd[k] = (float)exp((double)log_std[k]);
    }
  };
  if (!kStrided) load_head(probs);
  float* const p_act = reinterpret_cast<float*>(a.act);
  bool any_bad = false;
  uint64_t cur_blk = ~0ull, cur_pair = ~0ull;
  U4 w{0, 0, 0, 0};
  float ze = 0.0f, zo = 0.0f;
  int c = c_begin;
  if constexpr (DIM == 1 && !kStrided) {
    // one action per step: when the chunk starts on a Philox block, four steps per block in
    // straight-line code (the same draws, values and stores as the general loop below)
    if (((t0 + (uint64_t)c_begin) & 3) == 0) {
      const float nan = __int_as_float(0x7fc00000);
      for (; c + 4 <= c_end; c += 4) {
        const U4 b = block(key, (t0 + (uint64_t)c) >> 2, eg, 0, kGauss);
        float zz[4];
        gauss_pair(b, 0, zz[0], zz[1]);
        gauss_pair(b, 1, zz[2], zz[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const size_t idx = (size_t)(c + k) * (size_t)E + (size_t)e;
          st_cs(p_act + idx, ok ? mean[0] + sd[0] * zz[k] : nan);
          const double lp = 0.0 + (((-0.5 * (double)zz[k]) * (double)zz[k] - (double)log_std[0]) - kHalfLog2Pi);
          if (a.write_logp) st_cs(a.logp + idx, ok ? (float)lp : nan);
        }
      }
      any_bad = !ok;
    }
  }
  for (; c < c_end; ++c) {
    if (kStrided) load_head(probs + (int64_t)c * step_stride);
    const uint64_t j0 = (t0 + (uint64_t)c) * (uint64_t)DIM;
    float z[DIM];
    // draws j0 .. j0 + DIM - 1; one Box-Muller per aligned pair (2p, 2p+1) and one Philox
    // call per block, both carried across steps (warp-uniform: every lane has the same j)
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      const uint64_t j = j0 + (uint64_t)k;
      if ((j >> 1) != cur_pair) {
        if ((j >> 2) != cur_blk) {
          cur_blk = j >> 2;
          w = block(key, cur_blk, eg, 0, kGauss);
        }
        cur_pair = j >> 1;
        gauss_pair(w, (int)(cur_pair & 1), ze, zo);
      }
      z[k] = (j & 1) ? zo : ze;
    }
    double lp = 0.0;
    float act[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      act[k] = ok ? mean[k] + sd[k] * z[k] : __int_as_float(0x7fc00000);
      lp = lp + (((-0.5 * (double)z[k]) * (double)z[k] - (double)log_std[k]) - kHalfLog2Pi);
    }
    const size_t idx = (size_t)c * (size_t)E + (size_t)e;
#pragma unroll
    for (int k = 0; k < DIM; ++k) st_cs(p_act + idx * DIM + k, act[k]);
    if (a.write_logp) st_cs(a.logp + idx, ok ? (float)lp : __int_as_float(0x7fc00000));
    any_bad |= !ok;
  }
  if (any_bad) atomicOr(a.err, kErrProbs);
}

// =======================================================================================
// A7: fused roll-out, continuous single-agent envs (Pendulum, surface-D): the dynamics
// consume the planned actions from the act slab (prefetched one step ahead).
// =======================================================================================
template <class Env>
__global__ void __launch_bounds__(256) k_rollout_continuous(const KArgs a, const int T) {
  using L = Lane<Env>;
  using St = typename L::St;
  constexpr int DIM = L::kDim;
  const int lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = a.E;
  if (e - lane >= E) return;  // whole warp past the last replica
  const bool live = e < E;
  const int64_t ec = live ? e : E - 1;
  const uint32_t eg = (uint32_t)(a.offset + ec);
  const Key key{a.k0, a.k1};
  // 16-row statistics window (6.9 KiB per warp instead of 13.5): this throughput-bound kernel
  // is otherwise limited to 16 resident warps per SM by shared memory (measured: 8 rows flush
  // too often, 32 rows cost occupancy)
  constexpr int kRows = kContWinRows;
  extern __shared__ __align__(16) uint32_t ws_smem[];
  StatsWindow win;
  win.init(ws_smem + (threadIdx.x >> 5) * (3 * kRows * kWinStride), kRows);
  const float* const p_act = reinterpret_cast<const float*>(a.act) + ec * DIM;
  const size_t sE = (size_t)E;

  St s;
  L::load(a.state + ec * L::S, s);
  int32_t ep_step = a.ep_step[ec];
  uint32_t rc = a.reset_count[ec];
  float ep_ret = a.ep_ret[ec];
  uint32_t err = 0;
  float nxt[DIM];
#pragma unroll
  for (int k = 0; k < DIM; ++k) nxt[k] = __ldcg(p_act + k);

  for (int c = 0; c < T; ++c) {
    float act[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) act[k] = nxt[k];
    if (c + 1 < T) {
#pragma unroll
      for (int k = 0; k < DIM; ++k) nxt[k] = __ldcg(p_act + (size_t)(c + 1) * sE * DIM + k);
    }
    const size_t idx = (size_t)c * sE + (size_t)ec;
    St s2 = s;
    float r = 0.0f;
    bool term = false;
    bool ok;
    if constexpr (std::is_same<Env, Pendulum>::value) {  // one sincos serves the observation and the step
      float sn, cs;
      sincos_c(s.th, sn, cs);
      float* dst = a.obs + idx * L::D;  // (cos th, sin th, thdot); tail lanes store replica E-1's values
      st_cs(dst, cs);
      st_cs(dst + 1, sn);
      st_cs(dst + 2, s.thd);
      ok = isfinite(act[0]);
      if (ok) Pendulum::step_sin(s2, act[0], sn, r);
    } else {
      L::obs_store(a.obs + idx * L::D, s, true);  // tail lanes store replica E-1's identical values
      ok = L::step_c(s2, act, r, term);
    }
    if (live && !ok) err |= kErrAction;
    const int32_t es = ep_step + 1;
    const uint32_t d = ok ? ((term ? 1u : 0u) | (es >= a.max_steps ? 2u : 0u)) : 0u;
    const float ret = ep_ret + r;
    const float rw = ok ? r : 0.0f;
    if (d) L::init(key, eg, rc + 1, s2);
    s = ok ? s2 : s;
    rc += d ? 1u : 0u;
    ep_step = d ? 0 : (ok ? es : ep_step);
    ep_ret = d ? 0.0f : (ok ? ret : ep_ret);
    st_cs(a.rew + idx, rw);
    st_cs_u8(a.done + idx, (uint8_t)d);
    win.put(c & (kRows - 1), lane, d ? (uint32_t)es : 0u, d ? ret : 0.0f, rw);
    if ((c & (kRows - 1)) == kRows - 1 || c == T - 1)
      win.flush(lane, 0, c & (kRows - 1), c & ~(kRows - 1), a.stats, (int)min((int64_t)32, E - (e - lane)));
  }
  if (live) {
    L::save(a.state + e * L::S, s);
    a.ep_step[e] = ep_step;
    a.reset_count[e] = rc;
    a.ep_ret[e] = ep_ret;
    L::obs_store(a.obs_live + e * L::D, s, false);
    if (err) atomicOr(a.err, err);
  }
}

// =======================================================================================
// NEXT-N1 for continuous actions (R34): Pendulum with a Gaussian MLP policy inside the fused
// loop -- the R29 network (fp32 FMAs in R29's order) with one linear output as the mean and a
// learned log_std, sampled by the R14 Gaussian head (gauss_sample: the GAUSS draw j = t of
// the replica's stream, act = mean + exp(log_std) z, fp64 log-density); kCritic adds the R31
// value head (values[t] = V(obs[t]), bootstrap = V(obs_live)).  Weights W1 [3][H] | b1 [H] |
// W2 [H][1] | b2 [1] | log_std [1] (| wv [H] | bv) staged in shared memory.
// =======================================================================================
template <int H, bool kCritic>
__global__ void __launch_bounds__(128) k_rollout_gpolicy(const KArgs a, const int T, const uint64_t t0,
                                                        const float* __restrict__ weights,
                                                        float* __restrict__ values, float* __restrict__ bootstrap,
                                                        float* __restrict__ values_trunc) {
  using L = Lane<Pendulum>;
  using St = Pendulum::St;
  constexpr int D = 3;
  constexpr int NW = D * H + H + H + 1 + 1 + (kCritic ? H + 1 : 0);
  __shared__ float sw[NW];
  for (int i = threadIdx.x; i < NW; i += blockDim.x) sw[i] = weights[i];
  __syncthreads();
  const float* W1 = sw;
  const float* b1 = W1 + D * H;
  const float* W2 = b1 + H;
  const float* b2 = W2 + H;
  const float* ls = b2 + 1;
  const float* wv = ls + 1;  // kCritic only
  const int lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = a.E;
  if (e - lane >= E) return;
  const bool live = e < E;
  const int64_t ec = live ? e : E - 1;
  const uint32_t eg = (uint32_t)(a.offset + ec);
  const Key key{a.k0, a.k1};
  constexpr int kRows = kContWinRows;
  extern __shared__ __align__(16) uint32_t ws_smem[];
  StatsWindow win;
  win.init(ws_smem + (threadIdx.x >> 5) * (3 * kRows * kWinStride), kRows);
  const size_t sE = (size_t)E;
  St s;
  L::load(a.state + ec * L::S, s);
  int32_t ep_step = a.ep_step[ec];
  uint32_t rc = a.reset_count[ec];
  float ep_ret = a.ep_ret[ec];
  uint32_t err = 0;
  auto head = [&](const float (&o)[3], float& mean, float& v) {  // R29' quarter sums (in-lane)
    float hid[H];
#pragma unroll
    for (int j = 0; j < H; ++j) {
      float acc = b1[j];
#pragma unroll
      for (int k = 0; k < D; ++k) acc = __fmaf_rn(W1[k * H + j], o[k], acc);
      hid[j] = acc > 0.0f ? acc : 0.0f;
    }
    mean = quarter_dot<H>(W2, 1, hid, b2[0]);
    v = kCritic ? quarter_dot<H>(wv, 1, hid, wv[H]) : 0.0f;
  };
  for (int c = 0; c < T; ++c) {
    const uint64_t t = t0 + (uint64_t)c;
    const size_t idx = (size_t)c * sE + (size_t)ec;
    float sn, cs;
    sincos_c(s.th, sn, cs);
    float* dst = a.obs + idx * L::D;  // (cos th, sin th, thdot)
    st_cs(dst, cs);
    st_cs(dst + 1, sn);
    st_cs(dst + 2, s.thd);
    const float o[3] = {cs, sn, s.thd};
    float mean1, v;
    head(o, mean1, v);
    if (kCritic) st_cs(values + idx, v);
    const float mean[1] = {mean1}, lstd[1] = {ls[0]};
    float act[1], lp;
    const bool okp = gauss_sample<1>(key, eg, 0, t, mean, lstd, act, lp);
    st_cs(reinterpret_cast<float*>(a.act) + idx, act[0]);
    if (a.write_logp) st_cs(a.logp + idx, lp);
    St s2 = s;
    float r = 0.0f;
    const bool ok = isfinite(act[0]);
    if (live && !okp) err |= kErrProbs;
    if (live && !ok) err |= kErrAction;
    if (ok) Pendulum::step_sin(s2, act[0], sn, r);
    const int32_t es = ep_step + 1;
    const uint32_t d = ok ? (es >= a.max_steps ? 2u : 0u) : 0u;
    const float ret = ep_ret + r;
    const float rw = ok ? r : 0.0f;
    if (kCritic && values_trunc && d == 2u) {  // truncated only: V of the post-step state
      float sn2, cs2;
      sincos_c(s2.th, sn2, cs2);
      const float o2[3] = {cs2, sn2, s2.thd};
      float m_unused, vt;
      head(o2, m_unused, vt);
      if (live) st_cs(values_trunc + idx, vt);
    }
    if (d) L::init(key, eg, rc + 1, s2);
    s = ok ? s2 : s;
    rc += d ? 1u : 0u;
    ep_step = d ? 0 : (ok ? es : ep_step);
    ep_ret = d ? 0.0f : (ok ? ret : ep_ret);
    st_cs(a.rew + idx, rw);
    st_cs_u8(a.done + idx, (uint8_t)d);
    win.put(c & (kRows - 1), lane, d ? (uint32_t)es : 0u, d ? ret : 0.0f, rw);
    if ((c & (kRows - 1)) == kRows - 1 || c == T - 1)
      win.flush(lane, 0, c & (kRows - 1), c & ~(kRows - 1), a.stats, (int)min((int64_t)32, E - (e - lane)));
  }
  if (kCritic) {
    float sn, cs;
    sincos_c(s.th, sn, cs);
    const float o[3] = {cs, sn, s.thd};
    float m_unused, v;
    head(o, m_unused, v);
    if (live) bootstrap[e] = v;
  }
  if (live) {
    L::save(a.state + e * L::S, s);
    a.ep_step[e] = ep_step;
    a.reset_count[e] = rc;
    a.ep_ret[e] = ep_ret;
    L::obs_store(a.obs_live + e * L::D, s, false);
    if (err) atomicOr(a.err, err);
  }
}

// =======================================================================================
// surface-D (R23) with one WARP per replica and one lane per coordinate (D <= 32): the
// lane-per-replica kernel leaves C5's 2 000 replicas in 63 warps; this mapping gives 2 000.
// Sums over coordinates (spring energy, goal distance, Gaussian log-density) are gathered
// with shuffles: the spring energy in coordinate order (the oracle's sequential association,
// bit-identical), the goal distance (only compared with r_goal^2) and the Gaussian
// log-density (rounded to fp32, R18) by a fixed xor-butterfly; the four Mueller-Brown terms
// run on lanes 0..3.
// =======================================================================================
__device__ const double kMB[6][4] = {{-200, -100, -170, 15}, {-1, -1, -6.5, 0.7}, {0, 0, 11, 0.6},
                                      {-10, -10, -6.5, 0.7}, {1, 0, -0.5, -1}, {0, 0.5, 1.5, 1}};

// fixed-order xor-butterfly fp64 sum (all lanes get the same value): used where only an fp32
// rounding at <= 2 ulp tolerance follows (the Gaussian log-density, R18), so the association
// need not match the oracle's sequential loop
__device__ __forceinline__ double warp_tree_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// =======================================================================================
// A7 for surface-D, segmented: each replica is a segment of L = ceil(D/4) lanes holding four
// coordinates each, so a warp advances R = 32 / L replicas at once (D = 20: 5 lanes, 6
// replicas).  Coordinate-parallel work (action clip, update, observation stores, reset draws,
// squares) stays on the lanes; the energy's two fixed-order sums (R23: the Mueller-Brown terms
// as (t0 + t1) + (t2 + t3), the spring sum as the pairwise tree over the padded coordinate
// leaves) are assembled from register shuffles inside the segment: each lane's four leaves
// form one 4-leaf subtree of the oracle's tree, the segment's lanes 0..3 each evaluate one
// Mueller-Brown term (one fp64 exp per lane, in parallel), and every lane of the segment
// gathers the L subtrees and the four terms and adds them in the tree order.  The goal
// distance only feeds a comparison, so its lane partials are added in any fixed order.
// Actions are prefetched four steps ahead (register ring).
// =======================================================================================
template <int D>
struct SurfSeg {
  static constexpr int C = 4;                // coordinates per lane
  static constexpr int L = (D + C - 1) / C;  // lanes per replica
  static constexpr int R = 32 / L;           // replicas per warp
};

// pairwise tree over the segment's per-lane 4-leaf subtrees g[0 .. G) (G = the tree's leaves / 4;
// subtrees >= L are padding, +0, skipped exactly as in spring_tree)
template <int L, int LO, int N>
__device__ __forceinline__ double group_tree(const double* g) {
  if constexpr (N == 1) {
    return LO < L ? g[LO] : 0.0;
  } else if constexpr (LO + N / 2 >= L) {
    return group_tree<L, LO, N / 2>(g);
  } else {
    return group_tree<L, LO, N / 2>(g) + group_tree<L, LO + N / 2, N / 2>(g);
  }
}

template <int D>
struct SurfSegWarp {
  using Env = Surface<D>;
  using G = SurfSeg<D>;
  static constexpr int C = G::C, L = G::L, R = G::R;
  static constexpr int kGroups = spring_leaves(D) / C;  // 4-leaf subtrees of the spring tree
  int lane, seg, sl, src;  // src: the segment's first lane
  bool used;
  double mc[6];  // Mueller-Brown coefficients (A, a, b, c, x0, y0) of term sl (L >= 4)

  __device__ __forceinline__ void load_coefficients() {
#pragma unroll
    for (int i = 0; i < 6; ++i) mc[i] = __ldg(&kMB[i][sl < 4 ? sl : 0]);
  }
  __device__ __forceinline__ bool valid(int i) const { return sl * C + i < D; }
  __device__ __forceinline__ double shfl_d(double v, int from) const {
    return __hiloint2double(__shfl_sync(kFull, __double2hiint(v), from), __shfl_sync(kFull, __double2loint(v), from));
  }
  // energy of the segment's state q (this lane's C coordinates); warp-collective; *spring_out
  // (optional) receives the spring sum
  __device__ __forceinline__ float energy(const float (&q)[C], double* spring_out = nullptr) const {
    // spring: this lane's leaves 4 sl .. 4 sl + 3 (coordinates 0, 1 and >= D are +0 leaves)
    double w[C];
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const int k = sl * C + i;
      w[i] = (k >= 2 && k < D) ? (double)q[i] * (double)q[i] : 0.0;
    }
    const double g = (w[0] + w[1]) + (w[2] + w[3]);
    // Mueller-Brown terms of (q0, q1), which live on the segment's first lane
    const double x = (double)__shfl_sync(kFull, q[0], src), y = (double)__shfl_sync(kFull, q[1], src);
    constexpr int kTermsPerLane = (4 + L - 1) / L;
    double tv[kTermsPerLane];
    if constexpr (L >= 4) {
      const double dx = x - mc[4], dy = y - mc[5];
      tv[0] = mc[0] * exp64(mc[1] * dx * dx + mc[2] * dx * dy + mc[3] * dy * dy);
    } else {
#pragma unroll
      for (int r = 0; r < kTermsPerLane; ++r) {
        const int m = min(r * L + sl, 3);
        const double dx = x - __ldg(&kMB[4][m]), dy = y - __ldg(&kMB[5][m]);
        tv[r] = __ldg(&kMB[0][m]) * exp64(__ldg(&kMB[1][m]) * dx * dx + __ldg(&kMB[2][m]) * dx * dy +
                                          __ldg(&kMB[3][m]) * dy * dy);
      }
    }
    double t[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) t[m] = shfl_d(tv[m / L], src + m % L);
    double gs[L];
#pragma unroll
    for (int j = 0; j < L; ++j) gs[j] = shfl_d(g, src + j);
    const double E = (t[0] + t[1]) + (t[2] + t[3]);
    const double spring = group_tree<L, 0, kGroups>(gs);
    if (spring_out) *spring_out = spring;
    return (float)(E + 0.5 * Env::kappa * spring);
  }
  // squared distance of the segment's state to the goal (fixed association; comparison only)
  __device__ __forceinline__ double goal_d2(const float (&q)[C]) const {
    double p = 0.0;
#pragma unroll
    for (int i = 0; i < C; ++i) {
      if (valid(i)) {
        const double di = (double)q[i] - Env::goal(sl * C + i);
        p += di * di;
      }
    }
    double d2 = 0.0;
#pragma unroll
    for (int j = 0; j < L; ++j) d2 += shfl_d(p, src + j);
    return d2;
  }
};

template <int D>
__global__ void __launch_bounds__(256) k_rollout_surface_seg(const KArgs a, const int T) {
  using Env = Surface<D>;
  using SW = SurfSegWarp<D>;
  constexpr int C = SW::C, L = SW::L, R = SW::R;
  extern __shared__ __align__(16) uint32_t ws_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t E = a.E;
  const int64_t wg = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;  // global warp index
  if (wg * R >= E) return;  // whole warp past the last replica
  SW w;
  w.lane = lane;
  w.seg = lane / L;
  w.sl = lane % L;
  w.used = w.seg < R;  // lanes of the scratch segment R (if any) compute but never store
  w.src = (w.used ? w.seg : R - 1) * L;  // scratch lanes read a real segment (values unused)
  w.load_coefficients();
  const int seg = w.used ? w.seg : R - 1, sl = w.sl;
  const int64_t e_raw = wg * R + seg;
  const bool live = w.used && e_raw < E;      // this segment simulates a real replica
  const int64_t e = e_raw < E ? e_raw : E - 1;  // else it shadows replica E-1 (identical stores)
  const bool leader = live && sl == 0;
  const uint32_t eg = (uint32_t)(a.offset + e);
  const Key key{a.k0, a.k1};
  const size_t sE = (size_t)E;
  constexpr int kRows = 16;  // statistics window depth (slots per flush)
  StatsWindow win;           // per-warp window: leaders' (length, return, reward) per slot
  win.init(ws_smem + 2 * 256 + wib * (3 * kRows * kWinStride), kRows);
  // (the first 2 KB of the dynamic shared memory are not used by this kernel: the statistics
  // windows flush straight to the global slab, warp by warp)
  float lo[C], hi[C], q[C];
#pragma unroll
  for (int i = 0; i < C; ++i) {
    const int k = sl * C + i;
    lo[i] = Env::lo(k < D ? k : 0);
    hi[i] = Env::hi(k < D ? k : 0);
    q[i] = k < D ? a.state[e * D + k] : 0.0f;
  }
  float Ecur = w.energy(q);
  int32_t ep_step = a.ep_step[e];
  uint32_t rc = a.reset_count[e];
  float ep_ret = a.ep_ret[e];
  uint32_t err = 0;
  const float* const p_act = reinterpret_cast<const float*>(a.act) + e * D + sl * C;
  float* const p_obs = a.obs + e * (D + 1) + sl * C;
  auto load_act = [&](int c, float (&v)[C]) {
    if (c >= T) return;
    const float* p = p_act + (size_t)c * sE * D;
    if constexpr (D % 4 == 0) {
      const float4 t = __ldcg(reinterpret_cast<const float4*>(p));
      v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
#pragma unroll
      for (int i = 0; i < C; ++i) v[i] = w.valid(i) ? __ldcg(p + i) : 0.0f;
    }
  };
  // one fused step at slot c with the (prefetched) action ak
  auto one = [&](const int c, const float (&ak)[C]) {
    const size_t idx = (size_t)c * sE + (size_t)e;
    // pre-step observation (q, E(q))
    if (w.used) {
      float* po = p_obs + (size_t)c * sE * (D + 1);
#pragma unroll
      for (int i = 0; i < C; ++i)
        if (w.valid(i)) st_cs(po + i, q[i]);
      if (sl == L - 1) st_cs(po + (D - sl * C), Ecur);
    }
    // a replica step is valid iff all D action components are finite
    bool bad_lane = false;
#pragma unroll
    for (int i = 0; i < C; ++i) bad_lane = bad_lane || (w.valid(i) && !isfinite(ak[i]));
    const unsigned bm = __ballot_sync(kFull, w.used && bad_lane);
    const bool ok = ((bm >> (seg * L)) & ((1u << L) - 1u)) == 0u;
    float qn[C];
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const float ai = fminf(fmaxf(ak[i], -Env::delta), Env::delta);
      qn[i] = w.valid(i) ? fminf(fmaxf(q[i] + ai, lo[i]), hi[i]) : 0.0f;
      if (!ok) qn[i] = q[i];
    }
    const float En = w.energy(qn);
    const double d2 = w.goal_d2(qn);
    float r = 0.0f;
    uint32_t d = 0;
    if (ok) {
      const bool term = d2 < Env::r_goal * Env::r_goal;
      r = -(Env::w_E * (En - Ecur)) - Env::c_step;
      if (term) r = r + Env::bonus;
      const int32_t es = ep_step + 1;
      d = (term ? 1u : 0u) | (es >= a.max_steps ? 2u : 0u);
      const float ret = ep_ret + r;
      win.put(c & (kRows - 1), lane, (leader && d) ? (uint32_t)es : 0u, (leader && d) ? ret : 0.0f, 0.0f);
      ep_step = d ? 0 : es;
      ep_ret = d ? 0.0f : ret;
#pragma unroll
      for (int i = 0; i < C; ++i) q[i] = qn[i];
      Ecur = En;
    } else {
      win.put(c & (kRows - 1), lane, 0u, 0.0f, 0.0f);
      if (leader) err |= kErrAction;
    }
    win.rew[(c & (kRows - 1)) * kWinStride + lane] = leader ? r : 0.0f;  // slot reward (R20 at flush)
    if (leader) {
      st_cs(a.rew + idx, r);
      st_cs_u8(a.done + idx, (uint8_t)d);
    }
    // A5 auto-reset: the segment's lanes draw their own coordinates (draws j = rc*D + k)
    if (__any_sync(kFull, w.used && d != 0)) {
      if (d) {
        rc += 1;
#pragma unroll
        for (int i = 0; i < C; ++i) {
          const int k = sl * C + i;
          if (k < D) {
            const uint64_t j = (uint64_t)rc * D + (uint64_t)k;
            const U4 b = block(key, j >> 2, eg, 0, kReset);
            q[i] = Env::start(k) + (-0.05f + 0.1f * u01(pick(b, (uint32_t)(j & 3))));
          }
        }
      }
      const float Er = w.energy(q);
      if (d) Ecur = Er;
    }
    if ((c & (kRows - 1)) == kRows - 1 || c == T - 1) {  // window -> CTA accumulator -> global atomics
      // per-warp global atomics (no CTA barrier between the latency-bound warps, as the
      // discrete latency build)
      win.cta_acc = nullptr;
      win.flush(lane, 0, c & (kRows - 1), c & ~(kRows - 1), a.stats, 32);
    }
  };
  // Fast 4-step trip (round 2).  The only loop-carried dependence of a step without a reset is
  // the clip-and-add state update; the energy (fp64 exp + shuffles, ~1300 cycles in one()) and the
  // goal test only feed the reward, the stores and the done flag.  So when no replica of the warp
  // can finish inside the trip -- every action finite, no truncation, and every post-step state
  // provably outside the goal ball -- the trip computes the four states first, then the four
  // energies as independent chains, then the rewards and stores: the same values in the same
  // order as four one() calls.  The goal proof: d2 is a sum of non-negative fp64 terms, so with
  // monotone rounding it is >= any lane's partial sum; one lane partial >= r_goal^2 rules the
  // goal out (R23's d2 < r_goal^2).  Otherwise (and for the rare trips with a done flag or an
  // invalid action) the trip returns false before changing anything and one() runs four times.
  auto fastK = [&](auto Kc, const int c, const auto& act) -> bool {  // act: float[K][C]
    constexpr int K = decltype(Kc)::value;
    bool bad = ep_step + K >= a.max_steps;  // a truncation inside the trip
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int i = 0; i < C; ++i) bad = bad || (w.valid(i) && !isfinite(act[k][i]));
    float qs[K][C];
    bool near = false;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float p = 0.0f;
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const float prev = k == 0 ? q[i] : qs[k - 1][i];
        const float ai = fminf(fmaxf(act[k][i], -Env::delta), Env::delta);
        qs[k][i] = w.valid(i) ? fminf(fmaxf(prev + ai, lo[i]), hi[i]) : 0.0f;
        if (w.valid(i)) {
          const float di = qs[k][i] - (float)Env::goal(sl * C + i);
          p = p + di * di;
        }
      }
      // the segment may be inside the goal ball only if none of its lanes rules it out.  The
      // lane partial is evaluated in fp32: against the fp64 partial its error is < 1e-6
      // relative + 1e-7 absolute (four terms, |goal| < 2), so p > r_goal^2 + 1e-4 proves the
      // fp64 partial > r_goal^2 as well
      const unsigned far = __ballot_sync(kFull, p > (float)(Env::r_goal * Env::r_goal) + 1e-4f);
      near = near || ((far >> (seg * L)) & ((1u << L) - 1u)) == 0u;
    }
    if (__any_sync(kFull, w.used && (bad || near))) return false;
    float En[K];
#pragma unroll
    for (int k = 0; k < K; ++k) En[k] = w.energy(qs[k]);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int ck = c + k;
      const float Epre = k == 0 ? Ecur : En[k - 1];
      if (w.used) {
        float* po = p_obs + (size_t)ck * sE * (D + 1);
#pragma unroll
        for (int i = 0; i < C; ++i)
          if (w.valid(i)) st_cs(po + i, k == 0 ? q[i] : qs[k - 1][i]);
        if (sl == L - 1) st_cs(po + (D - sl * C), Epre);
      }
      const float r = -(Env::w_E * (En[k] - Epre)) - Env::c_step;
      ep_step = ep_step + 1;
      ep_ret = ep_ret + r;
      win.put(ck & (kRows - 1), lane, 0u, 0.0f, 0.0f);
      win.rew[(ck & (kRows - 1)) * kWinStride + lane] = leader ? r : 0.0f;
      if (leader) {
        const size_t idx = (size_t)ck * sE + (size_t)e;
        st_cs(a.rew + idx, r);
        st_cs_u8(a.done + idx, (uint8_t)0);
      }
    }
#pragma unroll
    for (int i = 0; i < C; ++i) q[i] = qs[K - 1][i];
    Ecur = En[K - 1];
    const int cl = c + K - 1;  // K <= kRows: at most one window ends inside the trip, at its last step
    if ((cl & (kRows - 1)) == kRows - 1 || cl == T - 1) {
      win.cta_acc = nullptr;  // per-warp global atomics (see one())
      win.flush(lane, 0, cl & (kRows - 1), cl & ~(kRows - 1), a.stats, 32);
    }
    return true;
  };
  if constexpr (D % 4 == 0) {
    // 8-step trips (eight energies in flight).  The actions stream through a per-warp cp.async
    // ring in shared memory ([2 trips][8 steps][32 lanes] float4 after the statistics windows):
    // trip j + 2's group is issued once trip j's actions are in registers, so a trip's loads
    // have a whole trip to land and take no registers while in flight.
    constexpr int KT = WS_SURF_TRIP;  // steps per trip
    float4* const ring = reinterpret_cast<float4*>(ws_smem + 2 * 256 + (blockDim.x >> 5) * (3 * kRows * kWinStride)) +
                         wib * (2 * KT * 32);
    auto issue = [&](int j) {  // steps KT j .. KT j + KT - 1 into buffer j & 1 (an empty group past the end)
      float4* dst = ring + (j & 1) * (KT * 32) + lane;
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        const int ck = KT * j + k;
        if (ck < T) {
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + k * 32);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(p_act + (size_t)ck * sE * D) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int ntrip = (T + KT - 1) / KT;
    issue(0);
    issue(1);
    for (int j = 0; j < ntrip; ++j) {
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // trip j's group has landed (each lane reads its own)
      const int c = KT * j, n = min(KT, T - c);
      const float4* src = ring + (j & 1) * (KT * 32) + lane;
      bool done_fast = false;
      if (n == KT) {
        float A[KT][C];
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          const float4 t = src[k * 32];
          A[k][0] = t.x; A[k][1] = t.y; A[k][2] = t.z; A[k][3] = t.w;
        }
        done_fast = fastK(std::integral_constant<int, KT>{}, c, A);
      }
      if (!done_fast) {
#pragma unroll 1
        for (int k = 0; k < n; ++k) {
          const float4 t = src[k * 32];
          const float v[C] = {t.x, t.y, t.z, t.w};
          one(c + k, v);
        }
      }
      issue(j + 2);  // into buffer j & 1, whose values have been consumed
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    auto trip = [&](const int c, const float (&A)[4][C]) {
      if (!fastK(std::integral_constant<int, 4>{}, c, A)) {
        one(c, A[0]);
        one(c + 1, A[1]);
        one(c + 2, A[2]);
        one(c + 3, A[3]);
      }
    };
    // two action register sets used in turn (no copies: a copy placed by the compiler right after
    // the loads stalls on them): the next trip's actions load while this trip runs
    float a4[4][C] = {}, b4[4][C] = {};
#pragma unroll
    for (int k = 0; k < 4; ++k) load_act(k, a4[k]);
    int c = 0;
    for (; c + 8 <= T; c += 8) {
#pragma unroll
      for (int k = 0; k < 4; ++k) load_act(c + 4 + k, b4[k]);
      trip(c, a4);
#pragma unroll
      for (int k = 0; k < 4; ++k) load_act(c + 8 + k, a4[k]);
      trip(c + 4, b4);
    }
    if (c + 4 <= T) {  // one more full trip on set a; the tail's actions go to set b
#pragma unroll
      for (int k = 0; k < 3; ++k) load_act(c + 4 + k, b4[k]);
      trip(c, a4);
      c += 4;
      if (c < T) one(c, b4[0]);
      if (c + 1 < T) one(c + 1, b4[1]);
      if (c + 2 < T) one(c + 2, b4[2]);
    } else {
      if (c < T) one(c, a4[0]);
      if (c + 1 < T) one(c + 1, a4[1]);
      if (c + 2 < T) one(c + 2, a4[2]);
    }
  }
  if (live) {
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const int k = sl * C + i;
      if (k < D) {
        a.state[e * D + k] = q[i];
        a.obs_live[e * (D + 1) + k] = q[i];
      }
    }
    if (sl == L - 1) a.obs_live[e * (D + 1) + D] = Ecur;
    if (sl == 0) {
      a.ep_step[e] = ep_step;
      a.reset_count[e] = rc;
      a.ep_ret[e] = ep_ret;
      if (err) atomicOr(a.err, err);
    }
  }
}

// test hook (ws_test_surface_energy): the segmented energy on arbitrary states, one warp per
// R states
template <int D>
__global__ void __launch_bounds__(128) k_test_surface_energy(const float* q, int64_t n, float* energy, double* spring) {
  using SW = SurfSegWarp<D>;
  constexpr int C = SW::C, L = SW::L, R = SW::R;
  const int lane = threadIdx.x & 31;
  const int64_t wg = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wg * R >= n) return;
  SW w;
  w.lane = lane;
  w.seg = lane / L;
  w.sl = lane % L;
  w.used = w.seg < R;
  w.src = (w.used ? w.seg : R - 1) * L;
  w.load_coefficients();
  const int seg = w.used ? w.seg : R - 1;
  const int64_t i = min(wg * R + seg, n - 1);
  float v[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int k = w.sl * C + c;
    v[c] = k < D ? q[i * D + k] : 0.0f;
  }
  double sp = 0.0;
  const float en = w.energy(v, &sp);
  if (w.used && w.sl == 0 && wg * R + seg < n) {
    energy[i] = en;
    spring[i] = sp;
  }
}

// Gaussian plan with one warp per (replica, 32-step chunk), lane = action dimension; the
// log-density terms are summed by a fixed xor-butterfly (<= 2 ulp from the oracle's
// sequential sum after rounding, R18).
template <int DIM, bool kStrided>
__global__ void __launch_bounds__(128) k_plan_gauss_warp(const KArgs a, const int T, const uint64_t t0,
                                                        const float* __restrict__ probs, const int64_t row_stride,
                                                        const int64_t step_stride) {
  const int lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (e >= a.E) return;
  const uint32_t eg = (uint32_t)(a.offset + e);
  const Key key{a.k0, a.k1};
  const int c_begin = blockIdx.y * kGaussChunk;
  const int c_end = min(T, c_begin + kGaussChunk);
  const bool act_lane = lane < DIM;
  const int kk = act_lane ? lane : 0;
  float mean = 0.0f, ls = 0.0f, sd = 1.0f;
  bool ok = true;
  auto load_head = [&](const float* base) {
    mean = __ldg(base + e * row_stride + kk);
    ls = __ldg(base + e * row_stride + DIM + kk);
    ok = __all_sync(kFull, !act_lane || (isfinite(mean) && isfinite(ls)));
    sd = (float)exp((double)ls);
  };
  if (!kStrided) load_head(probs);
  // The chunk's GAUSS draws J0 .. J1-1 are Box-Muller pairs (2p, 2p+1): the warp's 32 lanes
  // each take one pair at a time (one fp64 log / sqrt / sincos per pair, no lane computing a
  // pair twice) and stage the normals in shared memory; the coordinate lanes then read them.
  __shared__ __align__(16) float zbuf[4][kGaussChunk * DIM];
  float* const zb = zbuf[(threadIdx.x >> 5) & 3];
  const uint64_t J0 = (t0 + (uint64_t)c_begin) * (uint64_t)DIM, J1 = (t0 + (uint64_t)c_end) * (uint64_t)DIM;
  // one Philox block (two pairs, four normals) per lane and iteration: no block computed twice
  const int nJ = (int)(J1 - J0);
  if ((J0 & 3) == 0 && (nJ & 3) == 0) {
    // aligned chunk (every chunk when D % 4 == 0): whole blocks, 32-bit indices, one 16-byte store
    const uint64_t b0 = J0 >> 2;
    for (int kb = lane; kb < (nJ >> 2); kb += 32) {
      const U4 w = block(key, b0 + (uint64_t)kb, eg, 0, kGauss);
      float z0, z1, z2, z3;
      gauss_pair(w, 0, z0, z1);
      gauss_pair(w, 1, z2, z3);
      *reinterpret_cast<float4*>(zb + 4 * kb) = make_float4(z0, z1, z2, z3);
    }
  } else
  for (uint64_t b = (J0 >> 2) + (uint64_t)lane; b < ((J1 + 3) >> 2); b += 32) {
    const U4 w = block(key, b, eg, 0, kGauss);
    const int64_t i0 = (int64_t)(4 * b) - (int64_t)J0;
    const int64_t n = (int64_t)(J1 - J0);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int64_t i = i0 + 2 * p;
      if (i + 1 >= 0 && i < n) {  // the pair has a draw inside [J0, J1)
        float ze, zo;
        gauss_pair(w, p, ze, zo);
        if (i >= 0) zb[i] = ze;
        if (i + 1 < n) zb[i + 1] = zo;
      }
    }
  }
  __syncwarp();
  float* const p_act = reinterpret_cast<float*>(a.act) + e * DIM + kk;
  bool any_bad = false;
  if constexpr (!kStrided) {
    // one head for the whole chunk: lanes = coordinates for the act rows, then lanes = steps for
    // the log-densities, lp = -(sum_k z_k^2) / 2 - sum_k (log sd_k + log(2 pi) / 2) in fp64 (R14;
    // the association is free: one fp32 rounding follows, R18 <= 2 ulp) -- no per-step warp
    // reduction
    for (int c = c_begin; c < c_end; ++c) {
      const float z = zb[(c - c_begin) * DIM + kk];
      if (act_lane) st_cs(p_act + (size_t)c * (size_t)a.E * DIM, ok ? mean + sd * z : __int_as_float(0x7fc00000));
    }
    const double cst = warp_tree_sum(act_lane ? (double)ls + kHalfLog2Pi : 0.0);
    const int c = c_begin + lane;
    if (a.write_logp && c < c_end) {
      double s2 = 0.0;
      const float* zr = zb + lane * DIM;
#pragma unroll
      for (int k = 0; k < DIM; ++k) s2 = fma((double)zr[k], (double)zr[k], s2);
      st_cs(a.logp + (size_t)c * (size_t)a.E + (size_t)e, ok ? (float)(-0.5 * s2 - cst) : __int_as_float(0x7fc00000));
    }
    any_bad = !ok;
  } else {
    for (int c = c_begin; c < c_end; ++c) {
      load_head(probs + (int64_t)c * step_stride);
      const float z = zb[(c - c_begin) * DIM + kk];
      const double term = act_lane ? (((-0.5 * (double)z) * (double)z - (double)ls) - kHalfLog2Pi) : 0.0;
      const double lp = warp_tree_sum(term);
      const size_t idx = (size_t)c * (size_t)a.E + (size_t)e;
      if (act_lane) st_cs(p_act + (size_t)c * (size_t)a.E * DIM, ok ? mean + sd * z : __int_as_float(0x7fc00000));
      if (lane == 0 && a.write_logp) st_cs(a.logp + idx, ok ? (float)lp : __int_as_float(0x7fc00000));
      any_bad |= !ok;
    }
  }
  if (lane == 0 && any_bad) atomicOr(a.err, kErrProbs);
}

// =======================================================================================
// Single-step path (ws_sample / ws_step) for the lane envs.
// =======================================================================================
// ws_sample, discrete rows (any A): warp-cooperative scan + search, one row per lane.
template <int N>
__global__ void __launch_bounds__(256) k_sample_discrete(const KArgs a, const int slot, const uint64_t t_host,
                                                        const float* __restrict__ probs,
                                                        const int64_t row_stride) {
  const uint64_t t = a.t_dev ? *a.t_dev : t_host;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // e*A + agent
  const int lane = threadIdx.x & 31;
  const int64_t n_rows = a.E * (int64_t)a.A;
  RowCDF<N> cdf;
  warp_row_cdf<N>(probs, row_stride, row - lane, n_rows, lane, cdf);
  if (row >= n_rows) return;
  const int64_t e = row / a.A;
  const uint32_t agent = (uint32_t)(row - e * a.A);
  const U4 b = block(Key{a.k0, a.k1}, t >> 2, (uint32_t)(a.offset + e), agent, kAction);
  int act = search<N>(cdf, u01(pick(b, (uint32_t)(t & 3))));
  float lp = logp_of<N>(cdf, act);
  if (cdf.bad) {
    act = -1;
    lp = __int_as_float(0x7fc00000);
    atomicOr(a.err, kErrProbs);
  }
  const size_t idx = (size_t)slot * (size_t)n_rows + (size_t)row;
  reinterpret_cast<int32_t*>(a.act)[idx] = act;
  if (a.write_logp) a.logp[idx] = lp;
}

template <int DIM>
__global__ void __launch_bounds__(256) k_sample_continuous(const KArgs a, const int slot, const uint64_t t_host,
                                                          const float* __restrict__ probs,
                                                          const int64_t row_stride) {
  const uint64_t t = a.t_dev ? *a.t_dev : t_host;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_rows = a.E * (int64_t)a.A;
  if (row >= n_rows) return;
  const int64_t e = row / a.A;
  const uint32_t agent = (uint32_t)(row - e * a.A);
  float mean[DIM], log_std[DIM], act[DIM], lp;
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    mean[k] = probs[row * row_stride + k];
    log_std[k] = probs[row * row_stride + DIM + k];
  }
  const bool ok = gauss_sample<DIM>(Key{a.k0, a.k1}, (uint32_t)(a.offset + e), agent, t, mean, log_std, act, lp);
  if (!ok) atomicOr(a.err, kErrProbs);
  const size_t idx = (size_t)slot * (size_t)n_rows + (size_t)row;
#pragma unroll
  for (int k = 0; k < DIM; ++k) reinterpret_cast<float*>(a.act)[idx * DIM + k] = act[k];
  if (a.write_logp) a.logp[idx] = lp;
}

// ws_step for lane envs: actions from the act slab (given == nullptr) or from `given`
// (copied into the slab, logp = NaN, R27).  Every lane of the warp executes the step
// (tail lanes on a shadow replica, nothing stored) so warp-collective code is legal.
template <class Env>
__global__ void __launch_bounds__(256) k_step_lane(const KArgs a, const int slot, const void* __restrict__ given) {
  using L = Lane<Env>;
  using St = typename L::St;
  const int lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a.t_dev && e == 0) *a.t_dev += 1;  // device clock: nothing in this kernel reads it
  if (e - lane >= a.E) return;  // whole warp past the last replica
  const bool live = e < a.E;
  const int64_t ec = live ? e : a.E - 1;
  const uint32_t eg = (uint32_t)(a.offset + ec);
  const Key key{a.k0, a.k1};
  const size_t idx = (size_t)slot * (size_t)a.E + (size_t)ec;
  StatsWindow win;
  win.init(warp_window());
  St s;
  L::load(a.state + ec * L::S, s);
  int32_t ep_step = a.ep_step[ec];
  uint32_t rc = a.reset_count[ec];
  float ep_ret = a.ep_ret[ec];
  if (live) L::obs_store(a.obs + idx * L::D, s, false);
  bool term = false, ok;
  float r = 0.0f;
  St s2 = s;
  if constexpr (L::kDiscrete) {
    int act = given ? reinterpret_cast<const int32_t*>(given)[ec] : reinterpret_cast<const int32_t*>(a.act)[idx];
    if (given && live) {
      reinterpret_cast<int32_t*>(a.act)[idx] = act;
      if (a.write_logp) a.logp[idx] = __int_as_float(0x7fc00000);
    }
    ok = L::valid(act);
    L::template step<false>(s2, ok ? act : 0, r, term);
  } else {
    constexpr int DIM = L::kDim;
    float act[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      act[k] = given ? reinterpret_cast<const float*>(given)[ec * DIM + k]
                     : reinterpret_cast<const float*>(a.act)[idx * DIM + k];
      if (given && live) reinterpret_cast<float*>(a.act)[idx * DIM + k] = act[k];
    }
    if (given && live && a.write_logp) a.logp[idx] = __int_as_float(0x7fc00000);
    ok = L::step_c(s2, act, r, term);
  }
  const int32_t es = ep_step + 1;
  const uint32_t d = ok ? ((term ? 1u : 0u) | (es >= a.max_steps ? 2u : 0u)) : 0u;
  const float ret = ep_ret + r;
  const float rw = ok ? r : 0.0f;
  if (d) L::init(key, eg, rc + 1, s2);
  if (live) {
    if (ok) {
      L::save(a.state + e * L::S, s2);
      a.ep_step[e] = d ? 0 : es;
      a.reset_count[e] = rc + (d ? 1u : 0u);
      a.ep_ret[e] = d ? 0.0f : ret;
      L::obs_store(a.obs_live + e * L::D, s2, false);
    } else {
      atomicOr(a.err, kErrAction);
    }
    a.rew[idx] = rw;
    a.done[idx] = (uint8_t)d;
  }
  win.put(0, lane, (live && d) ? (uint32_t)es : 0u, (live && d) ? ret : 0.0f, live ? rw : 0.0f);
  win.flush(lane, 0, 0, slot, a.stats);
}

template <class Env>
__global__ void k_reset_lane(const KArgs a) {
  using L = Lane<Env>;
  using St = typename L::St;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.E) return;
  St s;
  L::init(Key{a.k0, a.k1}, (uint32_t)(a.offset + e), 0u, s);
  L::save(a.state + e * L::S, s);
  a.ep_step[e] = 0;
  a.reset_count[e] = 0;
  a.ep_ret[e] = 0.0f;
  L::obs_store(a.obs_live + e * L::D, s, false);
}

// =======================================================================================
// Tag gridworld (R22): one CTA per replica, one thread per agent.
// =======================================================================================
enum TagMode : int { kTagRollout = 0, kTagStepSlab = 1, kTagStepGiven = 2 };
constexpr int kTagN = 5;

// Shared memory of k_tag: occupancy grids taggers_on / tagged_on [G*G] ints, the reduction
// buffer (3 int64 per warp) and the observation table x / (G - 1) for x in [0, G).
__host__ __device__ inline int tag_red_offset(int G) { return 2 * G * G + ((2 * G * G) & 1); }  // in ints
__host__ __device__ inline int tag_tab_offset(int G, int nwarps) { return tag_red_offset(G) + 6 * nwarps; }

// NEXT-N1 for the multi-agent env: the R29 policy of one agent on its observation o[D]
// (weights `sw` = W1 [D][H] | b1 | W2 [H][N] | b2 (| wv [H] | bv)), in R29 / R29's operation order:
// the probabilities p_i = e_i / S with e_i = (float)exp((double)(l_i - m)), as the fp64-prefix
// CDF of the R13 sampler; v = the R31 critic when kCritic.
template <int D, int H, int N, bool kCritic>
__device__ __forceinline__ void policy_cdf(const float* sw, const float (&o)[D], RowCDF<N>& cdf, float& v) {
  const float* W1 = sw;
  const float* b1 = W1 + D * H;
  const float* W2 = b1 + H;
  const float* b2 = W2 + H * N;
  const float* wv = b2 + N;
  float hid[H];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    float acc = b1[j];
#pragma unroll
    for (int k = 0; k < D; ++k) acc = __fmaf_rn(W1[k * H + j], o[k], acc);
    hid[j] = acc > 0.0f ? acc : 0.0f;
  }
  if (kCritic) v = quarter_dot<H>(wv, 1, hid, wv[H]);
  float lg[N];  // R29' quarter sums
#pragma unroll
  for (int i = 0; i < N; ++i) lg[i] = quarter_dot<H>(W2 + i, N, hid, b2[i]);
  float m = lg[0];
#pragma unroll
  for (int i = 1; i < N; ++i) m = lg[i] > m ? lg[i] : m;
  float S = 0.0f;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    cdf.P[i] = (float)exp((double)fsub(lg[i], m));
    S = fadd(S, cdf.P[i]);
  }
  double run = 0.0;
  bool badp = false;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    cdf.P[i] = fdiv(cdf.P[i], S);
    run += (double)cdf.P[i];
    cdf.C[i] = run;
    badp = badp || !(cdf.P[i] >= 0.0f) || !isfinite(cdf.P[i]);
  }
  cdf.bad = badp || !(run > 0.0) || !isfinite(run);
}

// kHoisted: roll-out with per-step-constant probabilities (thresholds hoisted, no per-step
// CDF code in the kernel); otherwise the general kernel (per-step rows, ws_step modes).
// kPolH > 0 (NEXT-N1, R29 / R36): every agent thread draws its action from the R29 policy
// (hidden kPolH, weights in `given`, staged in shared memory after the observation table)
// on its pre-step observation; kCritic also writes values [T, E, A] and bootstrap [E, A].
template <int kMaxThreads, int kMinBlocks, bool kHoisted, int kPolH, bool kCritic>
__global__ void __launch_bounds__(kMaxThreads, kMinBlocks) k_tag(const KArgs a, const int mode, const int T, const uint64_t t0,
                                              const int slot0, const float* __restrict__ probs,
                                              const int64_t row_stride, const int64_t step_stride,
                                              const void* __restrict__ given, float* __restrict__ values,
                                              float* __restrict__ bootstrap) {
  extern __shared__ int smem[];
  if (a.t_dev && mode != kTagRollout && blockIdx.x == 0 && threadIdx.x == 0) *a.t_dev += 1;  // device clock
  const int G = a.p0, NT = a.p1, A = a.A;
  const int nwarps = blockDim.x >> 5;
  int* taggers_on = smem;
  int* tagged_on = smem + G * G;
  long long* red = reinterpret_cast<long long*>(smem + tag_red_offset(G));
  float* obs_tab = reinterpret_cast<float*>(smem + tag_tab_offset(G, nwarps));
  const int64_t e = blockIdx.x;
  const int ag = threadIdx.x;
  const int lane = ag & 31, wid = ag >> 5;
  const bool is_agent = ag < A;
  const bool tagger = ag < NT;
  const uint32_t eg = (uint32_t)(a.offset + e);
  const Key key{a.k0, a.k1};

  // the grids start empty and every step removes its own marks (see below); the coordinate
  // observations are the G values x / (G - 1) (IEEE division, R22), tabulated once
  for (int i = ag; i < 2 * G * G; i += blockDim.x) smem[i] = 0;
  for (int i = ag; i < G; i += blockDim.x) obs_tab[i] = (float)i / (float)(G - 1);
  constexpr int kPolHH = kPolH > 0 ? kPolH : 1;
  constexpr int kNW = 4 * kPolHH + kPolHH + kPolHH * kTagN + kTagN + (kCritic ? kPolHH + 1 : 0);
  float* sw = obs_tab + G;  // policy weights (kPolH > 0)
  if (kPolH > 0)
    for (int i = ag; i < kNW; i += blockDim.x) sw[i] = reinterpret_cast<const float*>(given)[i];

  int32_t x = 0, y = 0, active = 0;
  if (is_agent) {
    const int32_t* ts = a.tstate + ((size_t)e * A + ag) * 3;
    x = ts[0];
    y = ts[1];
    active = ts[2];
  }
  int32_t ep_step = a.ep_step[e];
  uint32_t rc = a.reset_count[e];
  float ep_ret = is_agent ? a.ep_ret[e * A + ag] : 0.0f;
  const int n_runners = A - NT;

  Thresholds<kTagN> th;
  const int64_t row0 = e * A;  // rows of this replica
  constexpr bool hoisted = kHoisted;  // == (mode == kTagRollout && step_stride == 0)
  if (hoisted) {
    RowCDF<kTagN> cdf;
    warp_row_cdf<kTagN>(probs + row0 * row_stride, row_stride, (int64_t)(ag - lane), A, lane, cdf);
    make_thresholds<kTagN>(cdf, th);
  }
  // with fixed probabilities an invalid row is invalid at every step: one vote up front
  const bool any_bad_rows = hoisted ? (__syncthreads_or(is_agent && th.bad) != 0) : false;
  __syncthreads();
  U4 w{0, 0, 0, 0};
  for (int c = 0; c < T; ++c) {
    const int slot = slot0 + c;
    const uint64_t t = t0 + (uint64_t)c;
    const size_t idx = ((size_t)slot * (size_t)a.E + (size_t)e) * (size_t)A + (size_t)ag;
    int act = 0;
    bool bad_probs = false;
    if (kHoisted || mode == kTagRollout) {
      if (c == 0 || (t & 3) == 0) w = block(key, t >> 2, eg, (uint32_t)ag, kAction);
      const uint32_t word = pick(w, (uint32_t)(t & 3));
      float lp;
      if constexpr (kPolH > 0) {  // the agent's policy on its pre-step observation (R22 obs)
        const float o[4] = {obs_tab[x], obs_tab[y], tagger ? 1.0f : 0.0f, active ? 1.0f : 0.0f};
        RowCDF<kTagN> cdf;
        float v = 0.0f;
        policy_cdf<4, kPolHH, kTagN, kCritic>(sw, o, cdf, v);
        bad_probs = cdf.bad;
        act = search<kTagN>(cdf, u01(word));
        lp = logp_of_normalised<kTagN>(cdf, act);
        if (kCritic && is_agent) st_cs(values + idx, v);
      } else if (kHoisted) {
        act = search_k<kTagN>(th, word >> 8, lp);
        bad_probs = th.bad;
      } else {
        RowCDF<kTagN> cdf;
        warp_row_cdf<kTagN>(probs + (int64_t)c * step_stride + row0 * row_stride, row_stride,
                            (int64_t)(ag - lane), A, lane, cdf);
        bad_probs = cdf.bad;
        act = search<kTagN>(cdf, u01(word));
        lp = logp_of<kTagN>(cdf, act);
      }
      if (bad_probs) {
        act = -1;
        lp = __int_as_float(0x7fc00000);
      }
      if (is_agent) {
        st_cs(reinterpret_cast<int32_t*>(a.act) + idx, act);
        if (a.write_logp) st_cs(a.logp + idx, lp);
      }
    } else if (is_agent) {
      if (mode == kTagStepGiven) {
        act = reinterpret_cast<const int32_t*>(given)[e * A + ag];
        reinterpret_cast<int32_t*>(a.act)[idx] = act;
        if (a.write_logp) a.logp[idx] = __int_as_float(0x7fc00000);
      } else {
        act = reinterpret_cast<const int32_t*>(a.act)[idx];
      }
    }
    // pre-step observation (x/(G-1), y/(G-1), is_tagger, active)  (R22)
    if (is_agent) {
      const float4 o = make_float4(obs_tab[x], obs_tab[y], tagger ? 1.0f : 0.0f, active ? 1.0f : 0.0f);
      st_cs(reinterpret_cast<float4*>(a.obs) + idx, o);
    }
    const bool invalid = is_agent && (act < 0 || act > 4);
    const bool any_invalid = hoisted ? any_bad_rows : (__syncthreads_or(invalid) != 0);
    float r = 0.0f;
    uint8_t d = 0;
    if (!any_invalid) {
      // simultaneous moves, clipped to the grid; tagged runners frozen;
      // branch-free: N (y+1), S (y-1), E (x+1), W (x-1), stay
      const bool mv = is_agent && (tagger || active);
      const int dxv = (act == 3 ? 1 : 0) - (act == 4 ? 1 : 0), dyv = (act == 1 ? 1 : 0) - (act == 2 ? 1 : 0);
      x = mv ? min(max(x + dxv, 0), G - 1) : x;
      y = mv ? min(max(y + dyv, 0), G - 1) : y;
      const int cell = y * G + x;
      if (is_agent && tagger) atomicAdd(&taggers_on[cell], 1);
      __syncthreads();
      bool newly = false;
      if (is_agent && !tagger && active) {
        newly = taggers_on[cell] >= 1;
        r = newly ? -1.0f : 0.01f;
        active = newly ? 0 : active;
        if (newly) atomicAdd(&tagged_on[cell], 1);
      }
      __syncthreads();
      if (is_agent && tagger) r = (float)tagged_on[cell] / (float)taggers_on[cell];
      if (is_agent) ep_ret = ep_ret + r;
      // A8 + termination in ONE CTA barrier: per warp the exact fixed-point reward sum (REDUX,
      // warp_sum_u64) and the count of still-active runners; every thread adds the partials
      const unsigned long long wrs = warp_sum_u64(is_agent ? (unsigned long long)to_fx(r) : 0ull);
      const int wst = __popc(__ballot_sync(kFull, is_agent && !tagger && active));
      if (lane == 0) {
        red[3 * wid] = (long long)wrs;
        red[3 * wid + 2] = wst;
      }
      __syncthreads();
      long long srs = 0, still = 0;
      for (int i = 0; i < nwarps; ++i) {
        srs += red[3 * i];
        still += red[3 * i + 2];
      }
      // every reader of the grids is past that barrier: remove this step's marks, so the grids
      // are empty again before the next step's first barrier (adds commute)
      if (is_agent && tagger) atomicAdd(&taggers_on[cell], -1);
      if (newly) atomicAdd(&tagged_on[cell], -1);
      const bool term = n_runners > 0 && still == 0;
      ep_step += 1;
      const bool trunc = ep_step >= a.max_steps;
      d = (uint8_t)((term ? 1 : 0) | (trunc ? 2 : 0));
      long long srt = 0;
      if (d) {  // episode ended (CTA-uniform, once per episode): sum of the agents' returns
        const unsigned long long wrt = warp_sum_u64(is_agent ? (unsigned long long)to_fx(ep_ret) : 0ull);
        if (lane == 0) red[3 * wid + 1] = (long long)wrt;
        __syncthreads();
        if (threadIdx.x == 0)
          for (int i = 0; i < nwarps; ++i) srt += red[3 * i + 1];
      }
      if (threadIdx.x == 0) {
        unsigned long long* st = a.stats + (size_t)slot * 4;
        if (d) {
          atomicAdd(st + kStEpisodes, 1ull);
          atomicAdd(st + kStLength, (unsigned long long)ep_step);
          if (srt) atomicAdd(st + kStReturn, (unsigned long long)srt);
        }
        if (srs) atomicAdd(st + kStReward, (unsigned long long)srs);
      }
    } else {
      if (threadIdx.x == 0) atomicOr(a.err, kErrAction | (mode == kTagRollout && bad_probs ? kErrProbs : 0u));
    }
    if (is_agent) st_cs(a.rew + idx, r);
    if (threadIdx.x == 0) st_cs_u8(a.done + ((size_t)slot * (size_t)a.E + (size_t)e), d);
    if (d) {  // A5 auto-reset, uniform across the CTA
      rc += 1;
      if (is_agent) {
        const U4 b = block(key, rc >> 1, eg, (uint32_t)ag, kReset);  // draws j = rc*2 + {0,1}
        const uint32_t wx = (rc & 1) ? b.z : b.x, wy = (rc & 1) ? b.w : b.y;
        x = (int32_t)__umulhi(wx, (uint32_t)G);
        y = (int32_t)__umulhi(wy, (uint32_t)G);
        active = 1;
      }
      ep_step = 0;
      ep_ret = 0.0f;
    }
    // (the reduction buffer is next written after the next valid step's first barrier, which
    // every thread reaches only after reading it)
  }
  if (kCritic && is_agent) {  // bootstrap value of the observation after the last step
    const float o[4] = {obs_tab[x], obs_tab[y], tagger ? 1.0f : 0.0f, active ? 1.0f : 0.0f};
    RowCDF<kTagN> cdf;
    float v = 0.0f;
    policy_cdf<4, kPolHH, kTagN, kCritic>(sw, o, cdf, v);
    bootstrap[e * A + ag] = v;
  }
  if (is_agent) {
    int32_t* ts = a.tstate + ((size_t)e * A + ag) * 3;
    ts[0] = x;
    ts[1] = y;
    ts[2] = active;
    a.ep_ret[e * A + ag] = ep_ret;
    reinterpret_cast<float4*>(a.obs_live)[e * A + ag] =
        make_float4(obs_tab[x], obs_tab[y], tagger ? 1.0f : 0.0f, active ? 1.0f : 0.0f);
  }
  if (threadIdx.x == 0) {
    a.ep_step[e] = ep_step;
    a.reset_count[e] = rc;
  }
}

__global__ void k_reset_tag(const KArgs a) {
  const int64_t e = blockIdx.x;
  const int ag = threadIdx.x;
  const int G = a.p0, NT = a.p1, A = a.A;
  if (ag < A) {
    const U4 b = block(Key{a.k0, a.k1}, 0, (uint32_t)(a.offset + e), (uint32_t)ag, kReset);
    const int32_t x = (int32_t)__umulhi(b.x, (uint32_t)G), y = (int32_t)__umulhi(b.y, (uint32_t)G);
    int32_t* ts = a.tstate + ((size_t)e * A + ag) * 3;
    ts[0] = x;
    ts[1] = y;
    ts[2] = 1;
    a.ep_ret[e * A + ag] = 0.0f;
    const float inv = (float)(G - 1);
    reinterpret_cast<float4*>(a.obs_live)[e * A + ag] =
        make_float4((float)x / inv, (float)y / inv, ag < NT ? 1.0f : 0.0f, 1.0f);
  }
  if (ag == 0) {
    a.ep_step[e] = 0;
    a.reset_count[e] = 0;
  }
}

// =======================================================================================
// Test hooks.
// =======================================================================================
__global__ void k_test_philox(const uint32_t* rows, int64_t n, uint32_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* r = rows + i * 6;
  const U4 v = philox(r[0], r[1], r[2], r[3], r[4], r[5]);
  out[i * 4 + 0] = v.x;
  out[i * 4 + 1] = v.y;
  out[i * 4 + 2] = v.z;
  out[i * 4 + 3] = v.w;
}

// every lane loads the same row (row_stride 0); thread i handles draws k = i, i + stride...
// Both the direct search and the hoisted thresholds are evaluated; a disagreement is
// counted in counts[n] (must stay 0).
template <int N>
__global__ void k_test_sample_grid(const float* p, int64_t* counts) {
  __shared__ unsigned long long local[N + 1];
  if (threadIdx.x <= N) local[threadIdx.x] = 0;
  __syncthreads();
  RowCDF<N> cdf;
  warp_row_cdf<N>(p, 0, 0, 1 << 30, threadIdx.x & 31, cdf);
  Thresholds<N> th;
  make_thresholds<N>(cdf, th);
  unsigned long long mine[N + 1];
#pragma unroll
  for (int i = 0; i <= N; ++i) mine[i] = 0;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < (1u << 24); k += gridDim.x * blockDim.x) {
    const int a1 = search<N>(cdf, (float)k * (1.0f / 16777216.0f));
    float lp;
    const int a2 = search_k<N>(th, k, lp);
#pragma unroll
    for (int i = 0; i < N; ++i) mine[i] += (a1 == i);
    mine[N] += (a1 != a2);
  }
#pragma unroll
  for (int i = 0; i <= N; ++i) atomicAdd(&local[i], mine[i]);
  __syncthreads();
  if (threadIdx.x <= N) atomicAdd(reinterpret_cast<unsigned long long*>(counts) + threadIdx.x, local[threadIdx.x]);
}

// elementary functions of the hot path, for the exhaustive / library comparisons
__device__ __forceinline__ float unary(int fn, float x, float p) {
  float s, c;
  switch (fn) {
    case 0: CartPole::sincos_theta(x, s, c); return s;
    case 1: CartPole::sincos_theta(x, c, s); return s;  // cos
    case 2: return CartPole::div_total_mass(x);
    case 3: return __fdiv_rn(x, CartPole::total_mass);
    case 4: return sin_c(x);
    case 5: return cos_c(x);
    case 6: return div_normal(x, p);
    case 7: return __fdiv_rn(x, p);
    case 8: return CartPole::div_total_mass_any(x);
    default: return 0.0f;
  }
}

__global__ void k_test_unary(int fn, float p, const float* x, int64_t n, float* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = unary(fn, x[i], p);
}

// counts bit patterns b in [lo, hi] where fn_a(x) and fn_b(x) differ (NaN == NaN)
__global__ void k_test_exhaustive(int fa, int fb, float p, uint32_t lo, uint32_t hi, unsigned long long* mism) {
  unsigned long long m = 0;
  const uint64_t n = (uint64_t)hi - lo + 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const float x = __uint_as_float((uint32_t)(lo + i));
    const float ya = unary(fa, x, p), yb = unary(fb, x, p);
    m += (__float_as_uint(ya) != __float_as_uint(yb)) && !(isnan(ya) && isnan(yb));
  }
  m = __reduce_add_sync(kFull, (unsigned)m);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(mism, m);
}

// =======================================================================================
// Host launchers.
// =======================================================================================
#define WS_SURFACE_DISPATCH(D, MACRO) \
  switch (D) {                        \
    case 2: MACRO(2); break;          \
    case 3: MACRO(3); break;          \
    case 4: MACRO(4); break;          \
    case 8: MACRO(8); break;          \
    case 16: MACRO(16); break;        \
    case 20: MACRO(20); break;        \
    case 32: MACRO(32); break;        \
    default: return cudaErrorInvalidValue; \
  }

static inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// up to about one warp per SM sub-partition the fused roll-out is latency-bound and uses its
// latency build; beyond, the throughput build
constexpr int64_t kLatencyReplicas = 148 * 4 * 32;

static size_t tag_smem(const KArgs& a, int block) {
  return (size_t)(tag_tab_offset(a.p0, block / 32) + a.p0) * sizeof(int);
}
static int tag_block(const KArgs& a) { return ((a.A + 31) / 32) * 32; }

// CTA per replica (A threads rounded up to a warp multiple)
static void tag_launch(const KArgs& a, const Launch& l, int b, int mode, int T, uint64_t t0, int slot0,
                       const float* probs, int64_t row_stride, int64_t step_stride, const void* given) {
#ifndef WS_TAG_MINB
#define WS_TAG_MINB 7
#endif
#define WS_TAG_LAUNCH(MT, MB, H)                                                                        \
  k_tag<MT, MB, H, 0, false><<<(unsigned)a.E, b, tag_smem(a, b), l.stream>>>(a, mode, T, t0, slot0, probs,     \
                                                                            row_stride, step_stride, given, \
                                                                            nullptr, nullptr)
  const bool h = mode == kTagRollout && step_stride == 0;
  if (b <= 128) {  // 6 CTAs of 128 threads per SM (measured best for C4: 7 and 8 force spills / fewer registers)
    if (h) WS_TAG_LAUNCH(128, WS_TAG_MINB, true); else WS_TAG_LAUNCH(128, WS_TAG_MINB, false);
  } else if (b <= 256) {
    if (h) WS_TAG_LAUNCH(256, 1, true); else WS_TAG_LAUNCH(256, 1, false);
  } else {
    if (h) WS_TAG_LAUNCH(1024, 1, true); else WS_TAG_LAUNCH(1024, 1, false);
  }
#undef WS_TAG_LAUNCH
}

// NEXT-N1 / R36: the tag roll-out with every agent's action from the in-kernel policy
static cudaError_t tag_policy_launch(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* weights,
                                     int hidden, float* values, float* bootstrap) {
  const int b = tag_block(a);
  if (b > 128) return cudaErrorInvalidValue;  // up to 128 agents per replica (launch bounds of the policy build)
  const size_t smem = tag_smem(a, b) + (size_t)(4 * hidden + hidden + hidden * kTagN + kTagN + hidden + 1) * 4;
#define WS_TAG_POL(HH, C)                                                                                   \
  k_tag<128, 4, false, HH, C><<<(unsigned)a.E, b, smem, l.stream>>>(a, kTagRollout, T, t0, 0, nullptr, 0, 0, weights, \
                                                                  values, bootstrap)
  if (values) {
    if (hidden == 32) WS_TAG_POL(32, true); else WS_TAG_POL(64, true);
  } else {
    if (hidden == 32) WS_TAG_POL(32, false); else WS_TAG_POL(64, false);
  }
#undef WS_TAG_POL
  return cudaGetLastError();
}

// lane kernels carry one statistics window per warp in dynamic shared memory
template <typename... Params, typename... Args>
static cudaError_t launch_lane(void (*k)(Params...), int64_t E, const Launch& l, Args... args) {
  const size_t smem = (size_t)(l.block / 32) * kWinWords * sizeof(uint32_t) + 256 * sizeof(unsigned long long);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<grid_for(E, l.block), l.block, smem, l.stream>>>(args...);
  return cudaGetLastError();
}

cudaError_t launch_reset(const KArgs& a, const Launch& l, uint64_t* launches) {
  const unsigned g = grid_for(a.E, l.block);
  l.m(kKReset, 0);
  switch (l.kind) {
    case kCartPole: k_reset_lane<CartPole><<<g, l.block, 0, l.stream>>>(a); break;
    case kAcrobot: k_reset_lane<Acrobot><<<g, l.block, 0, l.stream>>>(a); break;
    case kPendulum: k_reset_lane<Pendulum><<<g, l.block, 0, l.stream>>>(a); break;
    case kDummy: k_reset_lane<Dummy><<<g, l.block, 0, l.stream>>>(a); break;
    case kSurface: {
#define M(DD) k_reset_lane<Surface<DD>><<<g, l.block, 0, l.stream>>>(a)
      WS_SURFACE_DISPATCH(a.p0, M)
#undef M
      break;
    }
    case kTag: k_reset_tag<<<(unsigned)a.E, tag_block(a), 0, l.stream>>>(a); break;
  }
  l.m(kKReset, 1);
  *launches += 1;
  return cudaGetLastError();
}

// the plan kernel alone, for the runtime-composed (NVRTC) roll-out of a registered discrete env
// with constant probabilities (NEXT-N4): act / logp slabs and the packed plan, n_actions 2..8
cudaError_t launch_plan(const KArgs& a, int n_actions, int T, uint64_t t0, const float* probs, int64_t row_stride,
                        cudaStream_t s) {
  const dim3 grid(grid_for(a.E, 128), (unsigned)((T + kPlanChunk - 1) / kPlanChunk));
  switch (n_actions) {
#define WS_PLAN_N(NN) \
  case NN: k_plan_discrete<NN, false><<<grid, 128, 0, s>>>(a, T, t0, probs, row_stride, 0, 0); break;
    WS_PLAN_N(2) WS_PLAN_N(3) WS_PLAN_N(4) WS_PLAN_N(5) WS_PLAN_N(6) WS_PLAN_N(7) WS_PLAN_N(8)
#undef WS_PLAN_N
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <class Env>
static cudaError_t rollout_discrete(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* probs,
                                    int64_t row_stride, int64_t step_stride, uint64_t* launches) {
  constexpr int N = Lane<Env>::N;
  const dim3 grid(grid_for(a.E, 128), (unsigned)((T + kPlanChunk - 1) / kPlanChunk));
  l.m(kKPlan, 0);
  if (step_stride == 0)
    k_plan_discrete<N, false><<<grid, 128, 0, l.stream>>>(a, T, t0, probs, row_stride, step_stride, 1);
  else
    k_plan_discrete<N, true><<<grid, 128, 0, l.stream>>>(a, T, t0, probs, row_stride, step_stride, 1);
  l.m(kKPlan, 1);
  *launches += 1;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  l.m(kKRollout, 0);
  // results do not depend on the CTA size or the build (launch-shape invariance tests)
  const int block = l.block < Lane<Env>::kMaxThreads ? l.block : Lane<Env>::kMaxThreads;
  const bool lat = a.E <= kLatencyReplicas;
  const int rows = lat ? Lane<Env>::kWinRowsLat : Lane<Env>::kWinRowsThr;
  void (*k)(const KArgs, const int) = lat ? k_rollout_discrete<Env, true> : k_rollout_discrete<Env, false>;
  const size_t smem = (size_t)(block / 32) * 3 * rows * kWinStride * sizeof(uint32_t) + 256 * sizeof(unsigned long long);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<grid_for(a.E, block), block, smem, l.stream>>>(a, T);
  l.m(kKRollout, 1);
  return cudaGetLastError();
}

template <class Env>
static cudaError_t rollout_continuous(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* probs,
                                      int64_t row_stride, int64_t step_stride, uint64_t* launches) {
  constexpr int DIM = Lane<Env>::kDim;
  const dim3 grid(grid_for(a.E, 128), (unsigned)((T + kGaussChunk - 1) / kGaussChunk));
  l.m(kKPlan, 0);
  if (step_stride == 0)
    k_plan_gauss<DIM, false><<<grid, 128, 0, l.stream>>>(a, T, t0, probs, row_stride, step_stride);
  else
    k_plan_gauss<DIM, true><<<grid, 128, 0, l.stream>>>(a, T, t0, probs, row_stride, step_stride);
  l.m(kKPlan, 1);
  *launches += 1;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  l.m(kKRollout, 0);
  const size_t smem = (size_t)(l.block / 32) * 3 * kContWinRows * kWinStride * sizeof(uint32_t);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k_rollout_continuous<Env>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_rollout_continuous<Env><<<grid_for(a.E, l.block), l.block, smem, l.stream>>>(a, T);
  l.m(kKRollout, 1);
  return cudaGetLastError();
}

template <int D>
static cudaError_t rollout_surface(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* probs,
                                   int64_t row_stride, int64_t step_stride, uint64_t* launches) {
  const dim3 pgrid(grid_for(a.E, 4), (unsigned)((T + kGaussChunk - 1) / kGaussChunk));
  l.m(kKPlan, 0);
  if (step_stride == 0)
    k_plan_gauss_warp<D, false><<<pgrid, 128, 0, l.stream>>>(a, T, t0, probs, row_stride, step_stride);
  else
    k_plan_gauss_warp<D, true><<<pgrid, 128, 0, l.stream>>>(a, T, t0, probs, row_stride, step_stride);
  l.m(kKPlan, 1);
  *launches += 1;
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  const int wpb = l.block / 32;  // warps per CTA
  l.m(kKRollout, 0);
  {  // segments of ceil(D/4) lanes, 32 / ceil(D/4) replicas per warp
    // CTA statistics accumulator + one 16-slot statistics window per warp (energies via shuffles)
    // (+ D % 4 == 0: the per-warp cp.async action ring, 2 x 8 x 32 float4)
    const size_t smem = 256 * sizeof(unsigned long long) + (size_t)wpb * 3 * 16 * kWinStride * sizeof(uint32_t) +
                        (D % 4 == 0 ? (size_t)wpb * 2 * WS_SURF_TRIP * 32 * sizeof(float4) : 0);
    if (smem > 48 * 1024) {
      const cudaError_t e = cudaFuncSetAttribute(k_rollout_surface_seg<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_rollout_surface_seg<D><<<grid_for(a.E, (int64_t)wpb * SurfSeg<D>::R), l.block, smem, l.stream>>>(a, T);
  }
  l.m(kKRollout, 1);
  return cudaGetLastError();
}

cudaError_t launch_test_surface_energy(const float* q, int D, int64_t n, float* energy, double* spring,
                                      cudaStream_t s) {
#define M(DD) k_test_surface_energy<DD><<<grid_for(n, 4 * SurfSeg<DD>::R), 128, 0, s>>>(q, n, energy, spring)
  WS_SURFACE_DISPATCH(D, M)
#undef M
  return cudaGetLastError();
}

cudaError_t launch_rollout(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* probs,
                           int64_t row_stride, int64_t step_stride, uint64_t* launches) {
  cudaError_t err = cudaSuccess;
  switch (l.kind) {
    case kCartPole: err = rollout_discrete<CartPole>(a, l, T, t0, probs, row_stride, step_stride, launches); break;
    case kAcrobot: err = rollout_discrete<Acrobot>(a, l, T, t0, probs, row_stride, step_stride, launches); break;
    case kDummy: err = rollout_discrete<Dummy>(a, l, T, t0, probs, row_stride, step_stride, launches); break;
    case kPendulum: err = rollout_continuous<Pendulum>(a, l, T, t0, probs, row_stride, step_stride, launches); break;
    case kSurface: {
#define M(DD) err = rollout_surface<DD>(a, l, T, t0, probs, row_stride, step_stride, launches)
      WS_SURFACE_DISPATCH(a.p0, M)
#undef M
      break;
    }
    case kTag: {
      const int b = tag_block(a);
      l.m(kKRollout, 0);
      tag_launch(a, l, b, kTagRollout, T, t0, 0, probs, row_stride, step_stride, nullptr);
      l.m(kKRollout, 1);
      err = cudaGetLastError();
      break;
    }
  }
  *launches += 1;
  return err;
}

template <class Env>
static cudaError_t rollout_policy(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* weights,
                                  int hidden, float* values, float* bootstrap, float* vtr) {
  // warp-specialised: one env warp + four inference warps + one store warp per 32 replicas; the
  // store warp's 16-row statistics window is the dynamic shared memory
  const size_t smem = (size_t)3 * 16 * kWinStride * sizeof(uint32_t);
  const unsigned g = grid_for(a.E, 32);
  l.m(kKRollout, 0);
  if (values) {
    switch (hidden) {
      case 32: k_rollout_policy_ws<Env, 32, true><<<g, 192, smem, l.stream>>>(a, T, t0, weights, values, bootstrap, vtr); break;
      case 64: k_rollout_policy_ws<Env, 64, true><<<g, 192, smem, l.stream>>>(a, T, t0, weights, values, bootstrap, vtr); break;
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (hidden) {
      case 32: k_rollout_policy_ws<Env, 32, false><<<g, 192, smem, l.stream>>>(a, T, t0, weights, nullptr, nullptr, nullptr); break;
      case 64: k_rollout_policy_ws<Env, 64, false><<<g, 192, smem, l.stream>>>(a, T, t0, weights, nullptr, nullptr, nullptr); break;
      default: return cudaErrorInvalidValue;
    }
  }
  l.m(kKRollout, 1);
  return cudaGetLastError();
}

static cudaError_t rollout_gpolicy(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* weights,
                                   int hidden, float* values, float* bootstrap, float* vtr) {
  const size_t smem = (size_t)4 * 3 * kContWinRows * kWinStride * sizeof(uint32_t);  // 4 warps' windows
  const unsigned g = grid_for(a.E, 128);
  l.m(kKRollout, 0);
  if (values) {
    switch (hidden) {
      case 32: k_rollout_gpolicy<32, true><<<g, 128, smem, l.stream>>>(a, T, t0, weights, values, bootstrap, vtr); break;
      case 64: k_rollout_gpolicy<64, true><<<g, 128, smem, l.stream>>>(a, T, t0, weights, values, bootstrap, vtr); break;
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (hidden) {
      case 32: k_rollout_gpolicy<32, false><<<g, 128, smem, l.stream>>>(a, T, t0, weights, nullptr, nullptr, nullptr); break;
      case 64: k_rollout_gpolicy<64, false><<<g, 128, smem, l.stream>>>(a, T, t0, weights, nullptr, nullptr, nullptr); break;
      default: return cudaErrorInvalidValue;
    }
  }
  l.m(kKRollout, 1);
  return cudaGetLastError();
}

cudaError_t launch_rollout_policy(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* weights,
                                  int hidden, uint64_t* launches, float* values, float* bootstrap, float* vtr) {
  cudaError_t err = cudaErrorInvalidValue;
  switch (l.kind) {
    case kPendulum: err = rollout_gpolicy(a, l, T, t0, weights, hidden, values, bootstrap, vtr); break;
    case kTag:
      l.m(kKRollout, 0);
      err = tag_policy_launch(a, l, T, t0, weights, hidden, values, bootstrap);
      l.m(kKRollout, 1);
      break;
    case kCartPole: err = rollout_policy<CartPole>(a, l, T, t0, weights, hidden, values, bootstrap, vtr); break;
    case kAcrobot: err = rollout_policy<Acrobot>(a, l, T, t0, weights, hidden, values, bootstrap, vtr); break;
    case kDummy: err = rollout_policy<Dummy>(a, l, T, t0, weights, hidden, values, bootstrap, vtr); break;
    default: break;
  }
  *launches += 1;
  return err;
}

cudaError_t launch_sample(const KArgs& a, const Launch& l, int slot, uint64_t t, const float* probs,
                          int64_t row_stride, uint64_t* launches) {
  const int64_t rows = a.E * (int64_t)a.A;
  const unsigned g = grid_for(rows, 256);
  l.m(kKSample, 0);
  switch (l.kind) {
    case kCartPole:
    case kDummy: k_sample_discrete<2><<<g, 256, 0, l.stream>>>(a, slot, t, probs, row_stride); break;
    case kAcrobot: k_sample_discrete<3><<<g, 256, 0, l.stream>>>(a, slot, t, probs, row_stride); break;
    case kTag: k_sample_discrete<5><<<g, 256, 0, l.stream>>>(a, slot, t, probs, row_stride); break;
    case kPendulum: k_sample_continuous<1><<<g, 256, 0, l.stream>>>(a, slot, t, probs, row_stride); break;
    case kSurface: {
#define M(DD) k_sample_continuous<DD><<<g, 256, 0, l.stream>>>(a, slot, t, probs, row_stride)
      WS_SURFACE_DISPATCH(a.p0, M)
#undef M
      break;
    }
  }
  l.m(kKSample, 1);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_step(const KArgs& a, const Launch& l, int slot, const void* given, uint64_t* launches) {
  cudaError_t err = cudaSuccess;
  l.m(kKStep, 0);
  switch (l.kind) {
    case kCartPole: err = launch_lane(k_step_lane<CartPole>, a.E, l, a, slot, given); break;
    case kAcrobot: err = launch_lane(k_step_lane<Acrobot>, a.E, l, a, slot, given); break;
    case kDummy: err = launch_lane(k_step_lane<Dummy>, a.E, l, a, slot, given); break;
    case kPendulum: err = launch_lane(k_step_lane<Pendulum>, a.E, l, a, slot, given); break;
    case kSurface: {
#define M(DD) err = launch_lane(k_step_lane<Surface<DD>>, a.E, l, a, slot, given)
      WS_SURFACE_DISPATCH(a.p0, M)
#undef M
      break;
    }
    case kTag: {
      const int b = tag_block(a);
      tag_launch(a, l, b, given ? kTagStepGiven : kTagStepSlab, 1, 0, slot, nullptr, 0, 0, given);
      err = cudaGetLastError();
      break;
    }
  }
  l.m(kKStep, 1);
  *launches += 1;
  return err;
}

// ---------------------------------------------------------------------------------------
// A8 cross-GPU statistics all-reduce over peer memory (one CTA per rank, after the roll-out
// on the same stream).  Buffer of rank r: gather_r[parity][src][t_cap][4] int64, then one
// u64 arrival counter.  Epoch k uses parity k & 1: a rank can be at most one epoch ahead of
// a peer's reader (it must first see that peer's arrival for epoch k-1), so two parities
// suffice.  Sums are exact int64 (R20): the result is identical on every rank and equal to
// the single-GPU statistics of the union of the shards.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) k_peer_allreduce(const unsigned long long* local, const int T,
                                                       const PeerArgs p, const uint64_t epoch,
                                                       unsigned long long* out, uint32_t* err,
                                                       const uint64_t timeout_ns) {
  const int n = T * 4;
  const size_t slice = (size_t)p.t_cap * 4;
  const size_t par = (size_t)(epoch & 1) * (size_t)p.world * slice;
  const size_t counter = 2 * (size_t)p.world * slice;  // arrival counter after both parities
  // 1. publish this rank's slice to every rank (16-byte stores; slices are 32-byte aligned)
  for (int r = 0; r < p.world; ++r) {
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(p.gather[r] + par + (size_t)p.rank * slice);
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(local);
    for (int i = threadIdx.x; i < n / 2; i += blockDim.x) dst[i] = src[i];
  }
  __threadfence_system();
  __syncthreads();
  // 2. signal every rank (release: the barrier orders all threads' fenced stores before it)
  if ((int)threadIdx.x < p.world) atomicAdd_system(p.gather[threadIdx.x] + counter, 1ull);
  // 3. wait until every rank has published epoch `epoch` into this rank's buffer
  __shared__ int timed_out;
  if (threadIdx.x == 0) {
    timed_out = 0;
    const unsigned long long target = (unsigned long long)p.world * (epoch + 1);
    const unsigned long long* c = p.gather[p.rank] + counter;
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(c) < target) {
      if (global_ns() - t0 > timeout_ns) {
        timed_out = 1;
        atomicOr(err, kErrPeer);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
  if (timed_out) return;
  // 4. merged statistics = sum of the slices (exact integers; rank order for definiteness)
  const unsigned long long* g = p.gather[p.rank] + par;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long acc = 0;
    for (int r = 0; r < p.world; ++r) acc += g[(size_t)r * slice + i];
    out[i] = acc;
  }
}

cudaError_t launch_peer_allreduce(const unsigned long long* local, int T, const PeerArgs& p, uint64_t epoch,
                                  unsigned long long* out, uint32_t* err, double timeout_s, cudaStream_t s) {
  k_peer_allreduce<<<1, 256, 0, s>>>(local, T, p, epoch, out, err, (uint64_t)(timeout_s * 1e9));
  return cudaGetLastError();
}

cudaError_t launch_test_philox(const uint32_t* rows, int64_t n, uint32_t* out, cudaStream_t s) {
  k_test_philox<<<grid_for(n, 256), 256, 0, s>>>(rows, n, out);
  return cudaGetLastError();
}

cudaError_t launch_test_sample_grid(const float* p, int n, int64_t* counts, cudaStream_t s) {
  switch (n) {
    case 1: k_test_sample_grid<1><<<592, 256, 0, s>>>(p, counts); break;
    case 2: k_test_sample_grid<2><<<592, 256, 0, s>>>(p, counts); break;
    case 3: k_test_sample_grid<3><<<592, 256, 0, s>>>(p, counts); break;
    case 4: k_test_sample_grid<4><<<592, 256, 0, s>>>(p, counts); break;
    case 5: k_test_sample_grid<5><<<592, 256, 0, s>>>(p, counts); break;
    case 6: k_test_sample_grid<6><<<592, 256, 0, s>>>(p, counts); break;
    case 7: k_test_sample_grid<7><<<592, 256, 0, s>>>(p, counts); break;
    case 8: k_test_sample_grid<8><<<592, 256, 0, s>>>(p, counts); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_test_unary(int fn, float p, const float* x, int64_t n, float* out, cudaStream_t s) {
  k_test_unary<<<grid_for(n, 256), 256, 0, s>>>(fn, p, x, n, out);
  return cudaGetLastError();
}

cudaError_t launch_test_exhaustive(int fa, int fb, float p, uint32_t lo, uint32_t hi, unsigned long long* mism,
                                   cudaStream_t s) {
  k_test_exhaustive<<<148 * 16, 256, 0, s>>>(fa, fb, p, lo, hi, mism);
  return cudaGetLastError();
}

}  // namespace ws
