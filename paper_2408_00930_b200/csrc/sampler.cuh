// sampler.cuh -- A2: action sampling from given policy probabilities ("operating an
// agent that samples actions"; S:322-325 inverse CDF / mean + std * gaussian; BJ:5 "a
// warp-level prefix sum and search over per-agent probabilities").
//
// Discrete rows: a warp loads the probability rows of its 32 owners coalesced (lanes walk
// the flattened (row, action) index, floor(32/N) rows per 32-lane chunk), runs a segmented
// Hillis-Steele inclusive scan in fp64 with __shfl_up_sync, and each owner lane gathers its
// row's CDF with __shfl_sync.  The search then picks min{i : p_i > 0 and u*S < C_i}, with
// the last nonzero action as fallback (R13).  For fp32 inputs whose magnitudes span less
// than 2^29 the fp64 prefix sums are exact, so the result is independent of association
// order and bit-identical to a sequential fp64 CDF (R16).
//
// When the probabilities are the same every step (step_stride 0) the search is hoisted:
// per action i the integer threshold K_i = #{k in [0,2^24) : k 2^-24 S < C_i} is found once
// by bisection on the same fp64 predicate, and each step compares the 24-bit draw k = w>>8
// with K_i -- the identical decision for every k.
#pragma once

#include "common.cuh"

namespace ws {

template <int N>
struct RowCDF {
  double C[N];  // inclusive prefix sums (fp64)
  float P[N];   // the row itself
  bool bad;     // R13: p < 0, NaN / inf, or non-positive / non-finite sum
};

// Rows first_row + r (r = 0..31, row r owned by lane r).  Rows >= n_rows (the tail of the
// last warp) read row n_rows - 1, so tail lanes shadow the last real row exactly.
template <int N>
__device__ __forceinline__ void warp_row_cdf(const float* __restrict__ probs, int64_t row_stride,
                                             int64_t first_row, int64_t n_rows, int lane,
                                             RowCDF<N>& out) {
  static_assert(N >= 1 && N <= 32, "rows of 1..32 actions");
  constexpr int RPC = 32 / N;                 // rows per 32-lane chunk
  constexpr int NCH = (32 + RPC - 1) / RPC;   // chunks covering 32 rows
  const int col = lane % N;
  const int rl = lane / N;
  const int src_base = (lane % RPC) * N;      // where this lane's own row sits in its chunk
  const int my_chunk = lane / RPC;
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int rr = j * RPC + rl;
    const bool valid = (lane < RPC * N) && (rr < 32);
    const int64_t row = min(first_row + rr, n_rows - 1);
    const float p = valid ? __ldg(probs + row * row_stride + col) : 0.0f;
    double v = (double)p;
#pragma unroll
    for (int off = 1; off < N; off <<= 1) {
      const double t = __shfl_up_sync(kFull, v, off);
      if (col >= off) v += t;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double c = __shfl_sync(kFull, v, src_base + i);
      const float pi = __shfl_sync(kFull, p, src_base + i);
      if (my_chunk == j) {
        out.C[i] = c;
        out.P[i] = pi;
      }
    }
  }
  bool bad = false;
#pragma unroll
  for (int i = 0; i < N; ++i) bad = bad || !(out.P[i] >= 0.0f) || !isfinite(out.P[i]);
  const double S = out.C[N - 1];
  out.bad = bad || !(S > 0.0) || !isfinite(S);
}

template <int N>
__device__ __forceinline__ int last_nonzero(const RowCDF<N>& r) {
  int last = 0;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (r.P[i] > 0.0f) last = i;
  return last;
}

// Direct search for uniform u (fp32, exact multiple of 2^-24).
template <int N>
__device__ __forceinline__ int search(const RowCDF<N>& r, float u) {
  const double target = (double)u * r.C[N - 1];
  int a = -1;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (a < 0 && r.P[i] > 0.0f && target < r.C[i]) a = i;
  return a < 0 ? last_nonzero(r) : a;
}

// R13 log-probability: (float)(log p_a - log S), both logs in fp64 (R3).
template <int N>
__device__ __forceinline__ float logp_of(const RowCDF<N>& r, int a) {
  float pa = r.P[0];
#pragma unroll
  for (int i = 1; i < N; ++i)
    if (a == i) pa = r.P[i];
  return (float)(log((double)pa) - log(r.C[N - 1]));
}

// logp_of for a row normalised in fp32 (the policy softmax): the fp64 row sum C = 1 + d with
// |d| ~ 1e-7, so log C = d - d^2/2 + d^3/3 (truncation ~d^4/4, far below an fp64 ulp of
// the result) replaces the second fp64 log; log-probabilities are compared within 2 ulp
// (R18), actions are unaffected.
template <int N>
__device__ __forceinline__ float logp_of_normalised(const RowCDF<N>& r, int a) {
  float pa = r.P[0];
#pragma unroll
  for (int i = 1; i < N; ++i)
    if (a == i) pa = r.P[i];
  const double d = r.C[N - 1] - 1.0;
  const double lC = fabs(d) < 1e-6 ? d * (1.0 - d * (0.5 - d * (1.0 / 3.0))) : log(r.C[N - 1]);
  return (float)(log((double)pa) - lC);
}

// Hoisted search for step_stride == 0.
template <int N>
struct Thresholds {
  uint32_t K[N];     // draw k selects action i iff i is the first nonzero with k < K_i
  float lp[N];       // log-probability of each action
  uint32_t nzmask;
  int fallback;
  bool bad;
};

template <int N>
__device__ __forceinline__ void make_thresholds(const RowCDF<N>& r, Thresholds<N>& th) {
  th.bad = r.bad;
  th.nzmask = 0;
  th.fallback = last_nonzero(r);
  const double S = r.C[N - 1];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (r.P[i] > 0.0f) th.nzmask |= 1u << i;
    // smallest k in [0, 2^24] with !(k 2^-24 S < C_i): the monotone predicate is evaluated at
    // the estimate ceil(C_i / S 2^24) and the estimate stepped until it is the boundary --
    // the same K as a bisection on the predicate, in a few evaluations instead of 24
    auto below = [&](uint32_t k) { return (double)((float)k * (1.0f / 16777216.0f)) * S < r.C[i]; };
    uint32_t k = 0;
    if (!r.bad) {
      const double est = ceil(r.C[i] / S * 16777216.0);
      k = est <= 0.0 ? 0u : (est >= 16777216.0 ? (1u << 24) : (uint32_t)est);
      while (k < (1u << 24) && below(k)) ++k;
      while (k > 0 && !below(k - 1)) --k;
    }
    th.K[i] = k;
    th.lp[i] = (r.P[i] > 0.0f && !r.bad) ? (float)(log((double)r.P[i]) - log(S)) : 0.0f;
  }
}

// Hoisted search = #{i < N-1 : K_i <= k}.  K is nondecreasing (C is, under the same monotone
// predicate) and K_{last nonzero} = 2^24 > k (u S < S for u < 1), so the count is min{i : k < K_i};
// that i has p_i > 0 (a zero-probability action has C_i = C_{i-1}, hence K_i = K_{i-1}, and
// p_0 = 0 gives K_0 = 0), i.e. exactly R13's min{i : p_i > 0 and u S < C_i} -- the fallback is
// never needed for a valid row.  (Exhaustively checked against the direct search by
// ws_test_sample_grid.)
template <int N>
__device__ __forceinline__ int search_k(const Thresholds<N>& th, uint32_t k, float& lp) {
  int a = 0;
#pragma unroll
  for (int i = 0; i < N - 1; ++i) a += k >= th.K[i] ? 1 : 0;
  lp = th.lp[0];
#pragma unroll
  for (int i = 1; i < N; ++i) lp = a == i ? th.lp[i] : lp;
  return a;
}

// ---------------------------------------------------------------------------------------
// Continuous head: z_k of agent a at step t is Gaussian draw j = t*d + k of the GAUSS
// stream: Box-Muller on the word pair (2p, 2p+1), p = (j & 3) >> 1, u1 in (0, 1],
// u2 in [0, 1); even j -> r cos, odd j -> r sin; fp64, one rounding (R14, R3).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ float gauss_z(const Key& key, uint32_t eg, uint32_t agent, uint64_t j) {
  const U4 b = block(key, j >> 2, eg, agent, kGauss);
  const bool second = ((j & 3) >> 1) != 0;
  const uint32_t w0 = second ? b.z : b.x, w1 = second ? b.w : b.y;
  const double u1 = (double)((w0 >> 8) + 1) * (1.0 / 16777216.0);
  const double u2 = (double)(w1 >> 8) * (1.0 / 16777216.0);
  const double r = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.14159265358979323846 * u2;
  double sr, cr;
  int q;
  sincos64_core(ang, sr, cr, q);  // ang in [0, 2 pi): no wide-argument check needed
  const bool odd = (j & 1) != 0;  // r sin(ang) : r cos(ang)
  const double v = (((q & 1) != 0) == odd) ? cr : sr;  // odd quadrants swap sin and cos
  const int sign = (odd ? (q & 2) : ((q + 1) & 2)) << 30;
  return __int_as_float(__float_as_int((float)(r * v)) ^ sign);  // r (-x) = -(r x), rounding symmetric
}

// Both normals of the Box-Muller pair p of block b (draws 4 (b) + 2p and 4 (b) + 2p + 1).
__device__ __forceinline__ void gauss_pair(const U4& b, int p, float& z_even, float& z_odd) {
  const uint32_t w0 = p ? b.z : b.x, w1 = p ? b.w : b.y;
  const double u1 = (double)((w0 >> 8) + 1) * (1.0 / 16777216.0);
  const double u2 = (double)(w1 >> 8) * (1.0 / 16777216.0);
  const double r = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.14159265358979323846 * u2;
  double sr, cr;
  int q;
  sincos64_core(ang, sr, cr, q);  // ang in [0, 2 pi): no wide-argument check needed
  // the quadrant's swap before the products, its signs on the rounded fp32 bits (r (-x) = -(r x)
  // exactly and rounding to nearest is symmetric: the values of (float)(r cos), (float)(r sin))
  const double s0 = (q & 1) ? cr : sr, c0 = (q & 1) ? sr : cr;
  z_even = __int_as_float(__float_as_int((float)(r * c0)) ^ (((q + 1) & 2) << 30));
  z_odd = __int_as_float(__float_as_int((float)(r * s0)) ^ ((q & 2) << 30));
}

// R14 log-density constant 0.5 * log(fl64(2 pi)) (= 0.5 * log(6.283185307179586)).
constexpr double kHalfLog2Pi = 0.9189385332046727;

}  // namespace ws
