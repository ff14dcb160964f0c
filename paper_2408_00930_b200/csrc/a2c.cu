// a2c.cu -- NEXT-N2: on-device actor-critic (A2C) update over the time-major roll-out
// store, on sm_100a (include/ws.h "NEXT-N2: A2C update"; SPEC a2c_update S:402-406; P:41
// "supports actor-critic algorithms"; DESIGN reading R31).
//
// Network (R29 policy + value head on the shared hidden layer):
//   h = relu(W1^T o + b1), logits = W2^T h + b2, pi = softmax(logits), V = wv^T h + bv
// Loss: -mean(log pi(a|o) A_hat) + c_v mean((V - R)^2) - c_e mean(Ent), with
//   dL/dlogit_j = (A_hat/B)(pi_j - [j = a]) + (c_e/B) pi_j (log pi_j + Ent)
//   dL/dV = 2 c_v (V - R) / B,  dL/dz_k = [z_k > 0] (sum_j W2[k][j] dL/dlogit_j + wv_k dL/dV)
//
// Kernels (all on the FMA pipe: the contractions here are [B x D] x [D x H] with D <= 6 and
// [B x H] x [H x n] with n <= 5 -- K or N far below a tensor-core tile -- and the weight
// gradients are reductions over B = T*E rows):
//  - k_ac_values<D,H>: thread per row, weights broadcast from shared memory, H*(D+1) FMA.
//  - k_moments / k_moments_final: fp64 sum and sum of squares, fixed grid -> deterministic.
//  - k_a2c_grad<D,H,N>: persistent CTAs of 128 threads walk 128-row tiles.  Phase A: thread
//    per row -- forward (h kept in shared memory, row stride H+1: conflict-free both ways),
//    softmax / entropy / value, dL/dlogit and dL/dV, then dL/dz.  Phase B: the weight
//    gradients are contractions over the tile's rows; warp w takes rows w, w+4, ..., lane l
//    owns hidden units l (+32): per row it reads h and dz (2 x H/32 conflict-free loads) and
//    the row's o / dlogit / dV (broadcast float4 loads) and accumulates D+1+N+1 FMA chains
//    per unit in registers across all tiles.  The CTA reduces its 4 warps in a fixed order
//    and writes one fp64 partial row; k_grad_final sums the rows in fixed order.
//  - k_adam: one CTA: fp64 norm (fixed tree), clip, bias-corrected Adam in fp64, fp32 store.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "../../include/ws.h"

namespace {

constexpr int kTile = 128;       // rows per tile == threads per CTA of k_a2c_grad
constexpr int kWarps = kTile / 32;
constexpr int kMaxGrid = 1184;   // 148 SMs x 8: bound of the partial-row workspace
constexpr int kMomBlocks = 296;  // fixed grid of k_moments (order depends only on n)

struct Layout {
  int D, H, N, oW1, ob1, oW2, ob2, owv, obv, P;
  int ols;  // Gaussian (R35): log_std [N] after b2; == ob2 + N for the discrete layout too (empty)
};

// G = 1: Gaussian head (R35) -- N mean outputs, then log_std [N] before the value head
__host__ __device__ inline Layout layout(int D, int H, int N, int G = 0) {
  Layout L;
  L.D = D; L.H = H; L.N = N;
  L.oW1 = 0;
  L.ob1 = D * H;
  L.oW2 = L.ob1 + H;
  L.ob2 = L.oW2 + H * N;
  L.ols = L.ob2 + N;
  L.owv = L.ols + G * N;
  L.obv = L.owv + H;
  L.P = L.obv + 1;
  return L;
}

bool supported(int D, int H, int N, int G = 0) {
  if (G) return D == 3 && (H == 32 || H == 64) && N == 1;  // Pendulum (R34 / R35)
  return (D == 4 || D == 6) && (H == 32 || H == 64) && (N == 2 || N == 3 || N == 5);
}

// Per-hidden-unit weight record in shared memory: W1[0..D-1][k], b1[k], wv[k], W2[k][0..N-1],
// padded to 16 B, so the thread-per-row loops fetch a unit's weights with 2-3 broadcast
// LDS.128 instead of D+N+2 scalar loads.
template <int D, int N>
struct Rec {
  static constexpr int kB1 = D, kWv = D + 1, kW2 = D + 2;
  static constexpr int kLen = (D + 2 + N + 3) & ~3;
};

template <int D, int H, int N, int G = 0>
__device__ __forceinline__ void load_records(float* wrec, const float* params) {
  using RC = Rec<D, N>;
  const Layout L = layout(D, H, N, G);
  for (int i = threadIdx.x; i < H * RC::kLen; i += blockDim.x) {
    const int k = i / RC::kLen, f = i % RC::kLen;
    float x = 0.0f;
    if (f < D) x = __ldg(params + L.oW1 + f * H + k);
    else if (f == RC::kB1) x = __ldg(params + L.ob1 + k);
    else if (f == RC::kWv) x = __ldg(params + L.owv + k);
    else if (f < RC::kW2 + N) x = __ldg(params + L.oW2 + k * N + (f - RC::kW2));
    wrec[i] = x;
  }
}

// The gradient kernel's records, interleaved by unit pairs (round 2): field f of unit k at
// [(k / 2) * 2 kLen + 2 f + (k & 1)], so one LDS.128 yields two fields of both units of a pair
// -- the operands of the packed (FFMA2) forward pass.
template <int D, int N>
__device__ __forceinline__ int rec_pair_index(int k, int f) {
  return (k >> 1) * (2 * Rec<D, N>::kLen) + 2 * f + (k & 1);
}
template <int D, int H, int N, int G = 0>
__device__ __forceinline__ void load_records_paired(float* wrec, const float* params) {
  using RC = Rec<D, N>;
  const Layout L = layout(D, H, N, G);
  for (int i = threadIdx.x; i < H * RC::kLen; i += blockDim.x) {
    const int rem = i % (2 * RC::kLen);
    const int k = 2 * (i / (2 * RC::kLen)) + (rem & 1), f = rem >> 1;
    float x = 0.0f;
    if (f < D) x = __ldg(params + L.oW1 + f * H + k);
    else if (f == RC::kB1) x = __ldg(params + L.ob1 + k);
    else if (f == RC::kWv) x = __ldg(params + L.owv + k);
    else if (f < RC::kW2 + N) x = __ldg(params + L.oW2 + k * N + (f - RC::kW2));
    wrec[i] = x;
  }
}

// ------------------------------------------------------------------------------ values
template <int D, int H, int N>
__global__ void __launch_bounds__(256) k_ac_values(const float* __restrict__ params, const float* __restrict__ obs,
                                                   int64_t rows, float* __restrict__ values) {
  using RC = Rec<D, N>;
  constexpr int kLoad = (D + 2 + 3) / 4;  // float4s holding W1[.][k], b1[k], wv[k]
  extern __shared__ __align__(16) float wrec[];
  load_records<D, H, N>(wrec, params);
  const float bv = __ldg(params + layout(D, H, N).obv);
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    float o[D];
#pragma unroll
    for (int d = 0; d < D; ++d) o[d] = __ldg(obs + r * D + d);
    float v0 = bv, v1 = 0.0f;
#pragma unroll
    for (int k = 0; k < H; ++k) {
      float w[4 * kLoad];
      const float4* rk = reinterpret_cast<const float4*>(wrec + k * RC::kLen);
#pragma unroll
      for (int c = 0; c < kLoad; ++c) {
        const float4 t = rk[c];
        w[4 * c] = t.x; w[4 * c + 1] = t.y; w[4 * c + 2] = t.z; w[4 * c + 3] = t.w;
      }
      float z = w[RC::kB1];
#pragma unroll
      for (int d = 0; d < D; ++d) z = fmaf(w[d], o[d], z);
      if (k & 1) v1 = fmaf(w[RC::kWv], fmaxf(z, 0.0f), v1);
      else v0 = fmaf(w[RC::kWv], fmaxf(z, 0.0f), v0);
    }
    __stcs(values + r, v0 + v1);
  }
}

// ------------------------------------------------------------------------------ moments
__global__ void __launch_bounds__(256) k_moments(const float* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double s1[256], s2[256];
  double a = 0.0, b = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = (double)__ldg(x + i);
    a += v;
    b = fma(v, v, b);
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s1[threadIdx.x] += s1[threadIdx.x + w];
      s2[threadIdx.x] += s2[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s1[0];
    part[2 * blockIdx.x + 1] = s2[0];
  }
}

__global__ void k_moments_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[2 * b + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

// ------------------------------------------------------------------------------ gradient
struct GradDev {
  const float* params;
  const float* obs;
  const int32_t* act;
  const float* adv;
  const float* ret;
  const double* moments;
  double batch;
  float c_v, c_e;
  int64_t rows;
  double* partial;  // [gridDim.x][P + 3]
  const float* act_f;     // Gaussian (R35): actions [rows][N] f32
  const float* logp_old;  // PPO (R33): behaviour log-probs [rows]; null = A2C
  float clip_eps;
  double norm_batch;      // rows the moments were summed over (minibatches: the whole batch)
};

template <int D, int H, int N, int G = 0>
struct GradSmem {
  static constexpr int kP = D * H + H + H * N + N + G * N + H + 1;
  static constexpr int kRec = Rec<D, N>::kLen;       // per-hidden-unit weight record
  static constexpr int kOg = (D + N + 1 + 3) & ~3;   // per-row record: o, dL/dlogit, dL/dV
  static constexpr int kHrow = H + 4;                // h row stride: 16-B rows, kHrow/4 odd
  static constexpr int kW = 0;                       // [H][kRec]
  static constexpr int kB2 = H * kRec;               // b2 [N], bv
  static constexpr int kHs = kB2 + 8;                // [kTile][kHrow]
  static constexpr int kOgs = kHs + kTile * kHrow;   // [kTile][kOg]
  static constexpr int kFloats = kOgs + kTile * kOg;
  static constexpr size_t kBytes = (size_t)kFloats * sizeof(float);
  static_assert((kHrow / 4) % 2 == 1, "conflict-free 16-B row stores");
  static constexpr int kTh = N + 4 + G * N;          // per-thread scalars: b2, bv, 3 loss terms (+ log_std)
  static_assert(kTile * kHrow >= 4 * kP + kTile * kTh, "reduction scratch fits the h tile");
  static_assert(!G || N <= 3, "Gaussian head: b2 | bv | log_std fit the 8-float slot");
};

template <int D, int H, int N, int G = 0>
__global__ void __launch_bounds__(kTile, 4) k_a2c_grad(const GradDev g) {
  using S = GradSmem<D, H, N, G>;
  using RC = Rec<D, N>;
  constexpr Layout L{D, H, N, 0, D * H, D * H + H, D * H + H + H * N, D * H + H + H * N + N + G * N,
                     D * H + H + H * N + N + G * N + H, S::kP, D * H + H + H * N + N};
  constexpr int KP = H / 32;  // hidden units per lane in phase B (consecutive: k = KP*lane + q)
  extern __shared__ __align__(16) float sm[];
  float* wrec = sm + S::kW;
  float* hs = sm + S::kHs;
  float* ogs = sm + S::kOgs;
  load_records_paired<D, H, N, G>(wrec, g.params);
  if (threadIdx.x < N) sm[S::kB2 + threadIdx.x] = __ldg(g.params + L.ob2 + threadIdx.x);
  if (threadIdx.x == N) sm[S::kB2 + N] = __ldg(g.params + L.obv);
  if (G && threadIdx.x < N) sm[S::kB2 + 4 + threadIdx.x] = __ldg(g.params + L.ols + threadIdx.x);

  // normalisation (R31): mu, sigma over the global batch; skipped when sigma < 1e-8
  const double mu = g.moments[0] / g.norm_batch;
  const double var = fmax(g.moments[1] / g.norm_batch - mu * mu, 0.0);
  const double sigma = sqrt(var);
  const bool norm = sigma >= 1e-8;
  const double inv_sigma = norm ? 1.0 / sigma : 1.0;
  const float invB = (float)(1.0 / g.batch);
  const float ce_b = g.c_e * invB;
  const float cv2_b = 2.0f * g.c_v * invB;
  const float cv_b = g.c_v * invB;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float aW1[KP][D], ab1[KP], aW2[KP][N], awv[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) {
#pragma unroll
    for (int d = 0; d < D; ++d) aW1[q][d] = 0.0f;
#pragma unroll
    for (int j = 0; j < N; ++j) aW2[q][j] = 0.0f;
    ab1[q] = 0.0f;
    awv[q] = 0.0f;
  }
  float ab2[N], abv = 0.0f, lpol = 0.0f, lval = 0.0f, lent = 0.0f, als[N];
#pragma unroll
  for (int j = 0; j < N; ++j) ab2[j] = 0.0f, als[j] = 0.0f;
  __syncthreads();
  // phase-B weights of this lane's hidden units, in registers for the whole kernel
  float w2k[KP][N], wvk[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    const int k = KP * lane + q;
    wvk[q] = wrec[rec_pair_index<D, N>(k, RC::kWv)];
#pragma unroll
    for (int j = 0; j < N; ++j) w2k[q][j] = wrec[rec_pair_index<D, N>(k, RC::kW2 + j)];
  }

  const int64_t n_tiles = (g.rows + kTile - 1) / kTile;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t base = tile * kTile;
    const int nrow = (int)(g.rows - base < kTile ? g.rows - base : kTile);
    __syncthreads();  // previous tile's phase B done with hs / ogs
    const float* ob = g.obs + base * D;
    for (int i = tid; i < nrow * D; i += kTile) ogs[(i / D) * S::kOg + (i % D)] = __ldg(ob + i);
    __syncthreads();

    // ---- phase A: thread per row: forward, softmax / entropy / value, dL/dlogit, dL/dV
    const int s = tid;
    float* og = ogs + s * S::kOg;
    if (s < nrow) {
      const int64_t r = base + s;
      const int a = G ? 0 : __ldg(g.act + r);
      const float A = __ldg(g.adv + r);
      const float R = __ldg(g.ret + r);
      float o[D];
#pragma unroll
      for (int d = 0; d < D; ++d) o[d] = og[d];
      float l0[N], l1[N], v0 = sm[S::kB2 + N], v1 = 0.0f;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        l0[j] = sm[S::kB2 + j];
        l1[j] = 0.0f;
      }
      float4* hrow = reinterpret_cast<float4*>(hs + s * S::kHrow);
      // units in pairs (2m, 2m + 1) as packed fp32 pairs: the even unit accumulates into l0 / v0,
      // the odd one into l1 / v1, exactly the scalar code's chains (FFMA2 rounds each element as
      // FFMA does)
#pragma unroll 2
      for (int kc = 0; kc < H; kc += 4) {
        float h[4];
#pragma unroll
        for (int pp = 0; pp < 2; ++pp) {
          const float4* rk = reinterpret_cast<const float4*>(wrec + ((kc >> 1) + pp) * (2 * RC::kLen));
          float2 w[RC::kLen];  // field f of the pair
#pragma unroll
          for (int c = 0; c < RC::kLen / 2; ++c) {
            const float4 t = rk[c];
            w[2 * c] = make_float2(t.x, t.y);
            w[2 * c + 1] = make_float2(t.z, t.w);
          }
          float2 z = w[RC::kB1];
#pragma unroll
          for (int d = 0; d < D; ++d) z = __ffma2_rn(w[d], make_float2(o[d], o[d]), z);
          const float2 hh = make_float2(fmaxf(z.x, 0.0f), fmaxf(z.y, 0.0f));
          h[2 * pp] = hh.x;
          h[2 * pp + 1] = hh.y;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const float2 lj = __ffma2_rn(w[RC::kW2 + j], hh, make_float2(l0[j], l1[j]));
            l0[j] = lj.x;
            l1[j] = lj.y;
          }
          const float2 vv = __ffma2_rn(w[RC::kWv], hh, make_float2(v0, v1));
          v0 = vv.x;
          v1 = vv.y;
        }
        hrow[kc >> 2] = make_float4(h[0], h[1], h[2], h[3]);
      }
      float dl[N], dv = 0.0f;
#pragma unroll
      for (int j = 0; j < N; ++j) dl[j] = 0.0f;
      if constexpr (G) {
        // Gaussian head (R35): mean = the linear outputs, log pi = sum_j -(a-mu)^2/(2 s^2)
        // - log s - log(2 pi)/2; rows with a non-finite action contribute nothing
        float act[N];
        bool okr = true;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          act[j] = __ldg(g.act_f + r * N + j);
          okr = okr && isfinite(act[j]);
        }
        if (okr) {
          const float v = v0 + v1;
          float diff[N], iv[N], lpa = 0.0f, ent = 0.0f;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const float ls = sm[S::kB2 + 4 + j];
            diff[j] = act[j] - (l0[j] + l1[j]);
            iv[j] = expf(-2.0f * ls);
            lpa += -0.5f * diff[j] * diff[j] * iv[j] - ls - 0.91893853320467274f;
            ent += ls + 1.41893853320467274f;  // log(2 pi e) / 2
          }
          float Ah = norm ? (float)(((double)A - mu) * inv_sigma) : A;
          float surr = lpa * Ah;
          if (g.logp_old) {
            const float rho = expf(lpa - __ldg(g.logp_old + r));
            const float rc = fminf(fmaxf(rho, 1.0f - g.clip_eps), 1.0f + g.clip_eps);
            const float s1 = rho * Ah, s2 = rc * Ah;
            surr = fminf(s1, s2);
            Ah = s1 <= s2 ? s1 : 0.0f;
          }
          const float Ab = Ah * invB;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            dl[j] = -Ab * diff[j] * iv[j];
            als[j] += -Ab * (diff[j] * diff[j] * iv[j] - 1.0f) - ce_b;
          }
          dv = cv2_b * (v - R);
          lpol -= surr * invB;
          lval += cv_b * (v - R) * (v - R);
          lent -= ce_b * ent;
#pragma unroll
          for (int j = 0; j < N; ++j) ab2[j] += dl[j];
          abv += dv;
        }
      } else if (a >= 0 && a < N) {
        float l[N];
#pragma unroll
        for (int j = 0; j < N; ++j) l[j] = l0[j] + l1[j];
        const float v = v0 + v1;
        float m = l[0];
#pragma unroll
        for (int j = 1; j < N; ++j) m = fmaxf(m, l[j]);
        float e[N], Ssum = 0.0f;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          e[j] = expf(l[j] - m);
          Ssum += e[j];
        }
        const float lS = logf(Ssum), invS = 1.0f / Ssum;
        float lp[N], p[N], ent = 0.0f, lpa = 0.0f;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          lp[j] = (l[j] - m) - lS;
          p[j] = e[j] * invS;
          ent -= p[j] * lp[j];
          if (j == a) lpa = lp[j];
        }
        float Ah = norm ? (float)(((double)A - mu) * inv_sigma) : A;
        float surr = lpa * Ah;  // A2C: the policy term is -log pi(a) A_hat
        if (g.logp_old) {       // PPO (R33): clipped surrogate; gradient rho A_hat where unclipped wins
          const float rho = expf(lpa - __ldg(g.logp_old + r));
          const float rc = fminf(fmaxf(rho, 1.0f - g.clip_eps), 1.0f + g.clip_eps);
          const float s1 = rho * Ah, s2 = rc * Ah;
          surr = fminf(s1, s2);
          Ah = s1 <= s2 ? s1 : 0.0f;
        }
        const float Ab = Ah * invB;
#pragma unroll
        for (int j = 0; j < N; ++j) dl[j] = Ab * (p[j] - (j == a ? 1.0f : 0.0f)) + ce_b * p[j] * (lp[j] + ent);
        dv = cv2_b * (v - R);
        lpol -= surr * invB;
        lval += cv_b * (v - R) * (v - R);
        lent -= ce_b * ent;
#pragma unroll
        for (int j = 0; j < N; ++j) ab2[j] += dl[j];
        abv += dv;
      }
#pragma unroll
      for (int j = 0; j < N; ++j) og[D + j] = dl[j];
      og[D + N] = dv;
    }
    __syncthreads();

    // ---- phase B: contractions over the tile's rows.  Warp w takes rows w, w + 4, ...; lane l
    // owns hidden units KP*l .. KP*l+KP-1: dL/dz from its register weights, then D+1+N+1
    // accumulations per unit.
    for (int r = warp; r < nrow; r += kWarps) {
      float ogv[S::kOg];
      const float4* og4 = reinterpret_cast<const float4*>(ogs + r * S::kOg);
#pragma unroll
      for (int c = 0; c < S::kOg / 4; ++c) {
        const float4 t = og4[c];
        ogv[4 * c] = t.x; ogv[4 * c + 1] = t.y; ogv[4 * c + 2] = t.z; ogv[4 * c + 3] = t.w;
      }
      float hv[KP];
      if constexpr (KP == 2) {
        const float2 t = reinterpret_cast<const float2*>(hs + r * S::kHrow)[lane];
        hv[0] = t.x;
        hv[1] = t.y;
      } else {
        hv[0] = hs[r * S::kHrow + lane];
      }
      const float dv = ogv[D + N];
      if constexpr (KP == 2) {
        // the lane's two units in packed fp32 pairs (FMUL2 / FFMA2 / FADD2: each element rounded
        // exactly like the scalar FMUL / FFMA / FADD, half the instructions)
        const float2 dvv = make_float2(dv, dv);
        float2 dh = __fmul2_rn(make_float2(wvk[0], wvk[1]), dvv);
#pragma unroll
        for (int j = 0; j < N; ++j)
          dh = __ffma2_rn(make_float2(w2k[0][j], w2k[1][j]), make_float2(ogv[D + j], ogv[D + j]), dh);
        const float2 dz = make_float2(hv[0] > 0.0f ? dh.x : 0.0f, hv[1] > 0.0f ? dh.y : 0.0f);
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const float2 t = __ffma2_rn(make_float2(ogv[d], ogv[d]), dz, make_float2(aW1[0][d], aW1[1][d]));
          aW1[0][d] = t.x;
          aW1[1][d] = t.y;
        }
        const float2 b = __fadd2_rn(make_float2(ab1[0], ab1[1]), dz);
        ab1[0] = b.x;
        ab1[1] = b.y;
        const float2 hh = make_float2(hv[0], hv[1]);
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const float2 t = __ffma2_rn(hh, make_float2(ogv[D + j], ogv[D + j]), make_float2(aW2[0][j], aW2[1][j]));
          aW2[0][j] = t.x;
          aW2[1][j] = t.y;
        }
        const float2 v = __ffma2_rn(hh, dvv, make_float2(awv[0], awv[1]));
        awv[0] = v.x;
        awv[1] = v.y;
      } else {
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          float dh = wvk[q] * dv;
#pragma unroll
          for (int j = 0; j < N; ++j) dh = fmaf(w2k[q][j], ogv[D + j], dh);
          const float dz = hv[q] > 0.0f ? dh : 0.0f;
#pragma unroll
          for (int d = 0; d < D; ++d) aW1[q][d] = fmaf(ogv[d], dz, aW1[q][d]);
          ab1[q] += dz;
#pragma unroll
          for (int j = 0; j < N; ++j) aW2[q][j] = fmaf(hv[q], ogv[D + j], aW2[q][j]);
          awv[q] = fmaf(hv[q], dv, awv[q]);
        }
      }
    }
  }
  __syncthreads();

  // ---- CTA reduction in a fixed order: per-warp unit partials, per-thread bias / loss terms
  double* out = g.partial + (size_t)blockIdx.x * (S::kP + 3);
  float* red = hs;                  // [kWarps][P]
  float* th = hs + kWarps * S::kP;  // [kTile][kTh]
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    const int k = KP * lane + q;
    float* rw = red + warp * S::kP;
#pragma unroll
    for (int d = 0; d < D; ++d) rw[L.oW1 + d * H + k] = aW1[q][d];
    rw[L.ob1 + k] = ab1[q];
#pragma unroll
    for (int j = 0; j < N; ++j) rw[L.oW2 + k * N + j] = aW2[q][j];
    rw[L.owv + k] = awv[q];
  }
  {
    float* t = th + tid * S::kTh;
#pragma unroll
    for (int j = 0; j < N; ++j) t[j] = ab2[j];
    t[N] = abv;
    t[N + 1] = lpol;
    t[N + 2] = lval;
    t[N + 3] = lent;
    if (G) {
#pragma unroll
      for (int j = 0; j < N; ++j) t[N + 4 + j] = als[j];
    }
  }
  __syncthreads();
  for (int i = tid; i < S::kP; i += kTile) {
    if ((i >= L.ob2 && i < L.ob2 + N + G * N) || i == L.obv) continue;
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) acc += (double)red[w * S::kP + i];
    out[i] = acc;
  }
  if (tid < S::kTh) {
    double acc = 0.0;
    for (int t = 0; t < kTile; ++t) acc += (double)th[t * S::kTh + tid];
    const int dst = tid < N ? L.ob2 + tid
                  : tid == N ? L.obv
                  : tid < N + 4 ? S::kP + (tid - N - 1)
                  : L.ols + (tid - N - 4);
    out[dst] = acc;
  }
}

__global__ void __launch_bounds__(128) k_grad_final(const double* __restrict__ part, int nb, int P,
                                                    float* __restrict__ grad, double* __restrict__ loss) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P + 3) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(size_t)b * (P + 3) + c];
  if (c < P) grad[c] = (float)s;
  else if (loss) loss[c - P] = s;
}

// ------------------------------------------------------------------------------ Adam
__global__ void __launch_bounds__(1024) k_adam(float* __restrict__ params, const float* __restrict__ grad,
                                               float* __restrict__ m, float* __restrict__ v, int n, int step,
                                               double lr, double b1, double b2, double eps, double max_norm,
                                               float* __restrict__ grad_norm) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = (double)grad[i];
    s = fma(x, x, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double norm = sqrt(red[0]);
  if (threadIdx.x == 0 && grad_norm) *grad_norm = (float)norm;
  const double scale = (max_norm > 0.0 && norm > max_norm) ? max_norm / norm : 1.0;
  const double c1 = 1.0 - pow(b1, (double)step), c2 = 1.0 - pow(b2, (double)step);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double gi = (double)grad[i] * scale;
    const double mi = b1 * (double)m[i] + (1.0 - b1) * gi;
    const double vi = b2 * (double)v[i] + (1.0 - b2) * gi * gi;
    const double upd = lr * (mi / c1) / (sqrt(vi / c2) + eps);
    params[i] = (float)((double)params[i] - upd);
    m[i] = (float)mi;
    v[i] = (float)vi;
  }
}

// ------------------------------------------------------------------------------ dispatch
template <int D, int H, int N, int G = 0>
cudaError_t launch_grad_t(const GradDev& g, cudaStream_t s, int* nb_out) {
  using S = GradSmem<D, H, N, G>;
  static int grid_cap = 0;  // CTAs per device at full residency (same for every B200)
  cudaError_t e = cudaSuccess;
  if (!grid_cap) {
    e = cudaFuncSetAttribute(k_a2c_grad<D, H, N, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::kBytes);
    if (e) return e;
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev))) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_a2c_grad<D, H, N, G>, kTile, S::kBytes))) return e;
    grid_cap = std::max(1, std::min(kMaxGrid, sms * std::max(per_sm, 1)));
  }
  const int64_t tiles = (g.rows + kTile - 1) / kTile;
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, grid_cap));
  k_a2c_grad<D, H, N, G><<<nb, kTile, S::kBytes, s>>>(g);
  *nb_out = nb;
  return cudaGetLastError();
}

template <int D, int H>
cudaError_t launch_grad_dh(int N, const GradDev& g, cudaStream_t s, int* nb) {
  switch (N) {
    case 2: return launch_grad_t<D, H, 2>(g, s, nb);
    case 3: return launch_grad_t<D, H, 3>(g, s, nb);
    default: return launch_grad_t<D, H, 5>(g, s, nb);
  }
}

cudaError_t launch_grad(int D, int H, int N, const GradDev& g, cudaStream_t s, int* nb, int G = 0) {
  if (G) return H == 32 ? launch_grad_t<3, 32, 1, 1>(g, s, nb) : launch_grad_t<3, 64, 1, 1>(g, s, nb);
  if (D == 4) return H == 32 ? launch_grad_dh<4, 32>(N, g, s, nb) : launch_grad_dh<4, 64>(N, g, s, nb);
  return H == 32 ? launch_grad_dh<6, 32>(N, g, s, nb) : launch_grad_dh<6, 64>(N, g, s, nb);
}

template <int D, int H, int N>
cudaError_t launch_values_t(const float* params, const float* obs, int64_t rows, float* values, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((rows + 255) / 256, 148 * 8);
  k_ac_values<D, H, N><<<(int)blocks, 256, H * Rec<D, N>::kLen * sizeof(float), s>>>(params, obs, rows, values);
  return cudaGetLastError();
}

template <int D, int H>
cudaError_t launch_values_dh(int N, const float* params, const float* obs, int64_t rows, float* values,
                             cudaStream_t s) {
  switch (N) {
    case 2: return launch_values_t<D, H, 2>(params, obs, rows, values, s);
    case 3: return launch_values_t<D, H, 3>(params, obs, rows, values, s);
    default: return launch_values_t<D, H, 5>(params, obs, rows, values, s);
  }
}

}  // namespace

extern "C" {

int32_t ws_a2c_n_params(int32_t D, int32_t H, int32_t N) {
  if (D < 1 || H < 1 || N < 1) return 0;
  return layout(D, H, N).P;
}

int32_t ws_a2c_n_params_ex(int32_t D, int32_t H, int32_t N, int32_t gaussian) {
  if (D < 1 || H < 1 || N < 1) return 0;
  return layout(D, H, N, gaussian ? 1 : 0).P;
}

size_t ws_a2c_workspace_bytes(int32_t D, int32_t H, int32_t N) {
  if (!supported(D, H, N) && !supported(D, H, N, 1)) return 0;
  const size_t g = (size_t)kMaxGrid * (layout(D, H, N, 1).P + 3) * sizeof(double);
  const size_t m = (size_t)kMomBlocks * 2 * sizeof(double);
  return std::max(g, m);
}

ws_status ws_ac_values(const float* params, int32_t D, int32_t H, int32_t N, const float* obs, int64_t rows,
                       float* values, void* stream) {
  if (!supported(D, H, N) || !params || rows < 0 || (rows > 0 && (!obs || !values))) return WS_ERR_INVALID_ARGUMENT;
  if (rows == 0) return WS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (D == 4) e = H == 32 ? launch_values_dh<4, 32>(N, params, obs, rows, values, s)
                          : launch_values_dh<4, 64>(N, params, obs, rows, values, s);
  else e = H == 32 ? launch_values_dh<6, 32>(N, params, obs, rows, values, s)
                   : launch_values_dh<6, 64>(N, params, obs, rows, values, s);
  return e ? WS_ERR_CUDA : WS_OK;
}

ws_status ws_a2c_moments(const float* x, int64_t n, double* out, void* workspace, void* stream) {
  if (!x || n < 1 || !out || !workspace) return WS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(workspace);
  k_moments<<<kMomBlocks, 256, 0, s>>>(x, n, part);
  k_moments_final<<<1, 32, 0, s>>>(part, kMomBlocks, out);
  return cudaGetLastError() ? WS_ERR_CUDA : WS_OK;
}

ws_status ws_a2c_grad(const ws_a2c_args* a, void* stream) {
  if (!a || !supported(a->obs_dim, a->hidden, a->n_actions, a->gaussian ? 1 : 0) || a->rows < 1 || !a->params ||
      !a->obs || !(a->gaussian ? a->act_f != nullptr : a->act != nullptr) || !a->adv || !a->ret || !a->moments ||
      !(a->batch > 0.0) || !a->workspace || !a->grad)
    return WS_ERR_INVALID_ARGUMENT;
  if (a->logp_old && !(a->clip_eps >= 0.0f && a->clip_eps < 1.0f)) return WS_ERR_INVALID_ARGUMENT;
  GradDev g{a->params, a->obs, a->act, a->adv, a->ret, a->moments, a->batch, a->c_v, a->c_e, a->rows,
            static_cast<double*>(a->workspace), a->act_f, a->logp_old, a->clip_eps,
            a->norm_batch > 0.0 ? a->norm_batch : a->batch};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int nb = 0;
  cudaError_t e = launch_grad(a->obs_dim, a->hidden, a->n_actions, g, s, &nb, a->gaussian ? 1 : 0);
  if (e) return WS_ERR_CUDA;
  const int P = layout(a->obs_dim, a->hidden, a->n_actions, a->gaussian ? 1 : 0).P;
  k_grad_final<<<(P + 3 + 127) / 128, 128, 0, s>>>(g.partial, nb, P, a->grad, a->loss);
  return cudaGetLastError() ? WS_ERR_CUDA : WS_OK;
}

__global__ void k_clamp(float* __restrict__ x, int n, float lo, float hi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = fminf(fmaxf(x[i], lo), hi);
}

ws_status ws_clamp(float* x, int32_t n, float lo, float hi, void* stream) {
  if (!x || n < 0 || !(lo <= hi)) return WS_ERR_INVALID_ARGUMENT;
  if (n == 0) return WS_OK;
  k_clamp<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(x, n, lo, hi);
  return cudaGetLastError() ? WS_ERR_CUDA : WS_OK;
}

ws_status ws_adam(float* params, const float* grad, float* m, float* v, int32_t n, int32_t step, float lr,
                  float beta1, float beta2, float eps, float max_norm, float* grad_norm, void* stream) {
  if (!params || !grad || !m || !v || n < 1 || n > 65536 || step < 1 || !(lr >= 0.0f) || !(beta1 >= 0.0f && beta1 < 1.0f) ||
      !(beta2 >= 0.0f && beta2 < 1.0f) || !(eps >= 0.0f))
    return WS_ERR_INVALID_ARGUMENT;
  k_adam<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(params, grad, m, v, n, step, lr, beta1, beta2, eps,
                                                             max_norm, grad_norm);
  return cudaGetLastError() ? WS_ERR_CUDA : WS_OK;
}

}  // extern "C"
