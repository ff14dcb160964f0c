// common.cuh -- device primitives of libws (sm_100a): Philox4x32-10, the draw layout,
// uniform / Gaussian conversions, the transcendental contract, warp helpers, stores.
//
// Product code.  Shares nothing with oracle/ (DESIGN.md section 2).
// Citation keys: P:n PAPER.md, S:n SPEC.md, BJ:5 north_star, Rk = DESIGN.md reading k.
#pragma once

#ifdef __CUDACC_RTC__  // also compiled into the env composer's NVRTC programs (composer.cu)
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
#else
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace ws {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------------------
// A1. Philox4x32-10 (S:120-124 RngStream; BJ:5 "driven by a counter-based Philox RNG").
// Ten rounds of the Salmon et al. (SC'11) bijection; mul-hi via __umulhi, mul-lo via the
// 32-bit product.  Fully unrolled: ~70 integer instructions, no memory.
// ---------------------------------------------------------------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                     uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return U4{c0, c1, c2, c3};
}

// Philox4x32-10 with the key schedule precomputed (ks[r] = key + r (0x9E3779B9, 0xBB67AE85)):
// loops that draw many blocks under one key keep the 20 round keys in registers
struct KeySchedule {
  uint32_t k0[10], k1[10];
};
__device__ __forceinline__ KeySchedule key_schedule(uint32_t k0, uint32_t k1) {
  KeySchedule ks;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    ks.k0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
    ks.k1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
  }
  return ks;
}
__device__ __forceinline__ U4 philox_ks(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const KeySchedule& ks) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ ks.k0[r];
    const uint32_t n2 = hi0 ^ c3 ^ ks.k1[r];
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return U4{c0, c1, c2, c3};
}

__device__ __forceinline__ uint32_t pick(const U4& v, uint32_t i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// R15 stream layout: draw j of stream (env_global, agent, purpose) is word j & 3 of
// Philox(ctr = (j >> 2, env_global, agent, purpose), key = (seed_lo, seed_hi)).
enum Purpose : uint32_t { kAction = 1, kReset = 2, kGauss = 3 };

struct Key {
  uint32_t k0, k1;
};

__device__ __forceinline__ U4 block(const Key& key, uint64_t blk, uint32_t eg, uint32_t agent,
                                    uint32_t purpose) {
  return philox((uint32_t)blk, eg, agent, purpose, key.k0, key.k1);
}

// R14: u = (w >> 8) 2^-24 in [0, 1), exact in fp32.
__device__ __forceinline__ float u01(uint32_t w) { return (float)(w >> 8) * (1.0f / 16777216.0f); }

// ---------------------------------------------------------------------------------------
// R3 transcendental contract: evaluate in fp64 and round once to fp32 -- the same value
// (up to a 2^-28-rare double-rounding coincidence) as (float)libm((double)x) on the host.
//
// sincos64: branch-free fp64 sin and cos for |x| < 2^20 -- Cody-Waite reduction by pi/2 in
// three FMAs (x - k p1 exact, k p2 exact; the split's residual, 1e-37 k, is < 2e-25 relative to the
// smallest |r| an fp32 argument below 2^20 produces: 4.19e-9 at x = 252.8982, k = 161), quadrant from the
// 2^52+2^51 rounding trick, near-minimax polynomials of degree 13 / 14 on |r| <= pi/4 in Estrin
// form (Chebyshev interpolation in z = r^2, coefficients from tools/fit_sincos.py; max relative
// error of the rounded-coefficient polynomials 2.0e-17 / 5.8e-19, i.e. below 0.2 ulp, against
// 6.4e-18 / 1.3e-18 for the Taylor series through r^17 / r^18 they replace at four fewer DFMAs).
// Larger |x| (never reached by the dynamics) use libdevice.
// Pinned against the host libm by tests/test_gpu_kernels.py.
// ---------------------------------------------------------------------------------------
// fp64 constants in constant memory: DFMA / DMUL read them through the constant cache
// instead of re-materialising each 64-bit immediate with two UMOVs per use
__constant__ double kTrig[19] = {
    6.36619772367581382433e-01,  // 0  2/pi
    1.57079632673412561417e+00,  // 1  p1 (fdlibm pio2_1, 33 bits)   pi/2 = p1 + p2 + p2t
    6.07710050630396597660e-11,  // 2  p2 (pio2_2, 33 bits)
    2.02226624879595063154e-21,  // 3  p2t (pio2_2t, the rounded rest; residual 1.0e-37)
    6755399441055744.0,          // 4  2^52 + 2^51
    // sin r = r + r^3 P(r^2): P coefficients of z^0 .. z^5
    -0x1.5555555555555p-3, 0x1.1111111110bb2p-7, -0x1.a01a019e83aaep-13, 0x1.71de37968a100p-19,
    -0x1.ae600b02b6262p-26, 0x1.5e0b19f8b1451p-33,
    // cos r = 1 + r^2 Q(r^2): Q coefficients of z^0 .. z^6
    -0x1.0000000000000p-1, 0x1.5555555555551p-5, -0x1.6c16c16c15d79p-10, 0x1.a01a019de131fp-16,
    -0x1.27e4f8e4a2e74p-22, 0x1.1eea7f259b344p-29, -0x1.8ff9d439a204ap-37,
    0.0};  // 18: padding -- keeps the constant-bank offsets of the tables after it (measured)

// sincos64_core: the reduced-argument polynomials sr = sin r, cr = cos r and the quadrant q of x
// (valid for |x| < 2^20); sincos64 / sincos_c assemble the result from them.
__device__ __forceinline__ void sincos64_core(double x, double& sr, double& cr, int& q) {
  const double kd = fma(x, kTrig[0], kTrig[4]);
  const double k = kd - kTrig[4];
  q = __double2loint(kd);
  double r = fma(-k, kTrig[1], x);
  r = fma(-k, kTrig[2], r);
  r = fma(-k, kTrig[3], r);
  const double z = r * r, z2 = z * z, z4 = z2 * z2;
  // sin r = r + r^3 P(z), cos r = 1 + z Q(z), Estrin
  const double s_a = fma(z, kTrig[6], kTrig[5]);
  const double s_b = fma(z, kTrig[8], kTrig[7]);
  const double s_c = fma(z, kTrig[10], kTrig[9]);
  const double ps = fma(z4, s_c, fma(z2, s_b, s_a));
  const double c_a = fma(z, kTrig[12], kTrig[11]);
  const double c_b = fma(z, kTrig[14], kTrig[13]);
  const double c_c = fma(z, kTrig[16], kTrig[15]);
  const double pc = fma(z4, fma(z2, kTrig[17], c_c), fma(z2, c_b, c_a));
  sr = fma(r * z, ps, r);
  cr = fma(z, pc, 1.0);
}

// kChecked: |x| >= 2^20 (never reached by the environments' dynamics) falls back to
// libdevice; callers whose arguments are provably bounded pass false.
template <bool kChecked = true>
__device__ __forceinline__ void sincos64(double x, double& s, double& c) {
  double sr, cr;
  int q;
  sincos64_core(x, sr, cr, q);
  const double s0 = (q & 1) ? cr : sr;
  const double c0 = (q & 1) ? sr : cr;
  s = (q & 2) ? -s0 : s0;
  c = ((q + 1) & 2) ? -c0 : c0;
  if (kChecked && !(fabs(x) < 1048576.0)) sincos(x, &s, &c);
}

#ifdef __CUDACC_RTC__
// sincos_small (NVRTC programs of the env composer only): the R3 sin / cos of an fp32 angle with
// |x| <= 0.25 without range reduction -- the Taylor series through x^13 / x^14 (truncation < 3e-21)
// in Estrin form, rounded once (the built-in CartPole's sincos_poly uses near-minimax polynomials
// of degree 11 / 10 with the same accuracy; here they measured 3 % slower on C2U, so the composer
// keeps the series).  Pinned against the host libm on
// 40 M angles through CartPole (tests/test_gpu_kernels.py) and through the composer's
// bit-exact CartPole tests (tests/test_gpu_user_env.py).
__constant__ double kSinSmall[6] = {1.0 / 6227020800.0, -1.0 / 39916800.0, 1.0 / 362880.0, -1.0 / 5040.0,
                                    1.0 / 120.0, -1.0 / 6.0};
__constant__ double kCosSmall[8] = {-1.0 / 87178291200.0, 1.0 / 479001600.0, -1.0 / 3628800.0, 1.0 / 40320.0,
                                    -1.0 / 720.0, 1.0 / 24.0, -0.5, 1.0};
__device__ __forceinline__ void sincos_small(float th, float& s, float& c) {
  const double x = (double)th, z = x * x, z2 = z * z;
  const double ps_hi = fma(z, kSinSmall[0], kSinSmall[1]);   // c13 z + c11
  const double ps_mid = fma(z, kSinSmall[2], kSinSmall[3]);  // c9 z + c7
  const double ps_lo = fma(z, kSinSmall[4], kSinSmall[5]);   // c5 z + c3
  const double ps = fma(z2, fma(z2, ps_hi, ps_mid), ps_lo);
  const double c_l = fma(z, kCosSmall[6], kCosSmall[7]);     // c2 z + 1
  const double c_a = fma(z, kCosSmall[4], kCosSmall[5]);     // c6 z + c4
  const double c_b = fma(z, kCosSmall[2], kCosSmall[3]);     // c10 z + c8
  const double c_c = fma(z, kCosSmall[0], kCosSmall[1]);     // c14 z + c12
  const double z4 = z2 * z2;
  const double cA = fma(z2, c_a, c_l), cB = fma(z2, c_c, c_b);
  s = (float)fma(x * z, ps, x);
  c = (float)fma(z4, cB, cA);
}
#endif

// both rounded to fp32 first, then the quadrant's swap (one FSEL each) and sign (one LOP3 on the
// fp32 bit pattern each): rounding to nearest commutes with both, so the results are those of
// (float) of sincos64's, with half the select work of the fp64 assembly
template <bool kChecked = true>
__device__ __forceinline__ void sincos_c(float x, float& s, float& c) {
  double sr, cr;
  int q;
  sincos64_core((double)x, sr, cr, q);
  const float sf = (float)sr, cf = (float)cr;
  const float s0 = (q & 1) ? cf : sf;
  const float c0 = (q & 1) ? sf : cf;
  s = __int_as_float(__float_as_int(s0) ^ ((q & 2) << 30));
  c = __int_as_float(__float_as_int(c0) ^ (((q + 1) & 2) << 30));
  if (kChecked && !(fabsf(x) < 1048576.0f)) {
    double sd, cd;
    sincos((double)x, &sd, &cd);
    s = (float)sd;
    c = (float)cd;
  }
}
template <bool kChecked = true>
__device__ __forceinline__ float sin_c(float x) {
  double sd, cd;
  sincos64<kChecked>((double)x, sd, cd);
  return (float)sd;
}
template <bool kChecked = true>
__device__ __forceinline__ float cos_c(float x) {
  double sd, cd;
  sincos64<kChecked>((double)x, sd, cd);
  return (float)cd;
}

// exp64: branch-free fp64 e^x (no slow-path branch, so independent evaluations interleave;
// libdevice's exp(double) has one).  x is clamped to [-746, 710] (e^x is 0 / inf beyond in
// fp64; NaN propagates); k = round(x log2 e) by the 2^52 + 2^51 trick, r = x - k ln2 with the
// fdlibm two-part ln2 (k ln2_hi exact), e^r = 1 + r (1 + r (1/2 + r T(r))) with T the Taylor
// tail 1/3! .. r^10/13! (truncation < 2^-57 relative on |r| <= ln2 / 2) in Estrin form and the
// last three steps in Horner form (final rounding error ~0.5-0.8 ulp), then 2^k applied as two
// exact power-of-two factors (one rounding, gradual underflow).  The R3 contract rounds what
// is built from it to fp32 once; pinned against the host libm through the surface-energy and
// surface roll-out parity tests (tests/test_gpu_kernels.py, tests/test_gpu_parity.py).  (In the
// policy kernels' softmax it measured 5 % slower than libdevice's exp, so they keep the latter.)
__constant__ double kExp[15] = {
    1.44269504088896338700e+00,  // 0  log2 e
    6.93147180369123816490e-01,  // 1  ln2 hi (fdlibm)
    1.90821492927058770002e-10,  // 2  ln2 lo
    6755399441055744.0,          // 3  2^52 + 2^51
    1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0, 1.0 / 720.0, 1.0 / 5040.0, 1.0 / 40320.0, 1.0 / 362880.0,
    1.0 / 3628800.0, 1.0 / 39916800.0, 1.0 / 479001600.0, 1.0 / 6227020800.0};  // 4..14: 1/3! .. 1/13!

__device__ __forceinline__ double exp64(const double x0) {
  const double x = fmin(fmax(x0, -746.0), 710.0);
  const double kd = fma(x, kExp[0], kExp[3]);
  const double k = kd - kExp[3];
  const int ki = __double2loint(kd);
  double r = fma(-k, kExp[1], x);
  r = fma(-k, kExp[2], r);
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  const double t01 = fma(r, kExp[5], kExp[4]), t23 = fma(r, kExp[7], kExp[6]);
  const double t45 = fma(r, kExp[9], kExp[8]), t67 = fma(r, kExp[11], kExp[10]);
  const double t89 = fma(r, kExp[13], kExp[12]);
  const double u0 = fma(r2, t23, t01), u1 = fma(r2, t67, t45), u2 = fma(r2, kExp[14], t89);
  const double T = fma(r8, u2, fma(r4, u1, u0));
  const double p = fma(r, fma(r, fma(r, T, 0.5), 1.0), 1.0);
  const int k1 = ki >> 1, k2 = ki - k1;  // 2^k = 2^k1 2^k2, each a normal double
  const double y = (p * __hiloint2double((k1 + 1023) << 20, 0)) * __hiloint2double((k2 + 1023) << 20, 0);
  return x0 == x0 ? y : x0;
}

// IEEE fp32 arithmetic without contraction: the library is built with --fmad=false, and
// these make the intended rounding explicit where it matters.
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }

// ---------------------------------------------------------------------------------------
// Streaming (evict-first) stores for the roll-out store: written once, read by the trainer
// later, larger than L2 at the headline shapes (BJ:5 "coalesced, vectorised stores").
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void st_cs(float* p, float v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(int32_t* p, int32_t v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(float2* p, float2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs_u8(uint8_t* p, uint8_t v) {
  asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
}

// Device error word bits (sticky until ws_reset, R19).
constexpr uint32_t kErrAction = 1u, kErrProbs = 2u, kErrPeer = 4u;

__device__ __forceinline__ float warp_sum_f32(float v) {
  // xor butterfly; lane 0's value is the deterministic result used by the caller
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fadd(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// Exact warp sum of 64-bit integers (mod 2^64, i.e. exact for two's-complement values whose
// sum fits): each value is split into four 16-bit chunks, each chunk column is summed with
// one REDUX (32 x (2^16 - 1) < 2^32, no overflow) and the four sums are recombined.
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
  const unsigned c0 = __reduce_add_sync(kFull, (unsigned)(v & 0xFFFFu));
  const unsigned c1 = __reduce_add_sync(kFull, (unsigned)((v >> 16) & 0xFFFFu));
  const unsigned c2 = __reduce_add_sync(kFull, (unsigned)((v >> 32) & 0xFFFFu));
  const unsigned c3 = __reduce_add_sync(kFull, (unsigned)(v >> 48));
  return (unsigned long long)c0 + ((unsigned long long)c1 << 16) + ((unsigned long long)c2 << 32) +
         ((unsigned long long)c3 << 48);
}

// A8 statistics are exact fixed-point integers: stats[slot] = {episodes, sum of returns
// x 2^32, sum of lengths, sum of rewards x 2^32} as int64.  Every per-replica value is
// converted once (an fp32 reward r is represented exactly whenever |r| >= 2^-8 and
// |r| < 2^31; smaller values are rounded to a multiple of 2^-32), then summed with integer
// adds / atomics, so the result is independent of summation order, launch shape and the
// number of GPUs (DESIGN R20).
enum StatField : int { kStEpisodes = 0, kStReturn = 1, kStLength = 2, kStReward = 3 };
__device__ __forceinline__ long long to_fx(float v) { return __float2ll_rn(v * 4294967296.0f); }

}  // namespace ws
