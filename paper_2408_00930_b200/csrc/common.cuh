// common.cuh -- device primitives of libws (sm_100a): Philox4x32-10, the draw layout,
// uniform / Gaussian conversions, the transcendental contract, warp helpers, stores.
//
// Product code.  Shares nothing with oracle/ (DESIGN.md section 2).
// Citation keys: P:n PAPER.md, S:n SPEC.md, BJ:5 north_star, Rk = DESIGN.md reading k.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

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
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void sincos_c(float x, float& s, float& c) {
  double sd, cd;
  sincos((double)x, &sd, &cd);
  s = (float)sd;
  c = (float)cd;
}
__device__ __forceinline__ float sin_c(float x) { return (float)sin((double)x); }
__device__ __forceinline__ float cos_c(float x) { return (float)cos((double)x); }

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
constexpr uint32_t kErrAction = 1u, kErrProbs = 2u;

__device__ __forceinline__ float warp_sum_f32(float v) {
  // xor butterfly; lane 0's value is the deterministic result used by the caller
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fadd(v, __shfl_xor_sync(kFull, v, o));
  return v;
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
