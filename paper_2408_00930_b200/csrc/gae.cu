// gae.cu -- NEXT-N2 (first stage): generalised advantage estimation over the time-major
// roll-out store, on sm_100a.
//
// Operation (SPEC compute_gae S:389-397; "supports actor-critic algorithms"; DESIGN
// reading R30): for every column c = e*A + a of the [T, E, A] store and t = T-1 .. 0,
//   terminated, or truncated without a terminal value:  delta = r_t - v_t;            A_t = delta
//   truncated with v_trunc given:       delta = (r_t + g*vtr_t) - v_t;  A_t = delta
//   otherwise:  delta = (r_t + g*v_{t+1}) - v_t;  A_t = delta + (g*l)*A_{t+1}      (v_T = bootstrap)
//   returns_t = A_t + v_t
// every operation rounded to fp32 in exactly this order (explicit __f*_rn intrinsics), so
// the result is bit-identical to the oracle's fp32 instance.
//
// Bound: HBM.  The recursion runs backwards in time, one column per thread; per element
// the kernel reads r, v (4 + 4 B) and the replica's done byte and writes A, returns
// (4 + 4 B): 16 + 1/A algorithmic bytes, a few fp32 operations.  The recursion's
// dependent chain is ~2 fp32 latencies per row, far below the HBM time per row, so the
// design problem is keeping enough bytes in flight with only E*A threads (C2: 10 000):
//  - k_gae_tma: a CTA owns W consecutive columns; one elected thread streams [Tc x W]
//    tiles of r, v (and done when the done rows are TMA-addressable) from the END of the
//    store backwards into an S-stage shared-memory ring with 2-D TMA tensor copies
//    (cp.async.bulk.tensor, mbarrier complete_tx), so S-1 tiles are in flight per CTA
//    while the threads run the recursion out of shared memory; out-of-range rows /
//    columns of the ragged last tile are zero-filled by the TMA unit and skipped.
//    When the done rows are not TMA-addressable (A > 1, or E not a multiple of 16) each
//    thread prefetches its replica's done bytes one tile ahead into registers.
//  - k_gae_lane: fallback for stores whose rows are not 16-byte aligned (E*A not a
//    multiple of 4, or unaligned pointers): the same recursion with per-thread loads
//    prefetched one 8-row tile ahead.  Same arithmetic, same results.
// Stores of A and returns: one coalesced 128-byte row segment per warp and row, streaming.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "kernels.h"

namespace ws {
namespace {

struct GaeDev {
  const float* rew;
  const uint8_t* done;
  const float* values;
  const float* bootstrap;
  const float* v_trunc;  // may be null
  float* adv;
  float* ret;
  int64_t E, C;  // replicas, columns (E * A)
  int32_t A, T;
  float gamma, lambda;
};

// one row of the recursion for column c (shared by both kernels: identical arithmetic)
// Branch-free (round 2): the three cases are evaluated and selected, so the only dependence
// between rows is the FMUL + FADD of the last line; the v_trunc load is predicated.  Each case
// keeps its own operation order (the values are those of the branching form).
__device__ __forceinline__ float gae_row(const GaeDev& g, float gl, float r, float v, uint32_t d, float v_next,
                                         float a_next, int64_t i) {
  const bool trunc = (d & 2u) != 0u, has_vt = g.v_trunc != nullptr;
  const bool stop = (d & 1u) || (trunc && !has_vt);
  const float vt = (trunc && has_vt) ? __ldg(g.v_trunc + i) : 0.0f;
  const float a_stop = __fsub_rn(r, v);
  const float a_trunc = __fsub_rn(__fadd_rn(r, __fmul_rn(g.gamma, vt)), v);
  const float delta = __fsub_rn(__fadd_rn(r, __fmul_rn(g.gamma, v_next)), v);
  const float a_run = __fadd_rn(delta, __fmul_rn(gl, a_next));
  return stop ? a_stop : (trunc ? a_trunc : a_run);
}

__device__ __forceinline__ void st_cs(float* p, float x) {
  asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(x) : "memory");
}

// ------------------------------------------------------------------ TMA / mbarrier PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

template <int W, int TC, int S>
struct GaeSmem {
  float r[S][TC][W];
  float v[S][TC][W];
  uint8_t d[S][TC][W];
  alignas(8) uint64_t full[S];
};

// W columns per CTA (= threads), TC rows per tile, S ring stages; kDoneTma: done tiles by TMA
template <int W, int TC, int S, bool kDoneTma>
__global__ void __launch_bounds__(W) k_gae_tma(const __grid_constant__ CUtensorMap tm_r,
                                               const __grid_constant__ CUtensorMap tm_v,
                                               const __grid_constant__ CUtensorMap tm_d, const GaeDev g) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<GaeSmem<W, TC, S>*>(smem_raw);
  const int j = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * W;
  const int64_t c = c0 + j;
  const bool live = c < g.C;
  const int K = (g.T + TC - 1) / TC;  // tiles; processed from the last (k = K-1) to the first
  constexpr uint32_t kTileBytes = 2u * TC * W * sizeof(float) + (kDoneTma ? TC * W : 0u);

  if (j == 0) {
    prefetch_tmap(&tm_r);
    prefetch_tmap(&tm_v);
    if (kDoneTma) prefetch_tmap(&tm_d);
    for (int s = 0; s < S; ++s) mbar_init(&sm.full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int q) {  // q-th tile in processing order -> stage q % S
    const int s = q % S;
    const int row0 = (K - 1 - q) * TC;
    mbar_expect_tx(&sm.full[s], kTileBytes);
    tma_load_2d(&sm.r[s][0][0], &tm_r, (int)c0, row0, &sm.full[s]);
    tma_load_2d(&sm.v[s][0][0], &tm_v, (int)c0, row0, &sm.full[s]);
    if (kDoneTma) tma_load_2d(&sm.d[s][0][0], &tm_d, (int)c0, row0, &sm.full[s]);
  };
  if (j == 0)
    for (int q = 0; q < S && q < K; ++q) issue(q);

  const float gl = __fmul_rn(g.gamma, g.lambda);
  const int64_t e = (live ? c : g.C - 1) / g.A;
  float v_next = live ? __ldg(g.bootstrap + c) : 0.0f;
  float a_next = 0.0f;
  uint8_t dn[TC];  // done bytes of the current tile (per-thread path)
  if (!kDoneTma) {
    const int row0 = (K - 1) * TC;
#pragma unroll
    for (int i = 0; i < TC; ++i) dn[i] = (row0 + i < g.T) ? __ldg(g.done + (int64_t)(row0 + i) * g.E + e) : 0;
  }
  for (int q = 0; q < K; ++q) {
    const int s = q % S;
    const int row0 = (K - 1 - q) * TC;
    uint8_t dn_next[TC];
    if (!kDoneTma) {  // prefetch the next tile's done bytes while this tile is processed
      const int nrow0 = row0 - TC;
#pragma unroll
      for (int i = 0; i < TC; ++i) dn_next[i] = (nrow0 >= 0) ? __ldg(g.done + (int64_t)(nrow0 + i) * g.E + e) : 0;
    }
    mbar_wait(&sm.full[s], (uint32_t)((q / S) & 1));
    if (row0 + TC <= g.T) {
      // full tile (every tile but a ragged last one): no row bounds checks, the element offset
      // stepped down by one row (C elements) per row instead of recomputed
      int64_t idx = (int64_t)(row0 + TC - 1) * g.C + c;
#pragma unroll
      for (int i = TC - 1; i >= 0; --i) {
        const float r = sm.r[s][i][j];
        const float v = sm.v[s][i][j];
        const uint32_t d = kDoneTma ? sm.d[s][i][j] : dn[i];
        const float a = gae_row(g, gl, r, v, d, v_next, a_next, idx);
        if (live) {
          st_cs(g.adv + idx, a);
          st_cs(g.ret + idx, __fadd_rn(a, v));
        }
        a_next = a;
        v_next = v;
        idx -= g.C;
      }
    } else {
#pragma unroll
      for (int i = TC - 1; i >= 0; --i) {
        const int t = row0 + i;
        if (t < g.T) {
          const float r = sm.r[s][i][j];
          const float v = sm.v[s][i][j];
          const uint32_t d = kDoneTma ? sm.d[s][i][j] : dn[i];
          const int64_t idx = (int64_t)t * g.C + c;
          const float a = gae_row(g, gl, r, v, d, v_next, a_next, idx);
          if (live) {
            st_cs(g.adv + idx, a);
            st_cs(g.ret + idx, __fadd_rn(a, v));
          }
          a_next = a;
          v_next = v;
        }
      }
    }
    if (!kDoneTma) {
#pragma unroll
      for (int i = 0; i < TC; ++i) dn[i] = dn_next[i];
    }
    __syncthreads();  // every thread is done with stage s before the TMA refills it
    if (j == 0 && q + S < K) issue(q + S);
  }
}

// fallback: per-thread loads, 8-row tiles prefetched one tile ahead
__global__ void __launch_bounds__(128) k_gae_lane(const GaeDev g) {
  constexpr int TC = 8;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.C) return;
  const int64_t e = c / g.A;
  const float gl = __fmul_rn(g.gamma, g.lambda);
  float v_next = __ldg(g.bootstrap + c), a_next = 0.0f;
  const int K = (g.T + TC - 1) / TC;
  float r[TC], v[TC];
  uint8_t d[TC];
  auto load = [&](int row0, float* rr, float* vv, uint8_t* dd) {
#pragma unroll
    for (int i = 0; i < TC; ++i) {
      const int t = row0 + i;
      const bool ok = t >= 0 && t < g.T;
      rr[i] = ok ? __ldg(g.rew + (int64_t)t * g.C + c) : 0.0f;
      vv[i] = ok ? __ldg(g.values + (int64_t)t * g.C + c) : 0.0f;
      dd[i] = ok ? __ldg(g.done + (int64_t)t * g.E + e) : 0;
    }
  };
  load((K - 1) * TC, r, v, d);
  for (int q = 0; q < K; ++q) {
    const int row0 = (K - 1 - q) * TC;
    float rn[TC], vn[TC];
    uint8_t dnx[TC];
    load(row0 - TC, rn, vn, dnx);
#pragma unroll
    for (int i = TC - 1; i >= 0; --i) {
      const int t = row0 + i;
      if (t < g.T) {
        const int64_t idx = (int64_t)t * g.C + c;
        const float a = gae_row(g, gl, r[i], v[i], d[i], v_next, a_next, idx);
        st_cs(g.adv + idx, a);
        st_cs(g.ret + idx, __fadd_rn(a, v[i]));
        a_next = a;
        v_next = v[i];
      }
    }
#pragma unroll
    for (int i = 0; i < TC; ++i) {
      r[i] = rn[i];
      v[i] = vn[i];
      d[i] = dnx[i];
    }
  }
}

// ------------------------------------------------------------------ host side
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  return fn;
}

// 2-D row-major [rows, cols] map with a [box_rows, box_cols] box; false if not encodable
bool make_map(CUtensorMap* m, CUtensorMapDataType dt, int elem, const void* base, int64_t rows, int64_t cols,
              int box_rows, int box_cols) {
  EncodeTiled enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * elem};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <int W, int TC, int S, bool kDoneTma>
cudaError_t launch_tma(const GaeDev& g, const CUtensorMap& mr, const CUtensorMap& mv, const CUtensorMap& md,
                       cudaStream_t s) {
  constexpr size_t smem = sizeof(GaeSmem<W, TC, S>);
  static uint64_t attr_done = 0;  // devices whose attribute is set (bit = ordinal)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64 || !((attr_done >> dev) & 1u)) {
    cudaError_t e = cudaFuncSetAttribute(k_gae_tma<W, TC, S, kDoneTma>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e) return e;
    if (dev < 64) attr_done |= 1ull << dev;
  }
  const unsigned grid = (unsigned)((g.C + W - 1) / W);
  k_gae_tma<W, TC, S, kDoneTma><<<grid, W, smem, s>>>(mr, mv, md, g);
  return cudaGetLastError();
}

}  // namespace

int gae_path(int64_t E, int32_t A, const void* rew, const void* values, const void* done) {
  const int64_t C = E * A;
  if (C % 4 != 0 || C > INT32_MAX || !aligned16(rew) || !aligned16(values) || !encoder()) return 0;
  return (A == 1 && E % 16 == 0 && aligned16(done)) ? 2 : 1;
}

cudaError_t launch_gae(const GaeArgs& a, cudaStream_t s, uint64_t* launches) {
  GaeDev g{a.rew, a.done, a.values, a.bootstrap, a.v_trunc, a.adv, a.ret, a.E, a.E * a.A, a.A, a.T,
           a.gamma, a.lambda};
  const int path = a.force_lane ? 0 : gae_path(a.E, a.A, a.rew, a.values, a.done);
  *launches += 1;
  if (path == 0) {
    k_gae_lane<<<(unsigned)((g.C + 127) / 128), 128, 0, s>>>(g);
    return cudaGetLastError();
  }
  // few columns (C2: 10 000): 32-column CTAs, a deep ring per CTA; many columns: 128
  const bool narrow = g.C < 148LL * 128 * 2;
  constexpr int TC = 32;
  const int W = narrow ? 32 : 128;
  CUtensorMap mr, mv, md;
  if (!make_map(&mr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.rew, a.T, g.C, TC, W) ||
      !make_map(&mv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.values, a.T, g.C, TC, W))
    return cudaErrorInvalidValue;
  const bool done_tma = path == 2 && make_map(&md, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.done, a.T, a.E, TC, W);
  if (!done_tma) md = mr;  // unused
  if (narrow)
    return done_tma ? launch_tma<32, TC, 6, true>(g, mr, mv, md, s) : launch_tma<32, TC, 6, false>(g, mr, mv, md, s);
  return done_tma ? launch_tma<128, TC, 3, true>(g, mr, mv, md, s) : launch_tma<128, TC, 3, false>(g, mr, mv, md, s);
}

}  // namespace ws
