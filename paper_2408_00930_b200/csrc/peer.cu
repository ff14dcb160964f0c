// peer.cu -- data-parallel training collectives over CUDA-IPC peer memory (NVLink /
// NVSwitch), fused with the optimizer step: the compute-then-collective pattern of the
// A2C / PPO update (gradient -> all-reduce -> clip + Adam) as ONE kernel, no NCCL call and no
// host round trip (include/ws.h "peer groups").
//
// A group is created on every rank with the same (world, n); each rank exports one buffer
//   [2 parities][world][n_pad] fp64 | arrival counter
// through a CUDA IPC handle; after the handles are exchanged (e.g. all_gather_object) every
// rank opens its peers' buffers.  A reduction with epoch k: every rank writes its n values
// (as fp64) into slot [k & 1][rank] of EVERY rank's buffer, fences at system scope, adds 1 to
// every rank's counter, waits (acquire, %globaltimer timeout -> sticky error) until its own
// counter reaches world * (k + 1), and sums the world slots of its own buffer in rank order --
// identical bits on every rank.  Two parities suffice: a rank can be at most one epoch ahead
// of any reader (it cannot pass epoch k+1's wait before every rank published k+1, i.e.
// finished reading k).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/ws.h"

struct ws_peer_group {
  int world = 0, rank = -1, n = 0, n_pad = 0, device = -1;
  double* own = nullptr;           // this rank's buffer
  void* open[8] = {};              // peers' buffers (IPC)
  uint64_t epoch = 0;
  uint32_t* err = nullptr;         // sticky error word (device)
  double timeout_s = 30.0;
};

namespace {

constexpr uint32_t kErrTimeout = 1u;

struct PgArgs {
  double* buf[8];
  int world, rank, n, n_pad;
};

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

// publish + signal + wait; returns false on timeout (block-uniform)
template <typename In>
__device__ bool exchange(const PgArgs& p, const In* in, uint64_t epoch, uint32_t* err, uint64_t timeout_ns) {
  const size_t slice = (size_t)p.n_pad;
  const size_t par = (size_t)(epoch & 1) * (size_t)p.world * slice;
  const size_t counter_off = 2 * (size_t)p.world * slice;
  for (int r = 0; r < p.world; ++r) {
    double* dst = p.buf[r] + par + (size_t)p.rank * slice;
    for (int i = threadIdx.x; i < p.n; i += blockDim.x) dst[i] = (double)in[i];
  }
  __threadfence_system();
  __syncthreads();
  if ((int)threadIdx.x < p.world)
    atomicAdd_system(reinterpret_cast<unsigned long long*>(p.buf[threadIdx.x] + counter_off), 1ull);
  __shared__ int timed_out;
  if (threadIdx.x == 0) {
    timed_out = 0;
    const unsigned long long target = (unsigned long long)p.world * (epoch + 1);
    const unsigned long long* c = reinterpret_cast<const unsigned long long*>(p.buf[p.rank] + counter_off);
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(c) < target) {
      if (global_ns() - t0 > timeout_ns) {
        timed_out = 1;
        atomicOr(err, kErrTimeout);
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
  return !timed_out;
}

__device__ __forceinline__ double sum_slot(const PgArgs& p, uint64_t epoch, int i) {
  const size_t slice = (size_t)p.n_pad;
  const double* g = p.buf[p.rank] + (size_t)(epoch & 1) * (size_t)p.world * slice;
  double acc = 0.0;
  for (int r = 0; r < p.world; ++r) acc += g[(size_t)r * slice + i];
  return acc;
}

template <typename In>
__global__ void __launch_bounds__(1024) k_pg_allreduce(const PgArgs p, const In* in, double* out, uint64_t epoch,
                                                       uint32_t* err, uint64_t timeout_ns) {
  if (!exchange(p, in, epoch, err, timeout_ns)) return;
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) out[i] = sum_slot(p, epoch, i);
}

// gradient all-reduce fused with the clip + Adam step (same arithmetic as ws_adam, a2c.cu)
__global__ void __launch_bounds__(1024) k_pg_allreduce_adam(const PgArgs p, const float* grad_local, float* params,
                                                            float* m, float* v, int step, double lr, double b1,
                                                            double b2, double eps, double max_norm, float* grad_out,
                                                            float* grad_norm, uint64_t epoch, uint32_t* err,
                                                            uint64_t timeout_ns) {
  if (!exchange(p, grad_local, epoch, err, timeout_ns)) return;
  __shared__ double red[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
    const double g = (double)(float)sum_slot(p, epoch, i);  // the all-reduced fp32 gradient
    s = fma(g, g, s);
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
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
    const float gsum = (float)sum_slot(p, epoch, i);
    if (grad_out) grad_out[i] = gsum;
    const double gi = (double)gsum * scale;
    const double mi = b1 * (double)m[i] + (1.0 - b1) * gi;
    const double vi = b2 * (double)v[i] + (1.0 - b2) * gi * gi;
    params[i] = (float)((double)params[i] - lr * (mi / c1) / (sqrt(vi / c2) + eps));
    m[i] = (float)mi;
    v[i] = (float)vi;
  }
}

PgArgs args_of(const ws_peer_group* g) {
  PgArgs a{};
  for (int r = 0; r < g->world; ++r) a.buf[r] = r == g->rank ? g->own : static_cast<double*>(g->open[r]);
  a.world = g->world;
  a.rank = g->rank;
  a.n = g->n;
  a.n_pad = g->n_pad;
  return a;
}

void release(ws_peer_group* g) {
  for (int r = 0; r < 8; ++r)
    if (g->open[r]) {
      cudaIpcCloseMemHandle(g->open[r]);
      g->open[r] = nullptr;
    }
  if (g->own) cudaFree(g->own);
  if (g->err) cudaFree(g->err);
  g->own = nullptr;
  g->err = nullptr;
}

}  // namespace

extern "C" {

ws_status ws_pgroup_create(int32_t world, int32_t n, ws_peer_group** out, ws_ipc_handle* handle) {
  if (!out || !handle || world < 1 || world > 8 || n < 1 || n > 65536) return WS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  ws_peer_group* g = new ws_peer_group();
  g->world = world;
  g->n = n;
  g->n_pad = (n + 3) & ~3;  // 32-byte slots
  cudaGetDevice(&g->device);
  const size_t words = 2 * (size_t)world * (size_t)g->n_pad + 4;  // + arrival counter (32-byte pad)
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&g->own), words * sizeof(double));
  if (!e) e = cudaMemset(g->own, 0, words * sizeof(double));
  if (!e) e = cudaMalloc(reinterpret_cast<void**>(&g->err), sizeof(uint32_t));
  if (!e) e = cudaMemset(g->err, 0, sizeof(uint32_t));
  cudaIpcMemHandle_t ih;
  if (!e) e = cudaIpcGetMemHandle(&ih, g->own);
  if (e) {
    release(g);
    delete g;
    return WS_ERR_CUDA;
  }
  std::memset(handle, 0, sizeof(*handle));
  std::memcpy(handle->bytes, &ih, sizeof(ih));
  *out = g;
  return WS_OK;
}

ws_status ws_pgroup_attach(ws_peer_group* g, int32_t rank, const ws_ipc_handle* handles) {
  if (!g || !handles || rank < 0 || rank >= g->world) return WS_ERR_INVALID_ARGUMENT;
  for (int r = 0; r < g->world; ++r) {
    if (r == rank) continue;
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, handles[r].bytes, sizeof(ih));
    if (cudaIpcOpenMemHandle(&g->open[r], ih, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return WS_ERR_CUDA;
  }
  g->rank = rank;
  g->epoch = 0;
  return WS_OK;
}

ws_status ws_pgroup_destroy(ws_peer_group* g) {
  if (!g) return WS_OK;
  cudaDeviceSynchronize();
  release(g);
  delete g;
  return WS_OK;
}

ws_status ws_pgroup_status(ws_peer_group* g) {
  if (!g) return WS_ERR_INVALID_ARGUMENT;
  uint32_t w = 0;
  if (cudaMemcpy(&w, g->err, sizeof(w), cudaMemcpyDeviceToHost) != cudaSuccess) return WS_ERR_CUDA;
  return w ? WS_ERR_PEER : WS_OK;
}

ws_status ws_pgroup_allreduce(ws_peer_group* g, const void* in, int32_t in_is_f32, double* out, void* stream) {
  if (!g || g->rank < 0 || !in || !out) return WS_ERR_INVALID_ARGUMENT;
  const PgArgs a = args_of(g);
  const uint64_t to = (uint64_t)(g->timeout_s * 1e9);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (in_is_f32)
    k_pg_allreduce<float><<<1, 1024, 0, s>>>(a, static_cast<const float*>(in), out, g->epoch, g->err, to);
  else
    k_pg_allreduce<double><<<1, 1024, 0, s>>>(a, static_cast<const double*>(in), out, g->epoch, g->err, to);
  g->epoch += 1;
  return cudaGetLastError() ? WS_ERR_CUDA : WS_OK;
}

ws_status ws_pgroup_allreduce_adam(ws_peer_group* g, const float* grad, float* params, float* m, float* v, int32_t step,
                                   float lr, float beta1, float beta2, float eps, float max_norm, float* grad_out,
                                   float* grad_norm, void* stream) {
  if (!g || g->rank < 0 || !grad || !params || !m || !v || step < 1) return WS_ERR_INVALID_ARGUMENT;
  const PgArgs a = args_of(g);
  k_pg_allreduce_adam<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(
      a, grad, params, m, v, step, lr, beta1, beta2, eps, max_norm, grad_out, grad_norm, g->epoch, g->err,
      (uint64_t)(g->timeout_s * 1e9));
  g->epoch += 1;
  return cudaGetLastError() ? WS_ERR_CUDA : WS_OK;
}

}  // extern "C"
