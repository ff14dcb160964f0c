// runtime.cu -- host runtime of libws: the C ABI of include/ws.h (data manager, function
// manager dispatch, sampler and reset entry points), allocation, streams, sticky errors.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ws.h"
#include "common.cuh"
#include "kernels.h"

namespace {

struct EnvSpec {
  ws::EnvKind kind;
  int obs_dim, n_actions, act_dim, state_dim, max_steps;
  void* user = nullptr;  // NEXT-N4 registry entry (kind == kUser)
  int n_params = 0;
};

bool lookup_env(const char* name, int A, int p0, EnvSpec* out) {
  if (!name) return false;
  std::string n(name);
  if (n == "cartpole") { *out = {ws::kCartPole, 4, 2, 1, 4, 500}; return true; }
  if (n == "acrobot") { *out = {ws::kAcrobot, 6, 3, 1, 4, 500}; return true; }
  if (n == "pendulum") { *out = {ws::kPendulum, 3, 0, 1, 2, 200}; return true; }
  if (n == "tag") { *out = {ws::kTag, 4, 5, 1, 0, 200}; return true; }
  if (n == "surface") {
    const int D = p0 > 0 ? p0 : 20;
    *out = {ws::kSurface, D + 1, 0, D, D, 200};
    return true;
  }
  if (n == "dummy") { *out = {ws::kDummy, 4, 2, 1, 0, 100}; return true; }
  ws::UserSpec u;
  if (ws::user_env_spec(name, &u)) {  // NEXT-N4: registered at run time (composer.cu)
    *out = {ws::kUser, u.obs_dim, u.n_actions, u.act_dim > 0 ? u.act_dim : 1, u.state_dim, u.max_steps, u.handle,
            u.n_params};
    return true;
  }
  (void)A;
  return false;
}

bool surface_dim_supported(int D) {
  return D == 2 || D == 3 || D == 4 || D == 8 || D == 16 || D == 20 || D == 32;
}

// NVTX range per public call (SURVEY 5 tracing): header-only NVTX v3, a no-op unless a
// profiler (nsys / ncu --nvtx) is attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  explicit DeviceGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
      changed = cudaSetDevice(dev) == cudaSuccess;
    }
  }
  ~DeviceGuard() {
    if (changed) cudaSetDevice(prev);
  }
};

}  // namespace

struct ws_env {
  EnvSpec spec{};
  std::string env_name;
  int64_t E = 0, offset = 0, E_global = 0;
  int32_t A = 1;
  uint64_t seed = 0;
  int device = -1;
  cudaStream_t stream = nullptr;
  int32_t T_cap = 0, cursor = 0, sampled_slot = -1;
  uint64_t t = 0;
  int32_t max_steps = 0, write_logp = 1, p0 = 0, p1 = 0, block = 128;
  ws_alloc_fn alloc = nullptr;
  ws_free_fn free_fn = nullptr;
  void* alloc_user = nullptr;
  std::vector<std::pair<void*, size_t>> allocs;
  // live state
  float* state = nullptr;
  int32_t* tstate = nullptr;
  float* obs_live = nullptr;
  int32_t* ep_step = nullptr;
  uint32_t* reset_count = nullptr;
  float* ep_ret = nullptr;
  uint32_t* err = nullptr;
  // store
  float* obs = nullptr;
  void* act = nullptr;
  float* logp = nullptr;
  float* rew = nullptr;
  uint8_t* done = nullptr;
  unsigned long long* stats = nullptr;  // [T_cap, 4] fixed-point int64
  uint32_t* plan = nullptr;
  // NEXT-N4 per-replica parameters / shared data of a registered env (caller-owned)
  const float* user_prm = nullptr;
  const float* user_shared = nullptr;
  // e2e staging
  float* staging = nullptr;
  int64_t staging_n = 0;
  std::vector<long long> host_stats;
  // pipelined host roll-outs (ws_rollout_host_submit / _wait): two pinned result slots
  struct HostSlot {
    long long* st = nullptr;  // pinned [T_cap][4]
    cudaEvent_t done = nullptr;
    float* staging = nullptr;  // device copy of this slot's probabilities
    cudaEvent_t copied = nullptr, consumed = nullptr;
    bool used = false;
    int32_t T = 0;
    bool pending = false;
  } hslot[2];
  int64_t hslot_n = 0;                // probabilities per slot staging buffer
  cudaStream_t copy_stream = nullptr;  // H2D of the next submission, beside the running roll-out
  uint64_t launches = 0;
  std::string last_error;
  // optional per-kernel CUDA-event timing (ws_enable_kernel_timing)
  struct Ring {
    std::vector<cudaEvent_t> b, e;
    int n = 0, open = 0;
    uint64_t calls = 0;  // launches seen (the sampling period picks every period-th)
    bool skip = false;   // the open launch is not sampled
  };
  bool timing = false;
  int timing_period = 1;  // events on every period-th launch of a timed class
  uint32_t timed_mask = 0;  // kernels (bit = KernelId) that get events
  // cross-GPU statistics reduction over peer memory (ws_peer_export / ws_peer_attach)
  unsigned long long* peer_own = nullptr;  // this rank's gather buffer (cudaMalloc, IPC-exported)
  int32_t peer_world = 0, peer_rank = -1, peer_tcap = 0;
  bool peer_attached = false;
  void* peer_open[ws::kMaxPeers] = {};     // peers' buffers opened through CUDA IPC
  uint64_t peer_epoch = 0;
  double peer_timeout_s = 30.0;
  Ring rings[ws::kKCount];
  // device step counter (ws_enable_device_clock): authoritative while dev_clock is set
  uint64_t* t_dev = nullptr;
  bool dev_clock = false;
};

namespace {

ws_status fail(ws_env* h, ws_status s, const std::string& msg) {
  if (h) h->last_error = msg;
  return s;
}

ws_status cuda_fail(ws_env* h, cudaError_t e, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorString(e);
  if (h) h->last_error = m;
  return e == cudaErrorMemoryAllocation ? WS_ERR_OUT_OF_MEMORY : WS_ERR_CUDA;
}

void* dev_alloc(ws_env* h, size_t bytes, cudaError_t* err) {
  *err = cudaSuccess;
  if (bytes == 0) return nullptr;
  bytes = (bytes + 255) & ~size_t(255);
  void* p = nullptr;
  if (h->alloc) {
    p = h->alloc(bytes, (void*)h->stream, h->alloc_user);
    if (!p) *err = cudaErrorMemoryAllocation;
  } else {
    *err = cudaMalloc(&p, bytes);
    if (*err != cudaSuccess) p = nullptr;
  }
  if (p) h->allocs.emplace_back(p, bytes);
  return p;
}

void free_all(ws_env* h) {
  for (auto& pr : h->allocs) {
    if (h->free_fn) h->free_fn(pr.first, pr.second, (void*)h->stream, h->alloc_user);
    else cudaFree(pr.first);
  }
  h->allocs.clear();
}

void peer_release(ws_env* h) {
  for (int r = 0; r < ws::kMaxPeers; ++r)
    if (h->peer_open[r]) {
      cudaIpcCloseMemHandle(h->peer_open[r]);
      h->peer_open[r] = nullptr;
    }
  if (h->peer_own) cudaFree(h->peer_own);
  h->peer_own = nullptr;
  h->peer_attached = false;
  h->peer_world = 0;
  h->peer_rank = -1;
}

ws::KArgs kargs(const ws_env* h) {
  ws::KArgs a{};
  a.obs = h->obs;
  a.act = h->act;
  a.logp = h->logp;
  a.rew = h->rew;
  a.done = h->done;
  a.stats = h->stats;
  a.state = h->state;
  a.tstate = h->tstate;
  a.obs_live = h->obs_live;
  a.ep_step = h->ep_step;
  a.reset_count = h->reset_count;
  a.ep_ret = h->ep_ret;
  a.err = h->err;
  a.plan = h->plan;
  a.E = h->E;
  a.offset = h->offset;
  a.A = h->A;
  a.T_cap = h->T_cap;
  a.max_steps = h->max_steps;
  a.write_logp = h->write_logp;
  a.p0 = h->p0;
  a.p1 = h->p1;
  a.k0 = (uint32_t)h->seed;
  a.k1 = (uint32_t)(h->seed >> 32);
  a.t_dev = h->dev_clock ? h->t_dev : nullptr;
  return a;
}

constexpr int kTimingCap = 256;

void mark_kernel(void* ctx, int kernel, int phase) {
  ws_env* h = static_cast<ws_env*>(ctx);
  if (!((h->timed_mask >> kernel) & 1u)) return;
  ws_env::Ring& r = h->rings[kernel];
  const int i = r.n % kTimingCap;
  if (phase == 0) {
    r.skip = (r.calls++ % (uint64_t)h->timing_period) != 0;
    if (!r.skip) cudaEventRecord(r.b[i], h->stream);
  } else if (!r.skip) {
    cudaEventRecord(r.e[i], h->stream);
    r.n += 1;
  }
}

ws::Launch launch_of(ws_env* h) {
  ws::Launch l{h->spec.kind, h->block, h->stream};
  if (h->timing) {
    l.mark = mark_kernel;
    l.mark_ctx = h;
  }
  return l;
}

// Store allocation: once, the first time it is needed (lazy sizing, never regrown).
ws_status ensure_store(ws_env* h, int32_t T) {
  if (h->T_cap > 0) return WS_OK;
  if (T < 1) return fail(h, WS_ERR_INVALID_ARGUMENT, "store capacity must be >= 1");
  const size_t TEA = (size_t)T * (size_t)h->E * (size_t)h->A;
  const size_t act_elems = TEA * (size_t)(h->spec.n_actions ? 1 : h->spec.act_dim);
  cudaError_t e;
  h->obs = (float*)dev_alloc(h, TEA * h->spec.obs_dim * sizeof(float), &e);
  if (e) return cuda_fail(h, e, "alloc obs");
  h->act = dev_alloc(h, act_elems * 4, &e);
  if (e) return cuda_fail(h, e, "alloc act");
  h->logp = (float*)dev_alloc(h, TEA * sizeof(float), &e);
  if (e) return cuda_fail(h, e, "alloc logp");
  h->rew = (float*)dev_alloc(h, TEA * sizeof(float), &e);
  if (e) return cuda_fail(h, e, "alloc rew");
  h->done = (uint8_t*)dev_alloc(h, (size_t)T * h->E, &e);
  if (e) return cuda_fail(h, e, "alloc done");
  h->stats = (unsigned long long*)dev_alloc(h, (size_t)T * 4 * sizeof(unsigned long long), &e);
  if (e) return cuda_fail(h, e, "alloc stats");
  if (h->spec.n_actions && h->spec.kind != ws::kTag) {
    h->plan = (uint32_t*)dev_alloc(h, (size_t)((T + 3) / 4) * h->E * sizeof(uint32_t), &e);
    if (e) return cuda_fail(h, e, "alloc plan");
  }
  if ((e = cudaMemsetAsync(h->stats, 0, (size_t)T * 4 * sizeof(unsigned long long), h->stream)))
    return cuda_fail(h, e, "memset stats");
  h->T_cap = T;
  return WS_OK;
}

ws_status check(ws_env* h) {
  if (!h) return WS_ERR_INVALID_ARGUMENT;
  h->last_error.clear();
  return WS_OK;
}

}  // namespace

extern "C" {

int32_t ws_abi_version(void) { return WS_ABI_VERSION; }

const char* ws_status_string(ws_status s) {
  switch (s) {
    case WS_OK: return "ok";
    case WS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case WS_ERR_UNKNOWN_ENV: return "unknown environment";
    case WS_ERR_INVALID_ACTION: return "invalid action";
    case WS_ERR_INVALID_PROBS: return "invalid probabilities";
    case WS_ERR_OUT_OF_RANGE: return "slot out of range";
    case WS_ERR_BAD_STATE: return "bad call order";
    case WS_ERR_OUT_OF_MEMORY: return "out of memory";
    case WS_ERR_CUDA: return "CUDA error";
    case WS_ERR_PEER: return "peer reduction timed out";
  }
  return "unknown status";
}

const char* ws_last_error(const ws_env* h) { return h ? h->last_error.c_str() : ""; }

ws_status ws_config_init(ws_config* cfg) {
  if (!cfg) return WS_ERR_INVALID_ARGUMENT;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->n_agents = 1;
  cfg->device = -1;
  cfg->write_logp = 1;
  return WS_OK;
}

ws_status ws_create(int64_t n_envs, int32_t n_agents, const char* env, uint64_t seed, ws_env** out) {
  ws_config c;
  ws_config_init(&c);
  c.n_envs = n_envs;
  c.n_agents = n_agents;
  c.env = env;
  c.seed = seed;
  return ws_create_ex(&c, out);
}

ws_status ws_set_time(ws_env* h, uint64_t t) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (h->dev_clock) {
    DeviceGuard g(h->device);
    cudaError_t e;
    if ((e = cudaMemcpyAsync(h->t_dev, &t, sizeof(t), cudaMemcpyHostToDevice, h->stream)) ||
        (e = cudaStreamSynchronize(h->stream)))
      return cuda_fail(h, e, "ws_set_time device clock");
  }
  h->t = t;
  h->cursor = 0;
  h->sampled_slot = -1;
  return WS_OK;
}

ws_status ws_set_env_data(ws_env* h, const float* prm, const float* shared) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (h->spec.kind != ws::kUser) return fail(h, WS_ERR_INVALID_ARGUMENT, "ws_set_env_data: registered envs only");
  if (h->spec.n_params > 0 && !prm) return fail(h, WS_ERR_INVALID_ARGUMENT, "this env needs per-replica parameters");
  h->user_prm = prm;
  h->user_shared = shared;
  return WS_OK;
}

ws_status ws_create_ex(const ws_config* cfg, ws_env** out) {
  if (!out) return WS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (!cfg) return WS_ERR_INVALID_ARGUMENT;
  // ---- synchronous validation; no CUDA call before this point
  EnvSpec spec;
  if (!lookup_env(cfg->env, cfg->n_agents, cfg->param0, &spec)) return WS_ERR_UNKNOWN_ENV;
  if (cfg->n_envs < 1 || cfg->n_agents < 1 || cfg->env_offset < 0) return WS_ERR_INVALID_ARGUMENT;
  const int64_t Eg = cfg->n_envs_global > 0 ? cfg->n_envs_global : cfg->env_offset + cfg->n_envs;
  if (cfg->env_offset + cfg->n_envs > Eg || Eg > (int64_t)UINT32_MAX) return WS_ERR_INVALID_ARGUMENT;
  if (spec.kind != ws::kTag && cfg->n_agents != 1) return WS_ERR_INVALID_ARGUMENT;
  if (spec.kind == ws::kUser && spec.n_params > 0 && !cfg->env_prm) return WS_ERR_INVALID_ARGUMENT;
  if (cfg->t_capacity < 0 || cfg->max_steps < 0) return WS_ERR_INVALID_ARGUMENT;
  if (cfg->block_size != 0 && (cfg->block_size % 32 != 0 || cfg->block_size > 256 || cfg->block_size < 32))
    return WS_ERR_INVALID_ARGUMENT;
  int p0 = cfg->param0, p1 = cfg->param1;
  if (spec.kind == ws::kTag) {
    p0 = p0 > 0 ? p0 : 20;
    p1 = p1 > 0 ? p1 : std::max(1, cfg->n_agents / 10);
    if (p0 < 2 || p0 > 64 || p1 > cfg->n_agents || cfg->n_agents > 1024) return WS_ERR_INVALID_ARGUMENT;
  } else if (spec.kind == ws::kSurface) {
    p0 = p0 > 0 ? p0 : 20;
    if (!surface_dim_supported(p0)) return WS_ERR_INVALID_ARGUMENT;
  }
  // ---- handle
  ws_env* h = new ws_env();
  h->spec = spec;
  h->env_name = cfg->env;
  h->E = cfg->n_envs;
  h->offset = cfg->env_offset;
  h->E_global = Eg;
  h->A = cfg->n_agents;
  h->seed = cfg->seed;
  h->device = cfg->device;
  h->stream = (cudaStream_t)cfg->stream;
  h->max_steps = cfg->max_steps > 0 ? cfg->max_steps : spec.max_steps;
  h->write_logp = cfg->write_logp ? 1 : 0;
  h->p0 = p0;
  h->p1 = p1;
  h->block = cfg->block_size > 0 ? cfg->block_size : 128;
  h->alloc = cfg->alloc;
  h->free_fn = cfg->free;
  h->alloc_user = cfg->alloc_user;
  h->user_prm = cfg->env_prm;
  h->user_shared = cfg->env_shared;
  DeviceGuard g(h->device);
  if (h->device < 0) cudaGetDevice(&h->device);
  cudaError_t e;
  const size_t EA = (size_t)h->E * h->A;
  if (spec.state_dim) {
    h->state = (float*)dev_alloc(h, (size_t)h->E * spec.state_dim * sizeof(float), &e);
    if (e) { ws_status s = cuda_fail(h, e, "alloc state"); free_all(h); delete h; return s; }
  }
  if (spec.kind == ws::kTag) {
    h->tstate = (int32_t*)dev_alloc(h, EA * 3 * sizeof(int32_t), &e);
    if (e) { ws_status s = cuda_fail(h, e, "alloc tag state"); free_all(h); delete h; return s; }
  }
  h->obs_live = (float*)dev_alloc(h, EA * spec.obs_dim * sizeof(float), &e);
  if (!e) h->ep_step = (int32_t*)dev_alloc(h, (size_t)h->E * sizeof(int32_t), &e);
  if (!e) h->reset_count = (uint32_t*)dev_alloc(h, (size_t)h->E * sizeof(uint32_t), &e);
  if (!e) h->ep_ret = (float*)dev_alloc(h, EA * sizeof(float), &e);
  if (!e) h->err = (uint32_t*)dev_alloc(h, sizeof(uint32_t), &e);
  if (e) { ws_status s = cuda_fail(h, e, "alloc live state"); free_all(h); delete h; return s; }
  if (cfg->t_capacity > 0) {
    ws_status s = ensure_store(h, cfg->t_capacity);
    if (s != WS_OK) { free_all(h); delete h; return s; }
  }
  ws_status s = ws_reset(h);
  if (s != WS_OK) { free_all(h); delete h; return s; }
  *out = h;
  return WS_OK;
}

ws_status ws_destroy(ws_env* h) {
  if (!h) return WS_OK;
  DeviceGuard g(h->device);
  cudaStreamSynchronize(h->stream);
  for (auto& r : h->rings) {
    for (auto ev : r.b) cudaEventDestroy(ev);
    for (auto ev : r.e) cudaEventDestroy(ev);
  }
  peer_release(h);
  for (auto& hs : h->hslot) {
    if (hs.st) cudaFreeHost(hs.st);
    if (hs.done) cudaEventDestroy(hs.done);
    if (hs.copied) cudaEventDestroy(hs.copied);
    if (hs.consumed) cudaEventDestroy(hs.consumed);
  }
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  free_all(h);
  delete h;
  return WS_OK;
}

ws_status ws_reset(ws_env* h) {
  NvtxRange nvtx_("ws_reset");
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  cudaError_t e = cudaMemsetAsync(h->err, 0, sizeof(uint32_t), h->stream);
  if (e) return cuda_fail(h, e, "ws_reset memset");
  if (h->stats && (e = cudaMemsetAsync(h->stats, 0, (size_t)h->T_cap * 4 * sizeof(unsigned long long), h->stream)))
    return cuda_fail(h, e, "ws_reset memset stats");
  if (h->spec.kind == ws::kUser) {
    if (h->timing) mark_kernel(h, ws::kKReset, 0);
    e = ws::launch_user_reset(ws::UserLaunch{kargs(h), h->spec.user, h->user_prm, h->user_shared, h->stream});
    if (h->timing) mark_kernel(h, ws::kKReset, 1);
    h->launches += 1;
  } else {
    e = ws::launch_reset(kargs(h), launch_of(h), &h->launches);
  }
  if (e) return cuda_fail(h, e, "reset kernel");
  h->t = 0;
  h->cursor = 0;
  h->sampled_slot = -1;
  if (h->dev_clock && (e = cudaMemsetAsync(h->t_dev, 0, sizeof(uint64_t), h->stream)))
    return cuda_fail(h, e, "ws_reset device clock");
  return WS_OK;
}

ws_status ws_enable_device_clock(ws_env* h, int32_t enable) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  cudaError_t e;
  if (enable && !h->dev_clock) {
    if (!h->t_dev) {
      h->t_dev = (uint64_t*)dev_alloc(h, sizeof(uint64_t), &e);
      if (e) return cuda_fail(h, e, "alloc device clock");
    }
    const uint64_t t = h->t;
    if ((e = cudaMemcpyAsync(h->t_dev, &t, sizeof(t), cudaMemcpyHostToDevice, h->stream)) ||
        (e = cudaStreamSynchronize(h->stream)))
      return cuda_fail(h, e, "ws_enable_device_clock");
    h->dev_clock = true;
  } else if (!enable && h->dev_clock) {
    uint64_t t = 0;
    if ((e = cudaMemcpyAsync(&t, h->t_dev, sizeof(t), cudaMemcpyDeviceToHost, h->stream)) ||
        (e = cudaStreamSynchronize(h->stream)))
      return cuda_fail(h, e, "ws_enable_device_clock");
    h->t = t;
    h->dev_clock = false;
  }
  return WS_OK;
}

ws_status ws_rewind(ws_env* h) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  h->cursor = 0;
  h->sampled_slot = -1;
  return WS_OK;
}

ws_status ws_sample(ws_env* h, const float* probs, int64_t row_stride) {
  NvtxRange nvtx_("ws_sample");
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (!probs || row_stride < 0) return fail(h, WS_ERR_INVALID_ARGUMENT, "probs must be a device pointer, row_stride >= 0");
  DeviceGuard g(h->device);
  ws_status s = ensure_store(h, 1000);
  if (s) return s;
  if (h->cursor >= h->T_cap) return fail(h, WS_ERR_OUT_OF_RANGE, "cursor at store capacity (ws_rewind)");
  if (h->spec.kind == ws::kUser) return fail(h, WS_ERR_INVALID_ARGUMENT, "registered envs: ws_rollout only");
  cudaError_t e = ws::launch_sample(kargs(h), launch_of(h), h->cursor, h->t, probs, row_stride, &h->launches);
  if (e) return cuda_fail(h, e, "sample kernel");
  h->sampled_slot = h->cursor;
  return WS_OK;
}

ws_status ws_step(ws_env* h, const void* actions) {
  NvtxRange nvtx_("ws_step");
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  ws_status s = ensure_store(h, 1000);
  if (s) return s;
  if (h->cursor >= h->T_cap) return fail(h, WS_ERR_OUT_OF_RANGE, "cursor at store capacity (ws_rewind)");
  if (h->spec.kind == ws::kUser) return fail(h, WS_ERR_INVALID_ARGUMENT, "registered envs: ws_rollout only");
  if (!actions && h->sampled_slot != h->cursor) return fail(h, WS_ERR_BAD_STATE, "ws_step(NULL) needs ws_sample first");
  cudaError_t e = cudaMemsetAsync(h->stats + 4 * (size_t)h->cursor, 0, 4 * sizeof(unsigned long long), h->stream);
  if (!e) e = ws::launch_step(kargs(h), launch_of(h), h->cursor, actions, &h->launches);
  if (e) return cuda_fail(h, e, "step kernel");
  h->cursor += 1;
  h->t += 1;
  h->sampled_slot = -1;
  return WS_OK;
}

/* A8 across GPUs after any roll-out entry point (ws_rollout, the policy roll-outs, the staged
 * pipeline): when peer statistics are attached, merge the [T, 4] slab in place over peer memory
 * (k_peer_allreduce, no NCCL call).  No-op otherwise. */
static ws_status peer_merge(ws_env* h, int32_t T) {
  if (!h->peer_attached) return WS_OK;
  ws::PeerArgs pa{};
  for (int r = 0; r < h->peer_world; ++r)
    pa.gather[r] = r == h->peer_rank ? h->peer_own : static_cast<unsigned long long*>(h->peer_open[r]);
  pa.rank = h->peer_rank;
  pa.world = h->peer_world;
  pa.t_cap = h->peer_tcap;
  cudaError_t e = ws::launch_peer_allreduce(h->stats, T, pa, h->peer_epoch, h->stats, h->err, h->peer_timeout_s,
                                            h->stream);
  if (e) return cuda_fail(h, e, "peer statistics reduction");
  h->peer_epoch += 1;
  h->launches += 1;
  return WS_OK;
}

ws_status ws_rollout(ws_env* h, int32_t T, const float* probs, int64_t row_stride, int64_t step_stride) {
  NvtxRange nvtx_("ws_rollout");
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (h->dev_clock)
    return fail(h, WS_ERR_BAD_STATE, "device clock on (ws_enable_device_clock): fused roll-outs take the host step index");
  if (T < 1) return fail(h, WS_ERR_INVALID_ARGUMENT, "T must be >= 1 (S:166)");
  if (!probs || row_stride < 0 || step_stride < 0) return fail(h, WS_ERR_INVALID_ARGUMENT, "bad probs / strides");
  DeviceGuard g(h->device);
  ws_status s = ensure_store(h, T);
  if (s) return s;
  if (T > h->T_cap) return fail(h, WS_ERR_OUT_OF_RANGE, "T exceeds the store capacity (S:79)");
  // the discrete lane envs' plan kernel clears the statistics slab itself
  const bool plan_zeroes = h->spec.kind == ws::kCartPole || h->spec.kind == ws::kAcrobot || h->spec.kind == ws::kDummy;
  cudaError_t e = plan_zeroes ? cudaSuccess
                              : cudaMemsetAsync(h->stats, 0, (size_t)T * 4 * sizeof(unsigned long long), h->stream);
  if (!e && h->spec.kind == ws::kUser) {  // NEXT-N4: NVRTC-compiled fused roll-out
    if (h->timing) mark_kernel(h, ws::kKRollout, 0);
    e = ws::launch_user_rollout(ws::UserLaunch{kargs(h), h->spec.user, h->user_prm, h->user_shared, h->stream}, T,
                                h->t, probs, row_stride, step_stride);
    if (h->timing) mark_kernel(h, ws::kKRollout, 1);
    h->launches += 1;
  } else if (!e) {
    e = ws::launch_rollout(kargs(h), launch_of(h), T, h->t, probs, row_stride, step_stride, &h->launches);
  }
  if (e) return cuda_fail(h, e, "rollout kernel");
  if ((s = peer_merge(h, T))) return s;
  h->t += (uint64_t)T;
  h->cursor = T;
  h->sampled_slot = -1;
  return WS_OK;
}

static void sum_stats(const long long* st, int n, ws_stats* out) {
  long long ep = 0, ln = 0, ret = 0, rew = 0;  // exact integer sums (fixed point, R20)
  for (int i = 0; i < n; ++i) {
    ep += st[4 * i + 0];
    ret += st[4 * i + 1];
    ln += st[4 * i + 2];
    rew += st[4 * i + 3];
  }
  ws_stats r{};
  r.episodes = (double)ep;
  r.sum_return = (double)ret * 0x1.0p-32;
  r.sum_length = (double)ln;
  r.sum_reward = (double)rew * 0x1.0p-32;
  const double nan = std::numeric_limits<double>::quiet_NaN();
  r.mean_return = r.episodes > 0 ? r.sum_return / r.episodes : nan;
  r.mean_length = r.episodes > 0 ? r.sum_length / r.episodes : nan;
  *out = r;
}

static ws_status run_policy(ws_env* h, int32_t T, const float* weights, int32_t hidden, float* values,
                            float* bootstrap, float* values_trunc = nullptr) {
  NvtxRange nvtx_("ws_rollout_policy");
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (h->dev_clock)
    return fail(h, WS_ERR_BAD_STATE, "device clock on (ws_enable_device_clock): fused roll-outs take the host step index");
  if (T < 1) return fail(h, WS_ERR_INVALID_ARGUMENT, "T must be >= 1 (S:166)");
  if (!weights || (hidden != 32 && hidden != 64)) return fail(h, WS_ERR_INVALID_ARGUMENT, "weights / hidden (32 or 64)");
  if ((h->A != 1 && h->spec.kind != ws::kTag) || (h->spec.n_actions < 1 && h->spec.kind != ws::kPendulum) ||
      (h->spec.kind == ws::kTag && h->A > 128))
    return fail(h, WS_ERR_INVALID_ARGUMENT,
                "policy roll-out: discrete envs (tag: <= 128 agents) or pendulum (Gaussian)");
  DeviceGuard g(h->device);
  ws_status st = ensure_store(h, T);
  if (st) return st;
  if (T > h->T_cap) return fail(h, WS_ERR_OUT_OF_RANGE, "T exceeds the store capacity (S:79)");
  cudaError_t e = cudaMemsetAsync(h->stats, 0, (size_t)T * 4 * sizeof(unsigned long long), h->stream);
  if (!e && h->spec.kind == ws::kUser) {  // NEXT-N4 registered env: the template's policy loop
    if (h->timing) mark_kernel(h, ws::kKRollout, 0);
    e = ws::launch_user_policy(ws::UserLaunch{kargs(h), h->spec.user, h->user_prm, h->user_shared, h->stream}, T,
                               h->t, weights, hidden, values, bootstrap);
    if (h->timing) mark_kernel(h, ws::kKRollout, 1);
    h->launches += 1;
  } else if (!e) {
    e = ws::launch_rollout_policy(kargs(h), launch_of(h), T, h->t, weights, hidden, &h->launches, values, bootstrap,
                                  values_trunc);
  }
  if (e) return cuda_fail(h, e, "policy roll-out kernel");
  if ((st = peer_merge(h, T))) return st;
  h->t += (uint64_t)T;
  h->cursor = T;
  h->sampled_slot = -1;
  return WS_OK;
}

ws_status ws_rollout_policy(ws_env* h, int32_t T, const float* weights, int32_t hidden) {
  return run_policy(h, T, weights, hidden, nullptr, nullptr);
}

ws_status ws_rollout_actor_critic(ws_env* h, int32_t T, const float* params, int32_t hidden, float* values,
                                  float* bootstrap, float* values_trunc) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (!values || !bootstrap) return fail(h, WS_ERR_INVALID_ARGUMENT, "values and bootstrap are required");
  if (values_trunc && h->spec.kind == ws::kUser)
    return fail(h, WS_ERR_INVALID_ARGUMENT, "values_trunc: built-in envs only");
  return run_policy(h, T, params, hidden, values, bootstrap, values_trunc);
}

static ws_status run_gae(ws_env* h, const ws_gae_args* a, cudaStream_t s, const ws::Launch* l) {
  if (!a || a->T < 1 || a->n_envs < 1 || a->n_agents < 1 || !a->rew || !a->done || !a->values || !a->bootstrap ||
      !a->adv || !a->ret || !(a->gamma >= 0.0f && a->gamma <= 1.0f) || !(a->lambda >= 0.0f && a->lambda <= 1.0f))
    return fail(h, WS_ERR_INVALID_ARGUMENT, "ws_gae: T, E, A >= 1, non-NULL arrays, gamma and lambda in [0, 1]");
  ws::GaeArgs g{a->rew, a->done, a->values, a->bootstrap, a->v_trunc, a->adv, a->ret, a->n_envs, a->n_agents,
                a->T, a->gamma, a->lambda, 0};
  uint64_t launches = 0;
  if (l) l->m(ws::kKGae, 0);
  cudaError_t e = ws::launch_gae(g, s, h ? &h->launches : &launches);
  if (l) l->m(ws::kKGae, 1);
  if (e) return cuda_fail(h, e, "gae kernel");
  return WS_OK;
}

ws_status ws_gae(const ws_gae_args* args, void* stream) {
  return run_gae(nullptr, args, static_cast<cudaStream_t>(stream), nullptr);
}

ws_status ws_gae_store(ws_env* h, int32_t T, const float* values, const float* bootstrap, const float* v_trunc,
                       float gamma, float lambda, float* adv, float* ret) {
  NvtxRange nvtx_("ws_gae_store");
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (T < 1) return fail(h, WS_ERR_INVALID_ARGUMENT, "T must be >= 1");
  if (!h->rew) return fail(h, WS_ERR_BAD_STATE, "ws_gae_store needs the store (t_capacity or a first ws_rollout)");
  if (T > h->T_cap) return fail(h, WS_ERR_OUT_OF_RANGE, "T exceeds the store capacity");
  DeviceGuard g(h->device);
  ws_gae_args a{T, h->A, h->E, h->rew, h->done, values, bootstrap, v_trunc, gamma, lambda, adv, ret};
  const ws::Launch l = launch_of(h);
  return run_gae(h, &a, h->stream, &l);
}

ws_status ws_rollout_host(ws_env* h, int32_t T, const float* host_probs, int64_t n_probs, int64_t row_stride,
                          int64_t step_stride, ws_stats* out) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (!host_probs || n_probs < 1 || !out) return fail(h, WS_ERR_INVALID_ARGUMENT, "host_probs / n_probs / out");
  DeviceGuard g(h->device);
  cudaError_t e;
  if (h->staging_n < n_probs) {
    if (h->staging) return fail(h, WS_ERR_INVALID_ARGUMENT, "n_probs grew beyond the first call's staging size");
    h->staging = (float*)dev_alloc(h, (size_t)n_probs * sizeof(float), &e);
    if (e) return cuda_fail(h, e, "alloc staging");
    h->staging_n = n_probs;
  }
  if ((e = cudaMemcpyAsync(h->staging, host_probs, (size_t)n_probs * sizeof(float), cudaMemcpyHostToDevice, h->stream)))
    return cuda_fail(h, e, "H2D probs");
  ws_status s = ws_rollout(h, T, h->staging, row_stride, step_stride);
  if (s) return s;
  if ((int)h->host_stats.size() < 4 * T) h->host_stats.resize(4 * (size_t)T);
  if ((e = cudaMemcpyAsync(h->host_stats.data(), h->stats, (size_t)T * 4 * sizeof(long long), cudaMemcpyDeviceToHost,
                           h->stream)))
    return cuda_fail(h, e, "D2H stats");
  if ((e = cudaStreamSynchronize(h->stream))) return cuda_fail(h, e, "sync");
  sum_stats(h->host_stats.data(), T, out);
  return WS_OK;
}

ws_status ws_rollout_host_submit(ws_env* h, int32_t T, const float* host_probs, int64_t n_probs, int64_t row_stride,
                                 int64_t step_stride, int32_t slot) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (!host_probs || n_probs < 1 || slot < 0 || slot > 1)
    return fail(h, WS_ERR_INVALID_ARGUMENT, "host_probs / n_probs / slot (0 or 1)");
  ws_env::HostSlot& hs = h->hslot[slot];
  if (hs.pending) return fail(h, WS_ERR_BAD_STATE, "slot has a submission that was not waited for");
  DeviceGuard g(h->device);
  cudaError_t e;
  if (!h->copy_stream) {
    if ((e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking))) return cuda_fail(h, e, "copy stream");
    for (auto& x : h->hslot)
      if ((e = cudaEventCreateWithFlags(&x.copied, cudaEventDisableTiming)) ||
          (e = cudaEventCreateWithFlags(&x.consumed, cudaEventDisableTiming)) ||
          (e = cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming)))
        return cuda_fail(h, e, "pipeline events");
  }
  if (h->hslot_n < n_probs) {
    if (h->hslot_n) return fail(h, WS_ERR_INVALID_ARGUMENT, "n_probs grew beyond the first submission's size");
    for (auto& x : h->hslot) {
      x.staging = (float*)dev_alloc(h, (size_t)n_probs * sizeof(float), &e);
      if (e) return cuda_fail(h, e, "alloc staging");
    }
    h->hslot_n = n_probs;
  }
  // H2D of this slot's probabilities on the copy stream, after the roll-out that last read the
  // slot's staging buffer (two submissions ago) -- it overlaps the roll-out now running
  if (hs.used && (e = cudaStreamWaitEvent(h->copy_stream, hs.consumed, 0))) return cuda_fail(h, e, "wait consumed");
  if ((e = cudaMemcpyAsync(hs.staging, host_probs, (size_t)n_probs * sizeof(float), cudaMemcpyHostToDevice,
                           h->copy_stream)) ||
      (e = cudaEventRecord(hs.copied, h->copy_stream)) || (e = cudaStreamWaitEvent(h->stream, hs.copied, 0)))
    return cuda_fail(h, e, "H2D probs");
  ws_status s = ws_rollout(h, T, hs.staging, row_stride, step_stride);
  if (s) return s;
  if ((e = cudaEventRecord(hs.consumed, h->stream))) return cuda_fail(h, e, "record consumed");
  hs.used = true;
  if (!hs.st && (e = cudaMallocHost(&hs.st, (size_t)h->T_cap * 4 * sizeof(long long)))) {
    hs.st = nullptr;
    return cuda_fail(h, e, "alloc pinned result slot");
  }
  if ((e = cudaMemcpyAsync(hs.st, h->stats, (size_t)T * 4 * sizeof(long long), cudaMemcpyDeviceToHost, h->stream)) ||
      (e = cudaEventRecord(hs.done, h->stream)))
    return cuda_fail(h, e, "D2H stats");
  hs.T = T;
  hs.pending = true;
  return WS_OK;
}

ws_status ws_rollout_host_wait(ws_env* h, int32_t slot, ws_stats* out) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (slot < 0 || slot > 1 || !out) return fail(h, WS_ERR_INVALID_ARGUMENT, "slot (0 or 1) / out");
  ws_env::HostSlot& hs = h->hslot[slot];
  if (!hs.pending) return fail(h, WS_ERR_BAD_STATE, "no submission in this slot");
  DeviceGuard g(h->device);
  cudaError_t e = cudaEventSynchronize(hs.done);
  hs.pending = false;
  if (e) return cuda_fail(h, e, "wait");
  sum_stats(hs.st, hs.T, out);
  return WS_OK;
}

ws_status ws_rollout_staged(ws_env* h, int32_t T, const float* host_probs, int64_t n_probs, int64_t row_stride,
                            int64_t step_stride, const ws_host_store* dst, ws_staged_report* out) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (h->dev_clock)
    return fail(h, WS_ERR_BAD_STATE, "device clock on (ws_enable_device_clock): fused roll-outs take the host step index");
  if (T < 1) return fail(h, WS_ERR_INVALID_ARGUMENT, "T must be >= 1");
  if (!host_probs || n_probs < 1 || row_stride < 0 || step_stride < 0 || !dst)
    return fail(h, WS_ERR_INVALID_ARGUMENT, "host_probs / n_probs / strides / dst");
  DeviceGuard g(h->device);
  ws_status st = ensure_store(h, T);
  if (st) return st;
  if (T > h->T_cap) return fail(h, WS_ERR_OUT_OF_RANGE, "T exceeds the store capacity");
  cudaError_t e = cudaSuccess;
  if (h->staging_n < n_probs) {
    if (h->staging) return fail(h, WS_ERR_INVALID_ARGUMENT, "n_probs grew beyond the first call's staging size");
    h->staging = (float*)dev_alloc(h, (size_t)n_probs * sizeof(float), &e);
    if (e) return cuda_fail(h, e, "alloc staging");
    h->staging_n = n_probs;
  }
  const size_t EA = (size_t)h->E * h->A;
  const size_t act_w = h->spec.n_actions ? 1 : (size_t)h->spec.act_dim;
  struct Part { void* host; const void* dev; size_t bytes; };
  const Part parts[5] = {
      {dst->obs, h->obs, EA * h->spec.obs_dim * sizeof(float)},
      {dst->act, h->act, EA * act_w * 4},
      {dst->logp, h->logp, h->logp ? EA * sizeof(float) : 0},
      {dst->rew, h->rew, EA * sizeof(float)},
      {dst->done, h->done, (size_t)h->E},
  };
  cudaEvent_t ev[4];
  for (int i = 0; i < 4; ++i)
    if ((e = cudaEventCreate(&ev[i]))) return cuda_fail(h, e, "event");
  cudaEvent_t first = nullptr;
  if ((e = cudaEventCreate(&first))) return cuda_fail(h, e, "event");
  double transfer = 0.0, h2d = 0.0, d2h = 0.0;
  h->cursor = 0;
  h->sampled_slot = -1;
  for (int32_t t = 0; t < T && !e && st == WS_OK; ++t) {
    const size_t n = (size_t)n_probs;  // the floats the trainer sends for this step
    cudaEventRecord(ev[0], h->stream);
    if (t == 0) cudaEventRecord(first, h->stream);
    e = cudaMemcpyAsync(h->staging, host_probs + (size_t)t * step_stride, n * sizeof(float), cudaMemcpyHostToDevice,
                        h->stream);
    if (e) break;
    h2d += (double)(n * sizeof(float));
    cudaEventRecord(ev[1], h->stream);
    st = ws_sample(h, h->staging, row_stride);
    if (st) break;
    st = ws_step(h, nullptr);
    if (st) break;
    cudaEventRecord(ev[2], h->stream);
    for (const Part& p : parts) {
      if (!p.host || !p.bytes) continue;
      e = cudaMemcpyAsync(static_cast<char*>(p.host) + (size_t)t * p.bytes,
                          static_cast<const char*>(p.dev) + (size_t)t * p.bytes, p.bytes, cudaMemcpyDeviceToHost,
                          h->stream);
      if (e) break;
      d2h += (double)p.bytes;
    }
    if (e) break;
    cudaEventRecord(ev[3], h->stream);
    if ((e = cudaEventSynchronize(ev[3]))) break;  // the trainer waits for step t
    float a = 0.0f, b = 0.0f;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[2], ev[3]);
    transfer += (double)a + (double)b;
  }
  float total = 0.0f;
  if (!e && st == WS_OK) cudaEventElapsedTime(&total, first, ev[3]);
  for (int i = 0; i < 4; ++i) cudaEventDestroy(ev[i]);
  cudaEventDestroy(first);
  if (st) return st;
  if (e) return cuda_fail(h, e, "staged roll-out copy");
  if ((st = peer_merge(h, T))) return st;
  if (out) {
    out->total_ms = total;
    out->transfer_ms = transfer;
    out->h2d_bytes = h2d;
    out->d2h_bytes = d2h;
  }
  return WS_OK;
}

static ws_tensor tensor(void* p, ws_dtype dt, std::initializer_list<int64_t> shape) {
  ws_tensor t{};
  t.ptr = p;
  t.dtype = dt;
  t.ndim = (int32_t)shape.size();
  int i = 0;
  for (int64_t s : shape) t.shape[i++] = s;
  return t;
}

ws_status ws_get_buffers(const ws_env* h, ws_buffers* out) {
  if (!h || !out) return WS_ERR_INVALID_ARGUMENT;
  const int64_t T = h->T_cap, E = h->E, A = h->A, D = h->spec.obs_dim;
  std::memset(out, 0, sizeof(*out));
  out->obs = tensor(h->obs, WS_F32, {T, E, A, D});
  if (h->spec.n_actions) out->act = tensor(h->act, WS_I32, {T, E, A});
  else out->act = tensor(h->act, WS_F32, {T, E, A, h->spec.act_dim});
  out->logp = tensor(h->logp, WS_F32, {T, E, A});
  out->rew = tensor(h->rew, WS_F32, {T, E, A});
  out->done = tensor(h->done, WS_U8, {T, E});
  out->stats = tensor(h->stats, WS_I64, {T, 4});
  if (h->spec.kind == ws::kTag) out->state = tensor(h->tstate, WS_I32, {E, A, 3});
  else out->state = tensor(h->state, WS_F32, {E, h->spec.state_dim});
  out->obs_live = tensor(h->obs_live, WS_F32, {E, A, D});
  out->ep_step = tensor(h->ep_step, WS_I32, {E});
  out->reset_count = tensor(h->reset_count, WS_U32, {E});
  out->ep_ret = tensor(h->ep_ret, WS_F32, {E, A});
  return WS_OK;
}

ws_status ws_get_info(const ws_env* h, ws_info* out) {
  if (!h || !out) return WS_ERR_INVALID_ARGUMENT;
  std::memset(out, 0, sizeof(*out));
  out->obs_dim = h->spec.obs_dim;
  out->n_actions = h->spec.n_actions;
  out->act_dim = h->spec.act_dim;
  out->state_dim = h->spec.state_dim;
  out->max_steps = h->max_steps;
  out->n_agents = h->A;
  out->t_capacity = h->T_cap;
  out->cursor = h->cursor;
  out->n_envs = h->E;
  out->env_offset = h->offset;
  out->n_envs_global = h->E_global;
  out->t = h->t;
  if (h->dev_clock) {  // the device clock is authoritative
    DeviceGuard g(h->device);
    uint64_t t = 0;
    if (cudaMemcpyAsync(&t, h->t_dev, sizeof(t), cudaMemcpyDeviceToHost, h->stream) == cudaSuccess &&
        cudaStreamSynchronize(h->stream) == cudaSuccess)
      out->t = t;
  }
  out->launches = h->launches;
  out->probs_width = h->spec.n_actions ? h->spec.n_actions : 2 * h->spec.act_dim;
  return WS_OK;
}

ws_status ws_synchronize(ws_env* h) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e) return cuda_fail(h, e, "ws_synchronize");
  uint32_t word = 0;
  if ((e = cudaMemcpy(&word, h->err, sizeof(word), cudaMemcpyDeviceToHost))) return cuda_fail(h, e, "read error word");
  if (word & ws::kErrPeer) return fail(h, WS_ERR_PEER, "cross-GPU statistics reduction timed out waiting for a peer");
  if (word & ws::kErrProbs) return fail(h, WS_ERR_INVALID_PROBS, "a probability row was invalid (sticky until ws_reset)");
  if (word & ws::kErrAction) return fail(h, WS_ERR_INVALID_ACTION, "an action was invalid (sticky until ws_reset)");
  return WS_OK;
}

ws_status ws_read_stats(ws_env* h, int32_t t0, int32_t t1, ws_stats* out) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  if (!out || t0 < 0 || t1 < t0 || t1 > h->T_cap) return fail(h, WS_ERR_INVALID_ARGUMENT, "bad slot range");
  DeviceGuard g(h->device);
  std::vector<long long> st(4 * (size_t)(t1 - t0) + 4);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (!e && t1 > t0)
    e = cudaMemcpy(st.data(), h->stats + 4 * (size_t)t0, 4 * sizeof(long long) * (t1 - t0), cudaMemcpyDeviceToHost);
  if (e) return cuda_fail(h, e, "ws_read_stats");
  sum_stats(st.data(), t1 - t0, out);
  return WS_OK;
}

ws_status ws_test_philox(const uint32_t* rows, int64_t n, uint32_t* out, void* stream) {
  if (!rows || !out || n < 0) return WS_ERR_INVALID_ARGUMENT;
  if (n == 0) return WS_OK;
  cudaError_t e = ws::launch_test_philox(rows, n, out, (cudaStream_t)stream);
  if (!e) e = cudaStreamSynchronize((cudaStream_t)stream);
  return e ? WS_ERR_CUDA : WS_OK;
}

ws_status ws_test_sample_grid(const float* p, int32_t n, int64_t* counts, void* stream) {
  if (!p || !counts || n < 1 || n > 8) return WS_ERR_INVALID_ARGUMENT;
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)(n + 1) * sizeof(int64_t), (cudaStream_t)stream);
  if (!e) e = ws::launch_test_sample_grid(p, n, counts, (cudaStream_t)stream);
  if (!e) e = cudaStreamSynchronize((cudaStream_t)stream);
  return e ? WS_ERR_CUDA : WS_OK;
}

ws_status ws_test_unary(int32_t fn, float param, const float* x, int64_t n, float* out, void* stream) {
  if (!x || !out || n < 0 || fn < 0 || fn > 8) return WS_ERR_INVALID_ARGUMENT;
  if (n == 0) return WS_OK;
  cudaError_t e = ws::launch_test_unary(fn, param, x, n, out, (cudaStream_t)stream);
  if (!e) e = cudaStreamSynchronize((cudaStream_t)stream);
  return e ? WS_ERR_CUDA : WS_OK;
}

ws_status ws_test_surface_energy(const float* q, int32_t D, int64_t n, float* energy, double* spring, void* stream) {
  if (!q || !energy || !spring || n < 0) return WS_ERR_INVALID_ARGUMENT;
  if (D != 2 && D != 3 && D != 4 && D != 8 && D != 16 && D != 20 && D != 32) return WS_ERR_INVALID_ARGUMENT;
  if (n == 0) return WS_OK;
  cudaError_t e = ws::launch_test_surface_energy(q, D, n, energy, spring, (cudaStream_t)stream);
  if (!e) e = cudaStreamSynchronize((cudaStream_t)stream);
  return e ? WS_ERR_CUDA : WS_OK;
}

ws_status ws_test_exhaustive(int32_t fn_a, int32_t fn_b, float param, uint32_t lo_bits, uint32_t hi_bits,
                             uint64_t* mismatches, void* stream) {
  if (!mismatches || fn_a < 0 || fn_a > 8 || fn_b < 0 || fn_b > 8 || hi_bits < lo_bits) return WS_ERR_INVALID_ARGUMENT;
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(*d));
  if (!e) e = cudaMemsetAsync(d, 0, sizeof(*d), (cudaStream_t)stream);
  if (!e) e = ws::launch_test_exhaustive(fn_a, fn_b, param, lo_bits, hi_bits, d, (cudaStream_t)stream);
  unsigned long long h = 0;
  if (!e) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (!e) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (d) cudaFree(d);
  *mismatches = h;
  return e ? WS_ERR_CUDA : WS_OK;
}

static const char* kKernelNames[ws::kKCount] = {"plan", "rollout", "sample", "step", "reset", "gae"};

ws_status ws_peer_export(ws_env* h, int32_t world, ws_ipc_handle* out) {
  if (check(h) || !out || world < 1 || world > ws::kMaxPeers)
    return fail(h, WS_ERR_INVALID_ARGUMENT, "ws_peer_export: world must be in [1, 8]");
  if (h->T_cap < 1) return fail(h, WS_ERR_BAD_STATE, "ws_peer_export needs the store (t_capacity or a first ws_rollout)");
  DeviceGuard g(h->device);
  cudaStreamSynchronize(h->stream);
  peer_release(h);
  const size_t words = 2 * (size_t)world * (size_t)h->T_cap * 4 + 4;  // + arrival counter (32-byte pad)
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&h->peer_own), words * sizeof(unsigned long long));
  if (!e) e = cudaMemset(h->peer_own, 0, words * sizeof(unsigned long long));
  cudaIpcMemHandle_t ih;
  if (!e) e = cudaIpcGetMemHandle(&ih, h->peer_own);
  if (e) {
    peer_release(h);
    return cuda_fail(h, e, "ws_peer_export");
  }
  static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(ws_ipc_handle), "IPC handle size");
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out->bytes, &ih, sizeof(ih));
  h->peer_world = world;
  h->peer_tcap = h->T_cap;
  return WS_OK;
}

ws_status ws_peer_attach(ws_env* h, int32_t rank, int32_t world, const ws_ipc_handle* handles) {
  if (check(h) || !handles || world != h->peer_world || rank < 0 || rank >= world || !h->peer_own)
    return fail(h, WS_ERR_INVALID_ARGUMENT, "ws_peer_attach: call ws_peer_export(world) first; 0 <= rank < world");
  DeviceGuard g(h->device);
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, handles[r].bytes, sizeof(ih));
    const cudaError_t e = cudaIpcOpenMemHandle(&h->peer_open[r], ih, cudaIpcMemLazyEnablePeerAccess);
    if (e) {
      peer_release(h);
      return cuda_fail(h, e, "ws_peer_attach: cudaIpcOpenMemHandle");
    }
  }
  h->peer_rank = rank;
  h->peer_epoch = 0;
  h->peer_attached = world > 1;
  return WS_OK;
}

ws_status ws_peer_detach(ws_env* h) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  cudaStreamSynchronize(h->stream);
  peer_release(h);
  return WS_OK;
}

ws_status ws_enable_kernel_timing(ws_env* h, int32_t enable) {
  if (check(h)) return WS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  if ((enable & 0xFF) && h->rings[0].b.empty()) {
    for (auto& r : h->rings) {
      r.b.resize(kTimingCap);
      r.e.resize(kTimingCap);
      for (int i = 0; i < kTimingCap; ++i) {
        cudaError_t e = cudaEventCreate(&r.b[i]);
        if (!e) e = cudaEventCreate(&r.e[i]);
        if (e) return cuda_fail(h, e, "cudaEventCreate");
      }
    }
  }
  for (auto& r : h->rings) {
    r.n = 0;
    r.calls = 0;
    r.skip = false;
  }
  const int mode = enable & 0xFF, period = (enable >> 8) & 0xFF;
  h->timing = mode != 0;
  h->timing_period = period > 1 ? period : 1;
  h->timed_mask = mode == 2   ? (1u << ws::kKRollout)
                 : mode == 3 ? (1u << ws::kKRollout) | (1u << ws::kKGae)
                             : 0xFFFFFFFFu;
  return WS_OK;
}

ws_status ws_kernel_times(ws_env* h, ws_kernel_time* out, int32_t capacity, int32_t* n_out) {
  if (check(h) || !out || !n_out || capacity < ws::kKCount) return WS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e) return cuda_fail(h, e, "ws_kernel_times");
  for (int k = 0; k < ws::kKCount; ++k) {
    ws_env::Ring& r = h->rings[k];
    const int n = std::min(r.n, kTimingCap);
    float tot = 0.0f;
    for (int i = 0; i < n && h->timing; ++i) {
      float ms = 0.0f;
      if (cudaEventElapsedTime(&ms, r.b[i], r.e[i]) == cudaSuccess) tot += ms;
    }
    out[k].name = kKernelNames[k];
    out[k].launches = n;
    out[k].total_ms = tot;
    out[k].mean_ms = n ? tot / (float)n : 0.0f;
    r.n = 0;
  }
  *n_out = ws::kKCount;
  return WS_OK;
}

}  // extern "C"
