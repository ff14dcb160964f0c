// kernels.h -- internal (C++) interface between the host runtime (runtime.cu) and the
// device kernels (kernels.cu).  Not part of the C ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ws {

enum EnvKind : int { kCartPole = 0, kAcrobot = 1, kPendulum = 2, kTag = 3, kSurface = 4, kDummy = 5, kUser = 6 };

// Everything a kernel needs to find the handle's buffers (passed by value).
struct KArgs {
  // roll-out store (time-major)
  float* obs;
  void* act;
  float* logp;
  float* rew;
  uint8_t* done;
  unsigned long long* stats;  // [T_cap, 4] fixed-point int64 (common.cuh StatField)
  // live state
  float* state;       // [E, S]
  int32_t* tstate;    // tag: [E, A, 3]
  float* obs_live;    // [E, A, D]
  int32_t* ep_step;   // [E]
  uint32_t* reset_count;  // [E]
  float* ep_ret;      // [E, A]
  uint32_t* err;      // sticky device error word
  uint32_t* plan;     // discrete lane envs: [ceil(T_cap / 4), E] packed 8-bit actions
  int64_t E;          // replicas on this device
  int64_t offset;     // global index of replica 0
  int32_t A;
  int32_t T_cap;
  int32_t max_steps;
  int32_t write_logp;
  int32_t p0, p1;     // env params (tag G / taggers; surface D)
  uint32_t k0, k1;    // Philox key
  // device step counter (ws_enable_device_clock) or null: the single-step sampler reads its
  // ACTION draw index t from here and every single step advances it, so captured CUDA graphs of
  // sample / step sequences replay with fresh draws (NEXT-N1 policy graphs)
  uint64_t* t_dev;
};

// kernel classes for the optional per-kernel timing (ws_enable_kernel_timing)
enum KernelId : int { kKPlan = 0, kKRollout = 1, kKSample = 2, kKStep = 3, kKReset = 4, kKGae = 5, kKCount = 6 };

struct Launch {
  EnvKind kind;
  int block;          // lane-kernel block size
  cudaStream_t stream;
  void (*mark)(void* ctx, int kernel, int phase) = nullptr;  // CUDA-event bracketing hook
  void* mark_ctx = nullptr;
  void m(int kernel, int phase) const {
    if (mark) mark(mark_ctx, kernel, phase);
  }
};

// all return the cudaGetLastError() after the launch(es) and add to *launches
cudaError_t launch_reset(const KArgs& a, const Launch& l, uint64_t* launches);
cudaError_t launch_rollout(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* probs,
                           int64_t row_stride, int64_t step_stride, uint64_t* launches);
cudaError_t launch_plan(const KArgs& a, int n_actions, int T, uint64_t t0, const float* probs, int64_t row_stride,
                        cudaStream_t s);
cudaError_t launch_sample(const KArgs& a, const Launch& l, int slot, uint64_t t, const float* probs,
                          int64_t row_stride, uint64_t* launches);
cudaError_t launch_step(const KArgs& a, const Launch& l, int slot, const void* given, uint64_t* launches);
cudaError_t launch_test_philox(const uint32_t* rows, int64_t n, uint32_t* out, cudaStream_t s);
cudaError_t launch_test_sample_grid(const float* p, int n, int64_t* counts, cudaStream_t s);
cudaError_t launch_test_unary(int fn, float p, const float* x, int64_t n, float* out, cudaStream_t s);
cudaError_t launch_test_surface_energy(const float* q, int D, int64_t n, float* energy, double* spring,
                                      cudaStream_t s);
cudaError_t launch_test_exhaustive(int fa, int fb, float p, uint32_t lo, uint32_t hi, unsigned long long* mism,
                                   cudaStream_t s);

// NEXT-N1: fused roll-out with in-kernel MLP policy inference (hidden 32 or 64)
// values / bootstrap non-null: the weights carry the R31 value head and the kernel also writes
// the critic's values [T, E] and bootstrap [E] (NEXT-N2)
cudaError_t launch_rollout_policy(const KArgs& a, const Launch& l, int T, uint64_t t0, const float* weights,
                                  int hidden, uint64_t* launches, float* values = nullptr,
                                  float* bootstrap = nullptr, float* values_trunc = nullptr);

// NEXT-N2: generalised advantage estimation over the time-major store (gae.cu, R30)
struct GaeArgs {
  const float* rew;        // [T, E, A]
  const uint8_t* done;     // [T, E]
  const float* values;     // [T, E, A]
  const float* bootstrap;  // [E, A]
  const float* v_trunc;    // [T, E, A] or null
  float* adv;              // [T, E, A]
  float* ret;              // [T, E, A]
  int64_t E;
  int32_t A, T;
  float gamma, lambda;
  int force_lane;          // 1 = per-thread-load kernel regardless of alignment (tests)
};
// 0 = per-thread loads, 1 = TMA tiles for r / v (done per thread), 2 = TMA tiles for r / v / done
int gae_path(int64_t E, int32_t A, const void* rew, const void* values, const void* done);
cudaError_t launch_gae(const GaeArgs& a, cudaStream_t s, uint64_t* launches);

// A8 across GPUs without NCCL (section 8e "v2"): every rank publishes its [T,4] statistics
// into every peer's gather buffer through CUDA-IPC-mapped peer memory (NVLink / NVSwitch),
// signals the peers' arrival counters, waits for all ranks and sums the slices.
constexpr int kMaxPeers = 8;
struct PeerArgs {
  unsigned long long* gather[kMaxPeers];  // each rank's buffer [2][world][t_cap][4] + counter
  int rank, world, t_cap;
};
cudaError_t launch_peer_allreduce(const unsigned long long* local, int T, const PeerArgs& p, uint64_t epoch,
                                  unsigned long long* out, uint32_t* err, double timeout_s, cudaStream_t s);

// NEXT-N4: environments registered at run time (composer.cu, ws_register_env)
struct UserSpec {
  void* handle;  // registry entry
  int obs_dim, n_actions, state_dim, max_steps, n_params;
  int act_dim;  // 0: discrete; > 0: continuous (n_actions 0)
};
struct UserLaunch {
  KArgs k;
  void* handle;
  const float* prm;     // [E, n_params] per-replica parameters or null
  const float* shared;  // shared read-only data or null
  cudaStream_t stream;
};
bool user_env_spec(const char* name, UserSpec* out);
cudaError_t launch_user_reset(const UserLaunch& l);
cudaError_t launch_user_rollout(const UserLaunch& l, int T, uint64_t t0, const float* probs, int64_t row_stride,
                                int64_t step_stride);
// the R29 policy (hidden 32 / 64) inside the registered env's loop; values / bootstrap
// non-null: also the R31 critic
cudaError_t launch_user_policy(const UserLaunch& l, int T, uint64_t t0, const float* weights, int hidden,
                               float* values, float* bootstrap);

}  // namespace ws
