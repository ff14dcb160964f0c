"""bench.py -- env-steps/s of the fused roll-out step on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {ours,reference}] [--workload C2]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

One "step" = one ws_rollout over the whole workload: T fused env steps of every replica
(sample -> log -> dynamics -> reward/done -> auto-reset -> in-place store), the per-slot
statistics reduction, and (N > 1) the NCCL all-reduce of those statistics -- every row of
SURVEY 8(a).  Workload C2 (BASELINE.json configs[1]): CartPole-v1, 10K replicas x 1000
steps per GPU (weak scaling: every rank runs its own 10K-replica shard of a global
N*10K batch), uniform 2-action probabilities resident in HBM.

Prints ONE JSON line (rank 0).  See DESIGN.md section 6 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import wsinputs as W  # noqa: E402

# Algorithmic store bytes written per env-step, split by the kernel
# that writes them: the roll-out kernel writes obs (D_obs*4) + rew (4) + done (1); the plan
# kernel writes act (4) + logp (4).  Per agent; done is per replica.
OBS_DIM = {"cartpole": 4, "acrobot": 6, "dummy": 4, "pendulum": 3, "tag": 4, "surface": 21}
# NEXT-N4 registered env (k_user_rollout samples in-loop: it writes obs + act + logp + rew + done)
USER_BYTES = {"u_cartpole": 4 * 4 + 4 + 4 + 4 + 1}


def register_user(w, oracle_side: bool):
    """Register a NEXT-N4 workload's C-source env (product: NVRTC; oracle: g++)."""
    name = w.params.get("user")
    if not name:
        return
    import wsinputs.user_envs as U
    src, dims = U.ENVS[name]
    if oracle_side:
        import oracle as O
        O.register_user_env(name, src, **dims)
    else:
        from paper_2408_00930_b200 import register_env
        register_env(name, src, **dims)
# algorithmic bytes per env-step: the roll-out kernel writes obs + rew + done
# and reads its actions (discrete: the packed plan, 1 byte; continuous: the act slab, 4 d);
# the plan kernel writes act + logp (+ the packed plan for discrete envs)
ACT_DIM = {"pendulum": 1, "surface": 20}
ROLLOUT_BYTES = {k: 4 * d + 4 + 1 + (4 * ACT_DIM[k] if k in ACT_DIM else 0.25) for k, d in OBS_DIM.items()}
PLAN_BYTES = {k: (4 * ACT_DIM[k] + 4 if k in ACT_DIM else 8.25) for k in OBS_DIM}
KERNEL_NAME = {"cartpole": "k_rollout_discrete<CartPole>", "acrobot": "k_rollout_discrete<Acrobot>",
               "dummy": "k_rollout_discrete<Dummy>", "pendulum": "k_rollout_continuous<Pendulum>",
               "surface": "k_rollout_surface_seg<20>", "tag": "k_tag"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--csv", default=None, help="also append one row to this CSV (SURVEY 5 bench CSV)")
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ncu", action="store_true", help="profiling mode: no clocks / cpu baseline / e2e")
    ap.add_argument("--dist-backend", default="nccl", help="process-group backend for N > 1 (gloo only for tests)")
    ap.add_argument("--stats-reduce", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: statistics all-reduce by libws's peer-memory kernel (default) or NCCL")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="diagnostic: no per-kernel CUDA events in the timed region (roofline unavailable)")
    ap.add_argument("--same-device", action="store_true", help="all ranks on cuda:0 (multi-rank test on one GPU)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


_GAE_INPUTS = {}


def oracle_gae_inputs(w):
    """Given GAE inputs of a NEXT-N2 workload (generated once, outside any timing)."""
    if w.name not in _GAE_INPUTS:
        _GAE_INPUTS[w.name] = W.gae_inputs(w.T, w.n_envs, w.n_agents)
    return _GAE_INPUTS[w.name]


def oracle_rollout(b, w, T, probs, cores):
    """One oracle roll-out of workload w (policy-driven for NEXT-N1 workloads; followed by
    GAE over the slots it wrote for NEXT-N2 workloads)."""
    pol = W.workload_policy(w)
    if pol and w.n_actions == 0:  # Gaussian policy (R34): the policy prefix W1..log_std
        D, H, d = OBS_DIM[w.env], pol[0], w.act_dim
        st = b.rollout_policy_gauss(T, pol[1][:D * H + H + H * d + 2 * d], H, n_threads=cores)
    elif pol:
        st = b.rollout_policy(T, pol[1], pol[0], n_threads=cores)
    else:
        st = b.rollout(T, probs, n_threads=cores)
    if w.params.get("a2c") and w.n_actions == 0:  # NEXT-N2 continuous (R35): the oracle's Gaussian update
        import oracle as O
        from oracle import a2c as OA
        H, params = pol
        D, d = OBS_DIM[w.env], w.act_dim
        obs = b.array("obs")[:T].reshape(-1, D)
        _, _, _, _, V = OA.forward_gauss(params, obs, D, H, d)
        boot = OA.forward_gauss(params, b.array("obs_live").reshape(-1, D), D, H, d)[4]
        adv, ret = O.gae(b.array("rew")[:T].reshape(T, w.n_envs), b.array("done")[:T], V.reshape(T, w.n_envs),
                         boot, 0.99, 0.95, f64=True)
        g = OA.grad_gauss(params, obs, b.array("act")[:T].reshape(-1, d), OA.normalize(adv), ret.ravel(), D, H, d,
                          0.5, 0.01)
        z = np.zeros(params.size)
        OA.adam(params, OA.clip(g, 0.5), z, z, 1, 1e-4)
    elif w.params.get("a2c"):  # NEXT-N2: the oracle's A2C update on the slots just written
        import oracle as O
        from oracle import a2c as OA
        H, params = pol
        D = OBS_DIM[w.env]
        N = w.n_actions
        obs = b.array("obs")[:T].reshape(-1, D)
        EA = w.n_envs * w.n_agents  # multi-agent (R36): every agent is a column
        vals = OA.values(params, obs, D, H, N).reshape(T, w.n_envs, w.n_agents)
        boot = OA.values(params, b.array("obs_live").reshape(-1, D), D, H, N).reshape(w.n_envs, w.n_agents)
        adv, ret = O.gae(b.array("rew")[:T].reshape(T, w.n_envs, w.n_agents), b.array("done")[:T], vals, boot,
                         0.99, 0.95, f64=True)
        adv, ret = adv.reshape(T, EA), ret.reshape(T, EA)
        z = np.zeros(params.size)
        act = b.array("act")[:T].reshape(-1)
        ppo = w.params.get("ppo")
        if ppo:  # K epochs x M minibatches of the clipped surrogate (R33), whole-batch normalisation
            Ah, logp_old, p, m, v, k = OA.normalize(adv), b.array("logp")[:T].reshape(-1), params, z, z, 0
            E = EA
            for _ in range(ppo[0]):
                for mb in range(ppo[1]):
                    r0, r1 = T * mb // ppo[1] * E, T * (mb + 1) // ppo[1] * E
                    g = OA.ppo_grad(p, obs[r0:r1], act[r0:r1], Ah[r0:r1], ret.ravel()[r0:r1], logp_old[r0:r1],
                                    D, H, N, 0.5, 0.01, 0.2)
                    k += 1
                    p, m, v = OA.adam(p, OA.clip(g, 0.5), m, v, k, 1e-4)
        else:
            OA.update(params, z, z, 1, obs, act, adv.ravel(), ret.ravel(), D, H, N, lr=1e-4)
    gae = w.params.get("gae")
    if gae:
        import oracle as O
        values, boot, _ = oracle_gae_inputs(w)
        O.gae(b.array("rew")[:T].reshape(T, w.n_envs, w.n_agents), b.array("done")[:T], values[:T], boot,
              gae[0], gae[1])
    return st


def cpu_baseline(w, budget_s: float = 10.0):
    """The oracle as it stands (oracle/, never tuned for this), on this host's cores, on a
    bounded sample of the same workload: consecutive whole-workload roll-outs (the bench's
    steps) until ~budget_s of CPU work, or a prefix of one roll-out if one is longer."""
    import oracle as O
    cores = len(os.sched_getaffinity(0))
    probs = W.workload_probs(w)
    register_user(w, oracle_side=True)
    if w.params.get("gae"):
        oracle_gae_inputs(w)
    b = O.Batch(w.env, w.n_envs, w.n_agents, W.SEED, t_capacity=w.T)
    t0 = time.perf_counter()
    oracle_rollout(b, w, min(10, w.T), probs, cores)
    probe = time.perf_counter() - t0
    T_s = max(10, min(w.T, int(min(10, w.T) * budget_s / max(probe, 1e-6))))
    steps, dt, n = 0, 0.0, 0
    t0 = time.perf_counter()
    while True:
        oracle_rollout(b, w, T_s, probs, cores)
        steps += w.n_envs * T_s
        n += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s or n >= 1000:
            break
    return {"value": steps / dt, "unit": "env-steps/s", "cores": cores, "kind": "oracle",
            "sample": f"{w.name} {w.env}: {n} x ({w.n_envs} replicas x {T_s} steps) = {steps} env-steps "
                      f"in {dt:.1f} s on {cores} threads"}


def run_reference(args, w):
    world, rank, local = dist_env()
    if rank != 0:
        return
    import oracle as O
    cores = len(os.sched_getaffinity(0))
    probs = W.workload_probs(w)
    register_user(w, oracle_side=True)
    if w.params.get("gae"):
        oracle_gae_inputs(w)
    # each step = the workload's full roll-out (all replicas x T steps) unless one roll-out
    # would take more than ~5 s on this host, then a prefix of T_s steps
    b0 = O.Batch(w.env, w.n_envs, w.n_agents, W.SEED, t_capacity=min(10, w.T))
    t0 = time.perf_counter()
    oracle_rollout(b0, w, min(10, w.T), probs, cores)
    per_step = (time.perf_counter() - t0) / min(10, w.T)
    T_s = max(1, min(w.T, int(5.0 / max(per_step, 1e-9))))
    b = O.Batch(w.env, w.n_envs, w.n_agents, W.SEED, t_capacity=T_s)
    for _ in range(args.warmup):
        oracle_rollout(b, w, T_s, probs, cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle_rollout(b, w, T_s, probs, cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = w.n_envs * T_s * args.steps / tot
    line = {"metric": "env-steps/s", "value": value, "unit": "env-steps/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{w.name}: {w.note}", "env": w.env, "n_envs": w.n_envs, "T": w.T,
                       "sample_T_per_step": T_s, "device": f"host CPU, {cores} threads (oracle/)"},
            "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": cores, "kind": "oracle",
                             "sample": f"{w.n_envs} replicas x {T_s} steps per step"},
            "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def write_csv_row(path, w, world, E_g, A, T, line):
    """SURVEY 5 bench CSV: env,E,A,T,gpus,env_steps_per_s,agent_steps_per_s,kernel,achieved,unit,
    roofline_frac,oracle_steps_per_s,oracle_cores (header written for a new file)."""
    import csv
    r = line["roofline"]
    cb = line.get("cpu_baseline") or {}
    row = [w.env, E_g, A, T, world, line["value"], line["value"] * A, r.get("kernel"), r.get("achieved"),
           r.get("unit"), r.get("frac"), cb.get("value"), cb.get("cores")]
    new = not os.path.exists(path)
    with open(path, "a", newline="") as f:
        wr = csv.writer(f)
        if new:
            wr.writerow(["env", "E", "A", "T", "gpus", "env_steps_per_s", "agent_steps_per_s", "kernel", "achieved",
                         "unit", "roofline_frac", "oracle_steps_per_s", "oracle_cores"])
        wr.writerow(row)


def main():
    args = parse()
    w = W.CONFIGS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)

    import torch
    import torch.distributed as dist

    from paper_2408_00930_b200 import Env
    from paper_2408_00930_b200.parallel import allreduce_stats

    world, rank, local = dist_env()
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    local_dev = 0 if args.same_device else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    # weak scaling: each rank owns a full C2-sized shard of a world*E global batch
    E, A, T = w.n_envs, w.n_agents, w.T
    E_g = E * world
    offset = rank * E
    params = (w.params.get("grid", w.params.get("dim", 0)), w.params.get("taggers", 0))
    stream = torch.cuda.current_stream(dev)
    register_user(w, oracle_side=False)
    env = Env(E, A, w.env, W.SEED, env_offset=offset, n_envs_global=E_g, t_capacity=T,
              param0=params[0], param1=params[1], block_size=args.block)
    probs_host = W.workload_probs(w)
    probs = torch.from_numpy(probs_host).to(dev)
    stats_view = env.buffers()["stats"][:T]
    pol = W.workload_policy(w)  # NEXT-N1 workloads: actions from the in-kernel MLP policy
    pol_w = torch.from_numpy(pol[1]).to(dev) if pol else None
    gae = w.params.get("gae")   # NEXT-N2 workloads: GAE over the store after every roll-out
    if gae:
        g_vals, g_boot, _ = (torch.from_numpy(x).to(dev) if x is not None else None
                             for x in W.gae_inputs(T, E, A, seed=W.SEED + rank))
        g_out = (torch.empty((T, E, A), dtype=torch.float32, device=dev),
                 torch.empty((T, E, A), dtype=torch.float32, device=dev))

    trainer = None
    if w.params.get("a2c"):  # NEXT-N2: every step is one A2C iteration (roll-out + update)
        from paper_2408_00930_b200.a2c import A2C, PPO
        ppo = w.params.get("ppo")
        trainer = (PPO(env, pol[0], params=pol_w, epochs=ppo[0], minibatches=ppo[1], lr=1e-4) if ppo else
                   A2C(env, pol[0], params=pol_w, lr=1e-4, gamma=0.99, lam=0.95, c_v=0.5, c_e=0.01, max_norm=0.5))

    staged = w.params.get("staged")  # NEXT-N3: copy-based baseline pipeline
    staged_rep = {}
    if staged:
        st_probs = torch.from_numpy(probs_host).pin_memory()
        st_dst = env.host_store(T)

    def gpu_rollout(e_obj):
        if staged and e_obj is env:
            staged_rep.update(env.rollout_staged(T, st_probs, st_dst))
        elif trainer is not None and e_obj is env:
            trainer.iteration(T)
        elif pol:
            e_obj.rollout_policy(T, pol_w, pol[0])
        else:
            e_obj.rollout(T, probs)
        if gae:
            e_obj.gae_store(T, g_vals, g_boot, gae[0], gae[1], out=g_out)

    p2p = False
    if world > 1 and args.stats_reduce == "p2p":
        from paper_2408_00930_b200.parallel import attach_peer_stats
        p2p = attach_peer_stats(env)  # falls back to NCCL if CUDA IPC is unavailable on any rank

    def merge_stats():
        if not p2p:
            allreduce_stats(stats_view)

    def one_step():
        gpu_rollout(env)
        merge_stats()

    for _ in range(max(args.warmup, 0)):
        one_step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    if p2p:  # the peer-memory reduction must have worked on every rank, else fall back to NCCL
        ok = torch.tensor([1 if env.status() == 0 else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            print("warning: peer-memory statistics reduction failed during warm-up; using NCCL", file=sys.stderr)
            env.peer_detach()
            env.reset()
            p2p = False
            for _ in range(max(args.warmup, 1)):
                one_step()
            torch.cuda.synchronize(dev)
            dist.barrier()

    clocks = Clocks(local_dev)
    if not args.ncu:
        clocks.start()
        time.sleep(0.3)
    # two CUDA events per step around the fused roll-out kernel only (libws ws_kernel_times):
    # the dominant kernel is timed live with the least perturbation of the timed loop
    env.enable_kernel_timing(0 if (args.no_kernel_timing or staged) else (3 if gae else 2))
    env.kernel_times()
    launches0 = env.info().launches
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ev[0].record(stream)
    for k in range(args.steps):
        gpu_rollout(env)
        merge_stats()
    ev[1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    total_ms = ev[0].elapsed_time(ev[1])
    st = env.status()  # sticky device errors (invalid rows, peer reduction timeout) fail the run
    if st != 0:
        raise RuntimeError(f"libws reported status {st} during the timed region")
    launches = env.info().launches - launches0
    if trainer is not None:  # handle-free kernels per step: moments + final, then (grad + final, Adam) per update
        n_upd = (w.params["ppo"][0] * w.params["ppo"][1]) if w.params.get("ppo") else 1
        launches += (2 + 3 * n_upd) * args.steps
    ktimes = env.kernel_times()
    env.enable_kernel_timing(False)
    clk = clocks.stop() if not args.ncu else {}

    # merged per-slot statistics of the last timed roll-out (all ranks, exact int64; R20)
    from paper_2408_00930_b200.parallel import summarize
    merged = summarize(stats_view.cpu())

    # diagnostic pass after the timed region (not part of `value`): every kernel and the whole
    # ws_rollout call bracketed by events
    n_diag = max(1, min(args.steps, 5))
    env.enable_kernel_timing(1)
    env.kernel_times()
    dev_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n_diag)]
    for k in range(n_diag):
        dev_ev[2 * k].record(stream)
        gpu_rollout(env)
        dev_ev[2 * k + 1].record(stream)
    torch.cuda.synchronize(dev)
    kern_ms = [dev_ev[2 * k].elapsed_time(dev_ev[2 * k + 1]) for k in range(n_diag)]
    diag_times = env.kernel_times()
    env.enable_kernel_timing(False)
    upd_ms = None
    if trainer is not None:  # the update alone (critic, GAE, moments, gradient, Adam)
        for k in range(n_diag):
            dev_ev[2 * k].record(stream)
            trainer.update(T, values_ready=True)
            dev_ev[2 * k + 1].record(stream)
        torch.cuda.synchronize(dev)
        upd_ms = sum(dev_ev[2 * k].elapsed_time(dev_ev[2 * k + 1]) for k in range(n_diag)) / n_diag

    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = E_g * T * args.steps / (max_ms / 1e3)
    ms_per_step = max_ms / args.steps

    # Roofline of the dominant kernel (the fused roll-out kernel), timed live with CUDA
    # events on the handle's stream over the timed region (ws_kernel_times).
    peaks, peak_src = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    n_roll, roll_ms = ktimes.get("rollout", (0, 0.0))
    n_plan, plan_ms = diag_times.get("plan", (0, 0.0))
    # tag samples inside its roll-out kernel: obs 16 + rew 4 + act 4 + logp 4 per agent-step, done 1 per env-step
    roll_bytes = int(ROLLOUT_BYTES.get(w.env, 0) * E * A * T if w.env != "tag" else (16 + 4 + 4 + 4) * E * A * T + E * T)
    if w.env in USER_BYTES:
        roll_bytes = int(USER_BYTES[w.env] * E * A * T)
    if pol:  # the policy kernel also writes act + logp and reads no plan
        roll_bytes = int((4 * OBS_DIM[w.env] + 4 + 1 + 8) * E * A * T)
    achieved = roll_bytes / (roll_ms / 1e3) / 1e9 if roll_ms > 0 else 0.0
    call_ms = sum(kern_ms) / len(kern_ms)
    all_bytes = int(roll_bytes + (PLAN_BYTES.get(w.env, 8) * E * A * T
                                  if w.env not in ("tag",) and w.env not in USER_BYTES and not pol else 0))
    # NEXT-N2: GAE reads rew + values and writes adv + returns (16 B per agent-step), reads
    # the replica's done byte (1 B per replica-step) and the bootstrap row once
    gae_bytes = 16 * E * A * T + E * T + 4 * E * A if gae else 0
    all_bytes += gae_bytes
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None,
                "peak_source": f"{peak_src} hbm_gbs (copy, MEASURED_PEAKS.json)",
                "kernel": KERNEL_NAME.get(w.env, "k_user_rollout (NVRTC, registered env)" if w.env in USER_BYTES
                                          else "k_rollout"),
                "kernel_ms": round(roll_ms, 4), "launches_timed": n_roll,
                "bytes_per_launch": roll_bytes, "bytes_per_env_step": roll_bytes / (E * A * T),
                "other_kernels": {"note": f"diagnostic pass of {n_diag} steps after the timed region",
                                  "plan": {"ms": round(plan_ms, 4), "launches": n_plan,
                                           "achieved_GBps": round(PLAN_BYTES.get(w.env, 8) * E * A * T / (plan_ms / 1e3) / 1e9, 1) if plan_ms else None}},
                "ws_rollout_call": {"ms": round(call_ms, 4), "bytes": all_bytes,
                                    "achieved_GBps": round(all_bytes / (call_ms / 1e3) / 1e9, 1),
                                    "frac": round(all_bytes / (call_ms / 1e3) / 1e9 / peak, 4)}}
    if pol:
        # NEXT-N1: the MLP's fused multiply-adds per replica-step (D x H + H x n), against the
        # fp32 FMA peak from unit counts and clock: 148 SMs x 128 lanes x 2 flop x 1.965 GHz
        D_obs, Hh = OBS_DIM[w.env], pol[0]
        flops = 2.0 * (D_obs * Hh + Hh * max(w.n_actions, w.act_dim)) * E * A * T
        fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12
        tf = flops / (roll_ms / 1e3) / 1e12 if roll_ms > 0 else 0.0
        roofline["kernel"] = (f"k_rollout_gpolicy<{Hh}> (Gaussian, Pendulum)" if w.n_actions == 0
                              else f"k_tag<policy {Hh}> (agent threads)" if w.env == "tag"
                              else f"k_rollout_policy<{w.env},{Hh}>")
        roofline["other_kernels"] = {}
        roofline["alu_view"] = {"achieved": round(tf, 3), "peak": round(fp32_peak, 1), "unit": "TFLOP/s",
                                "frac": round(tf / fp32_peak, 4), "flops_per_launch": flops,
                                "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x 1.965 GHz (B200_PROFILING.md)"}
        if tf / fp32_peak > roofline["frac"]:  # report the binding one
            hbm_view = {k: roofline[k] for k in ("achieved", "peak", "unit", "frac")}
            roofline.update({"bound": "alu", "achieved": round(tf, 3), "peak": round(fp32_peak, 1),
                             "unit": "TFLOP/s", "frac": round(tf / fp32_peak, 4), "hbm_view": hbm_view})
    if staged:
        # the same kernels one step at a time (diagnostic pass timing of the step kernel) and
        # the transfer split of the last timed step
        n_st, st_ms = diag_times.get("step", (0, 0.0))
        sb = ROLLOUT_BYTES.get(w.env, 0) * E * A
        ach = sb / (st_ms / 1e3) / 1e9 if st_ms > 0 else 0.0
        roofline.update({"kernel": f"k_step_lane<{w.env}> (single step)", "kernel_ms": round(st_ms, 5),
                         "launches_timed": n_st, "bytes_per_launch": sb, "achieved": round(ach, 1),
                         "frac": round(ach / peak, 4), "other_kernels": {}})
        roofline["staged_pipeline"] = {k: (round(v, 4) if "ms" in k else v) for k, v in staged_rep.items()}
        roofline["staged_pipeline"]["transfer_share"] = round(staged_rep["transfer_ms"] / staged_rep["total_ms"], 4)
    if trainer is not None:
        roofline["a2c_update"] = {"ms": round(upd_ms, 4), "rows": E * A * T,
                                  "note": "gae + moments + gradient + clip/Adam (the critic comes from the roll-out kernel), diagnostic pass",
                                  "loss_last": [round(x, 6) for x in trainer.loss.cpu().tolist()]}
    if gae:
        n_gae, gae_ms = ktimes.get("gae", (0, 0.0))
        g_ach = gae_bytes / (gae_ms / 1e3) / 1e9 if gae_ms > 0 else 0.0
        roofline["gae_kernel"] = {"kernel": "k_gae_tma", "bound": "hbm", "achieved": round(g_ach, 1), "peak": peak,
                                  "unit": "GB/s", "frac": round(g_ach / peak, 4), "kernel_ms": round(gae_ms, 4),
                                  "launches_timed": n_gae, "bytes_per_launch": gae_bytes,
                                  "bytes_per_agent_step": gae_bytes / (E * A * T)}
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        try:
            tr = json.load(open(traffic_file)).get(w.name)
            if tr:
                roofline["traffic"] = tr
        except Exception:
            pass

    line = None
    if rank == 0:
        e2e = None
        if not args.ncu:
            # end to end through the public API with HOST buffers: pinned probs H2D + stats D2H per step
            henv = Env(E, A, w.env, W.SEED, env_offset=offset, n_envs_global=E_g, t_capacity=T,
                       param0=params[0], param1=params[1], block_size=args.block)
            if trainer is not None:  # NEXT-N2: one training iteration per step, loss + stats back to the host
                from paper_2408_00930_b200.a2c import A2C, PPO
                ppo = w.params.get("ppo")
                htr = (PPO(henv, pol[0], params=pol_w, epochs=ppo[0], minibatches=ppo[1], lr=1e-4) if ppo else
                       A2C(henv, pol[0], params=pol_w, lr=1e-4, gamma=0.99, lam=0.95, c_v=0.5, c_e=0.01,
                           max_norm=0.5))
                hl = torch.empty(3, dtype=torch.float64).pin_memory()
                hs = torch.empty((T, 4), dtype=torch.int64).pin_memory()

                def host_step():
                    htr.iteration(T)
                    hl.copy_(htr.loss, non_blocking=True)
                    hs.copy_(henv.buffers()["stats"][:T], non_blocking=True)
                    torch.cuda.synchronize(dev)
                h2d = 0
            elif staged:  # NEXT-N3: the staged pipeline is host-buffered by construction
                hdst = henv.host_store(T)

                def host_step():
                    henv.rollout_staged(T, st_probs, hdst)
                h2d = int(st_probs.numel() * 4 * T)
            elif pol:  # NEXT-N1: pinned host weights -> device each step, stats back to the host
                hw = torch.from_numpy(pol[1]).pin_memory()
                dw = torch.empty_like(hw, device=dev)
                hs = torch.empty((T, 4), dtype=torch.int64).pin_memory()

                def host_step():
                    dw.copy_(hw, non_blocking=True)
                    henv.rollout_policy(T, dw, pol[0])
                    hs.copy_(henv.buffers()["stats"][:T], non_blocking=True)
                    torch.cuda.synchronize(dev)
                h2d = int(hw.numel() * 4)
            else:
                hp = torch.from_numpy(probs_host).pin_memory()

                def host_step():
                    henv.rollout_host(T, hp)
                    if gae:
                        henv.gae_store(T, g_vals, g_boot, gae[0], gae[1], out=g_out)
                        torch.cuda.synchronize(dev)
                h2d = int(hp.numel() * 4)
            for _ in range(max(args.warmup, 1)):
                host_step()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                host_step()
            e2e_s = time.perf_counter() - t0
            d2h = (int(sum(v.numel() * v.element_size() for v in hdst.values())) if staged
                   else int(T * 4 * 8) + (24 if trainer is not None else 0))
            e2e = {"value": E * T * args.steps / e2e_s, "unit": "env-steps/s",
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                   "note": "rank 0, " + ("ws_rollout_staged (per-step copies)" if staged else
                                         "A2C iteration, loss + stats to pinned host memory" if trainer is not None
                                         else "ws_rollout_policy with pinned weights" if pol else "ws_rollout_host")
                           + (" + ws_gae_store" if gae else "")
                           + ", host wall clock"}
            henv.close()
        line = {
            "metric": "env-steps/s", "value": value, "unit": "env-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{w.name}: {w.note}", "env": w.env, "n_envs_per_gpu": E, "n_envs_global": E_g,
                       "n_agents": A, "T": T, "probs": "uniform, resident in HBM, step_stride 0",
                       "parallelism": (f"env-shard x{world} + " + ("peer-memory (CUDA IPC, NVLink) stats all-reduce kernel"
                                                                    if p2p else "NCCL stats all-reduce")) if world > 1 else "1 GPU",
                       "l2": f"store {all_bytes / 1e6:.0f} MB written per step > 126 MB L2 (no flush needed)"},
            "roofline": roofline, "gpu_launches": int(launches),
            "episode_stats_last_step": merged,
            "clocks": clk, "e2e": e2e,
            "paper_context": "A100 8.6M env-steps/s incl. training (P:39); not like-for-like",
        }
        if not args.no_cpu_baseline and not args.ncu and world == 1:
            line["cpu_baseline"] = cpu_baseline(w)
        print(json.dumps(line), flush=True)
        if args.csv:
            write_csv_row(args.csv, w, world, E_g, A, T, line)
    env.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
