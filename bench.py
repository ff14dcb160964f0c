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
    ap.add_argument("--stats-reduce", default="nccl", choices=["p2p", "nccl"],
                    help="N > 1: statistics all-reduce by NCCL (default, north_star's design) or libws's "
                         "peer-memory kernel (opt-in)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank runs the workload's full replica count (global = N x E); strong: the "
                         "workload's E is the global count, split by parallel.shard.  At N > 1 the other mode is "
                         "measured too and reported under `other_scaling`")
    ap.add_argument("--sustain-s", type=float, default=1.0,
                    help="after the K timed steps, a sustained pass of >= this many seconds (clock sampling, p10/p90)")
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


def host_cpu() -> dict:
    """CPU model and core counts of the host the oracle runs on (lscpu)."""
    info = {"model": None, "sockets": None, "physical_cores": None, "logical_cpus": os.cpu_count(),
            "affinity_cpus": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        sockets = int(kv.get("Socket(s)", "0") or 0)
        cps = int(kv.get("Core(s) per socket", "0") or 0)
        info["sockets"] = sockets or None
        info["physical_cores"] = sockets * cps or None
    except (OSError, ValueError, subprocess.SubprocessError):
        pass
    return info


def _oracle_rate(w, budget_s: float, cores: int):
    """Consecutive oracle roll-outs of workload w on `cores` threads for ~budget_s; returns
    (env-steps/s, sample description, per-roll-out seconds)."""
    import oracle as O
    probs = W.workload_probs(w)
    b = O.Batch(w.env, w.n_envs, w.n_agents, W.SEED, t_capacity=w.T)
    t0 = time.perf_counter()
    oracle_rollout(b, w, min(10, w.T), probs, cores)
    probe = time.perf_counter() - t0
    T_s = max(10, min(w.T, int(min(10, w.T) * budget_s / 3 / max(probe, 1e-6))))
    steps, n, per = 0, 0, []
    t0 = time.perf_counter()
    while True:
        t1 = time.perf_counter()
        oracle_rollout(b, w, T_s, probs, cores)
        per.append(time.perf_counter() - t1)
        steps += w.n_envs * T_s
        n += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s or n >= 1000:
            break
    return steps / dt, f"{n} x ({w.n_envs} replicas x {T_s} steps) = {steps} env-steps in {dt:.1f} s", per, \
        w.n_envs * T_s


def cpu_baseline(w, budget_s: float = 10.0, budget_w1_s: float = 6.0):
    """The oracle as it stands (oracle/, never tuned for this), on this host's cores, on a
    bounded sample of the same workload: consecutive roll-outs of every replica over a prefix
    of T_s steps until ~budget_s of CPU work -- once with W = all host threads (the reported
    value) and once with W = 1."""
    cores = len(os.sched_getaffinity(0))
    register_user(w, oracle_side=True)
    if w.params.get("gae"):
        oracle_gae_inputs(w)
    v, sample, per, units = _oracle_rate(w, budget_s, cores)
    v1, sample1, per1, units1 = _oracle_rate(w, budget_w1_s, 1)
    pct = lambda xs, q: float(np.percentile(np.asarray(xs), q))
    return {"value": v, "unit": "env-steps/s", "cores": cores, "kind": "oracle",
            "sample": f"{w.name} {w.env}: {sample} on {cores} threads",
            "p10_p90": [units / pct(per, 90), units / pct(per, 10)],
            "w1": {"value": v1, "cores": 1, "sample": sample1, "p10_p90": [units1 / pct(per1, 90), units1 / pct(per1, 10)]},
            "host": host_cpu()}


def shard_sizes(E_g: int, world: int) -> list:
    """parallel.shard's contiguous balanced partition (restated: the reference arm must not
    import the product package)."""
    return [E_g * (r + 1) // world - E_g * r // world for r in range(world)]


def layout(w, world: int, scaling: str):
    """(E_global, [E per rank]) of workload w on `world` ranks."""
    if scaling == "weak":
        return w.n_envs * world, [w.n_envs] * world
    return w.n_envs, shard_sizes(w.n_envs, world)


def inputs_desc(w) -> str:
    if W.workload_policy(w):
        return f"in-kernel MLP policy (hidden {w.params['policy_hidden']}), seeded weights"
    if w.n_actions:
        return f"uniform 1/{w.n_actions} probabilities, resident in HBM, step_stride 0"
    return "Gaussian head (mean, log_std) per replica, resident in HBM, step_stride 0"


def make_config(w, world: int, scaling: str, reduce: str) -> dict:
    """The `config` object -- identical for both arms (the driver compares them)."""
    E_g, per = layout(w, world, scaling)
    par = "1 GPU" if world == 1 else (
        f"{world} GPUs: contiguous replica shards (parallel.shard) + one sum all-reduce of the [T,4] statistics per "
        f"roll-out ({'NCCL' if reduce == 'nccl' else 'libws peer-memory kernel over CUDA IPC'})")
    return {"workload": f"{w.name}: {w.note}", "env": w.env, "n_envs_global": E_g, "n_envs_per_rank": per,
            "n_agents": w.n_agents, "T": w.T, "inputs": inputs_desc(w), "scaling": scaling, "parallelism": par}


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
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": make_config(w, args.gpus, args.scaling, args.stats_reduce),
            "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": cores, "kind": "oracle",
                             "sample": f"{w.n_envs} replicas x {T_s} of the {w.T} steps per step, on {cores} host "
                                       f"threads (oracle/); rank 0 only", "host": host_cpu()},
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


L2_BYTES = 126 * 2 ** 20  # B200 L2 (B200_PROFILING.md)


def issue_table() -> dict:
    """Per-workload ncu counters of the dominant kernel (profiles/ncu_inst.json, written from
    `ncu --set full` captures): warp instructions executed per launch, issue-active %, DRAM bytes."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_inst.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def pct(xs, q):
    return float(np.percentile(np.asarray(xs, np.float64), q)) if len(xs) else None


class Run:
    """One measured configuration (scaling mode) of workload w on this rank."""

    def __init__(self, args, w, world, rank, dev, scaling):
        import dataclasses
        from paper_2408_00930_b200 import Env
        self.args, self.world, self.rank, self.dev, self.scaling = args, world, rank, dev, scaling
        self.E_g, per = layout(w, world, scaling)
        self.E = per[rank]
        self.offset = sum(per[:rank])
        self.w = dataclasses.replace(w, n_envs=self.E)  # this rank's shard (inputs sized for it)
        self.A, self.T = w.n_agents, w.T
        self.params = (w.params.get("grid", w.params.get("dim", 0)), w.params.get("taggers", 0))
        self.Env = Env
        self.env = self.make_env()
        self.stream = torch.cuda.current_stream(dev)
        wl = self.w
        self.probs_host = W.workload_probs(wl)
        self.probs = torch.from_numpy(self.probs_host).to(dev)
        self.stats_view = self.env.buffers()["stats"][:self.T]
        self.pol = W.workload_policy(wl)
        self.pol_w = torch.from_numpy(self.pol[1]).to(dev) if self.pol else None
        self.gae = w.params.get("gae")
        if self.gae:
            self.g_vals, self.g_boot, _ = (torch.from_numpy(x).to(dev) if x is not None else None
                                           for x in W.gae_inputs(self.T, self.E, self.A, seed=W.SEED + rank))
            self.g_out = (torch.empty((self.T, self.E, self.A), dtype=torch.float32, device=dev),
                          torch.empty((self.T, self.E, self.A), dtype=torch.float32, device=dev))
        self.trainer = self.make_trainer(self.env) if w.params.get("a2c") else None
        self.staged = w.params.get("staged")
        self.staged_rep = {}
        if self.staged:
            self.st_probs = torch.from_numpy(self.probs_host).pin_memory()
            self.st_dst = self.env.host_store(self.T)
        self.p2p = False
        if world > 1 and args.stats_reduce == "p2p":
            from paper_2408_00930_b200.parallel import attach_peer_stats
            self.p2p = attach_peer_stats(self.env)  # falls back to NCCL if CUDA IPC is unavailable on any rank

    def make_env(self):
        return self.Env(self.E, self.A, self.w.env, W.SEED, env_offset=self.offset, n_envs_global=self.E_g,
                        t_capacity=self.T, param0=self.params[0], param1=self.params[1], block_size=self.args.block)

    def make_trainer(self, env):
        from paper_2408_00930_b200.a2c import A2C, PPO
        ppo = self.w.params.get("ppo")
        pol = self.pol
        return (PPO(env, pol[0], params=self.pol_w, epochs=ppo[0], minibatches=ppo[1], lr=1e-4) if ppo else
                A2C(env, pol[0], params=self.pol_w, lr=1e-4, gamma=0.99, lam=0.95, c_v=0.5, c_e=0.01, max_norm=0.5))

    def rollout(self):
        env, T = self.env, self.T
        if self.staged:
            self.staged_rep.update(env.rollout_staged(T, self.st_probs, self.st_dst))
        elif self.trainer is not None:
            self.trainer.iteration(T)
        elif self.pol:
            env.rollout_policy(T, self.pol_w, self.pol[0])
        else:
            env.rollout(T, self.probs)
        if self.gae:
            env.gae_store(T, self.g_vals, self.g_boot, self.gae[0], self.gae[1], out=self.g_out)

    def step(self):
        """One bench step: the whole hot path over the batch + (N > 1) the statistics all-reduce."""
        self.rollout()
        if self.world > 1 and not self.p2p:
            from paper_2408_00930_b200.parallel import allreduce_stats
            allreduce_stats(self.stats_view)

    def barrier(self):
        torch.cuda.synchronize(self.dev)
        if self.world > 1:
            dist.barrier()

    def warm(self, n):
        for _ in range(max(n, 0)):
            self.step()
        self.barrier()
        if self.p2p:  # the peer-memory reduction must have worked on every rank, else fall back to NCCL
            ok = torch.tensor([1 if self.env.status() == 0 else 0], dtype=torch.int32, device=self.dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0:
                print("warning: peer-memory statistics reduction failed during warm-up; using NCCL", file=sys.stderr)
                self.env.peer_detach()
                self.env.reset()
                self.p2p = False
                for _ in range(max(n, 1)):
                    self.step()
                self.barrier()

    def timed(self, K, flush, per_step=False):
        """K steps timed with CUDA events on the handle's stream: two events around the K steps
        (per_step: one event per step boundary, per-step times for p10 / p90).  flush: an L2
        flush (a 256 MB write) before every step, outside the events (stores smaller than L2)."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1 if not flush else 2 * K)]
        self.barrier()
        if not flush and not per_step:  # two events: an event between steps costs the loop ~3 us
            ev[0].record(self.stream)
            for k in range(K):
                self.step()
            ev[1].record(self.stream)
            self.barrier()
            per = [ev[0].elapsed_time(ev[1]) / K] * K
        elif not flush:
            ev[0].record(self.stream)
            for k in range(K):
                self.step()
                ev[k + 1].record(self.stream)
            self.barrier()
            per = [ev[k].elapsed_time(ev[k + 1]) for k in range(K)]
        else:
            for k in range(K):
                self.flush_buf.zero_()
                ev[2 * k].record(self.stream)
                self.step()
                ev[2 * k + 1].record(self.stream)
            self.barrier()
            per = [ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(K)]
        return per

    def max_over_ranks(self, x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        self.env.close()


def roofline_of(run, ktimes, diag_times, kern_ms, peak, peak_src, peaks, n_diag, upd_ms, w):
    E, A, T = run.E, run.A, run.T
    pol, gae, trainer, staged = run.pol, run.gae, run.trainer, run.staged
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
    all_bytes = store_bytes(w, E)
    gae_bytes = 16 * E * A * T + E * T + 4 * E * A if gae else 0
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
    # issue view (report max(f_HBM, f_issue) and name the binding one): warp
    # instructions the kernel executes per launch (ncu, profiles/ncu_inst.json, same workload and
    # shape) / its live launch time, against 148 SMs x 4 schedulers x 1 warp-instruction / clock
    tab = issue_table().get(w.name)
    if tab and tab.get("E") == E and roll_ms > 0 and not pol and not staged:
        clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        issue_peak = 148 * 4 * clk / 1e9  # G warp-instructions / s
        ach_i = tab["inst_per_launch"] / (roll_ms / 1e3) / 1e9
        roofline["issue_view"] = {"achieved": round(ach_i, 1), "peak": round(issue_peak, 1),
                                  "unit": "G warp-inst/s", "frac": round(ach_i / issue_peak, 4),
                                  "inst_per_launch": tab["inst_per_launch"],
                                  "ncu_issue_active_pct": tab.get("issue_active_pct"),
                                  "source": tab.get("source")}
        if tab.get("dram_bytes") is not None:
            roofline["traffic"] = tab["dram_bytes"]
        if ach_i / issue_peak > roofline["frac"]:
            hbm_view = {k: roofline[k] for k in ("achieved", "peak", "unit", "frac")}
            roofline.update({"bound": "alu", "achieved": round(ach_i, 1), "peak": round(issue_peak, 1),
                             "unit": "G warp-inst/s", "frac": round(ach_i / issue_peak, 4), "hbm_view": hbm_view,
                             "peak_source": f"derived: 148 SMs x 4 SMSPs x 1 warp-instruction/clk x "
                                            f"{clk / 1e6:.0f} MHz (MEASURED_PEAKS sm_max_mhz)"})
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
        n_st, st_ms = diag_times.get("step", (0, 0.0))
        sb = ROLLOUT_BYTES.get(w.env, 0) * E * A
        ach = sb / (st_ms / 1e3) / 1e9 if st_ms > 0 else 0.0
        roofline.update({"kernel": f"k_step_lane<{w.env}> (single step)", "kernel_ms": round(st_ms, 5),
                         "launches_timed": n_st, "bytes_per_launch": sb, "achieved": round(ach, 1),
                         "frac": round(ach / peak, 4), "other_kernels": {}})
        roofline["staged_pipeline"] = {k: (round(v, 4) if "ms" in k else v) for k, v in run.staged_rep.items()}
        roofline["staged_pipeline"]["transfer_share"] = round(run.staged_rep["transfer_ms"] / run.staged_rep["total_ms"], 4)
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
    if roofline["traffic"] is None:
        traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
        try:
            tr = json.load(open(traffic_file)).get(w.name)
            if tr and run.world == 1:
                roofline["traffic"] = tr
        except (OSError, ValueError):
            pass
    return roofline


def store_bytes(w, E: int) -> int:
    """Algorithmic bytes one step writes into (and reads from) the store on one rank."""
    A, T = w.n_agents, w.T
    if w.params.get("policy_hidden"):
        b = (4 * OBS_DIM[w.env] + 4 + 1 + 8) * E * A * T
    elif w.env == "tag":
        b = (16 + 4 + 4 + 4) * E * A * T + E * T
    elif w.env in USER_BYTES:
        b = USER_BYTES[w.env] * E * A * T
    else:
        b = (ROLLOUT_BYTES.get(w.env, 0) + PLAN_BYTES.get(w.env, 8)) * E * A * T
    if w.params.get("gae"):
        b += 16 * E * A * T + E * T + 4 * E * A
    return int(b)


def e2e_pass(run, args, dev, world):
    """End to end through the public API with HOST buffers, on every rank (the trainers'
    collectives and the statistics all-reduce need all of them): per step the pinned-host
    inputs go H2D and the step's result (statistics, loss) comes back D2H; host wall clock,
    max over ranks."""
    from paper_2408_00930_b200.parallel import allreduce_stats
    w, T, E, A = run.w, run.T, run.E, run.A
    henv = run.make_env()
    hstats = henv.buffers()["stats"][:T]
    trainer, staged, pol, gae = run.trainer, run.staged, run.pol, run.gae
    pipelined = False
    if trainer is not None:  # NEXT-N2: one training iteration per step, loss + stats back to the host
        htr = run.make_trainer(henv)
        hl = torch.empty(3, dtype=torch.float64).pin_memory()
        hs = torch.empty((T, 4), dtype=torch.int64).pin_memory()

        def host_step():
            htr.iteration(T)
            if world > 1:
                allreduce_stats(hstats)
            hl.copy_(htr.loss, non_blocking=True)
            hs.copy_(hstats, non_blocking=True)
            torch.cuda.synchronize(dev)
        h2d, d2h = 0, T * 4 * 8 + 24
    elif staged:  # NEXT-N3: the staged pipeline is host-buffered by construction
        hdst = henv.host_store(T)

        def host_step():
            henv.rollout_staged(T, run.st_probs, hdst)
            if world > 1:
                allreduce_stats(hstats)
                torch.cuda.synchronize(dev)
        h2d = int(run.st_probs.numel() * 4 * T)
        d2h = int(sum(v.numel() * v.element_size() for v in hdst.values()))
    elif pol:  # NEXT-N1: pinned host weights -> device each step, stats back to the host
        hw = torch.from_numpy(pol[1]).pin_memory()
        dw = torch.empty_like(hw, device=dev)
        hs = torch.empty((T, 4), dtype=torch.int64).pin_memory()

        def host_step():
            dw.copy_(hw, non_blocking=True)
            henv.rollout_policy(T, dw, pol[0])
            if world > 1:
                allreduce_stats(hstats)
            hs.copy_(hstats, non_blocking=True)
            torch.cuda.synchronize(dev)
        h2d, d2h = int(hw.numel() * 4), T * 4 * 8
    else:
        hp = torch.from_numpy(run.probs_host).pin_memory()
        hs = torch.empty((T, 4), dtype=torch.int64).pin_memory()
        if world == 1 and not gae:
            # the public pipelined host API (ws_rollout_host_submit / _wait, two deep): every step
            # still copies its pinned inputs H2D and reads its statistics back to the host, but the
            # next step is submitted before this one's result is awaited
            def host_steps(n):
                henv.rollout_host_submit(T, hp, 0)
                for k in range(n):
                    if k + 1 < n:
                        henv.rollout_host_submit(T, hp, (k + 1) & 1)
                    henv.rollout_host_wait(k & 1)
            pipelined = True

        def host_step():
            if world > 1:  # ws_rollout_host + the statistics all-reduce, then the merged slab to the host
                henv.rollout_host(T, hp)
                allreduce_stats(hstats)
                hs.copy_(hstats, non_blocking=True)
                torch.cuda.synchronize(dev)
            else:
                henv.rollout_host(T, hp)
            if gae:
                henv.gae_store(T, run.g_vals, run.g_boot, gae[0], gae[1], out=run.g_out)
                torch.cuda.synchronize(dev)
        h2d, d2h = int(hp.numel() * 4), T * 4 * 8
    if pipelined:
        host_steps(max(args.warmup, 1))
        run.barrier()
        t0 = time.perf_counter()
        host_steps(args.steps)
    else:
        for _ in range(max(args.warmup, 1)):
            host_step()
        run.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            host_step()
    e2e_s = time.perf_counter() - t0
    e2e_s = run.max_over_ranks(e2e_s)
    henv.close()
    return {"value": run.E_g * T * args.steps / e2e_s, "unit": "env-steps/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "note": ("every rank, " if world > 1 else "") +
                    ("ws_rollout_staged (per-step copies)" if staged else
                     "A2C iteration, loss + stats to pinned host memory" if trainer is not None
                     else "ws_rollout_policy with pinned weights" if pol else
                     "ws_rollout_host_submit / _wait (pipelined two deep)" if pipelined else "ws_rollout_host")
                    + (" + ws_gae_store" if gae else "") + (" + NCCL stats all-reduce" if world > 1 else "")
                    + ", host wall clock" + (", max over ranks" if world > 1 else "")}


def main():
    args = parse()
    w = W.CONFIGS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)

    global torch, dist
    import torch
    import torch.distributed as dist

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
    register_user(w, oracle_side=False)

    run = Run(args, w, world, rank, dev, args.scaling)
    E, A, T, E_g = run.E, run.A, run.T, run.E_g
    sb = store_bytes(w, E)
    flush = sb < 2 * L2_BYTES
    if flush:
        run.flush_buf = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
    run.warm(args.warmup)

    clocks = Clocks(local_dev)
    if not args.ncu:
        clocks.start()
        time.sleep(0.3)
    # two CUDA events around the fused roll-out kernel only (libws ws_kernel_times), on every
    # fourth launch of a >= 8-step timed loop: the dominant kernel is timed live with the least
    # perturbation of the timed loop (an event pair between kernels costs it ~6 us per step)
    kt_period = 4 if args.steps >= 8 else 1
    run.env.enable_kernel_timing(0 if (args.no_kernel_timing or run.staged) else (3 if run.gae else 2),
                                 period=kt_period)
    run.env.kernel_times()
    launches0 = run.env.info().launches
    per = run.timed(args.steps, flush)
    total_ms = sum(per)
    st = run.env.status()  # sticky device errors (invalid rows, peer reduction timeout) fail the run
    if st != 0:
        raise RuntimeError(f"libws reported status {st} during the timed region")
    launches = run.env.info().launches - launches0
    if run.trainer is not None:  # handle-free kernels per step: moments + final, then (grad + final, Adam) per update
        n_upd = (w.params["ppo"][0] * w.params["ppo"][1]) if w.params.get("ppo") else 1
        launches += (2 + 3 * n_upd) * args.steps
    ktimes = run.env.kernel_times()
    run.env.enable_kernel_timing(False)
    max_ms = run.max_over_ranks(total_ms)
    value = E_g * T * args.steps / (max_ms / 1e3)
    ms_per_step = max_ms / args.steps

    # merged per-slot statistics of the last timed roll-out (all ranks, exact int64; R20)
    from paper_2408_00930_b200.parallel import summarize
    merged = summarize(run.stats_view.cpu())

    # sustained pass (>= --sustain-s seconds; not part of `value`): clocks under a long load and
    # a stable p10 / p90 of the per-step time
    sustained = None
    if not args.ncu and args.sustain_s > 0:
        n_sus = int(min(100000, max(args.steps, np.ceil(args.sustain_s * 1e3 / max(ms_per_step, 1e-3)))))
        per_s = run.timed(n_sus, flush, per_step=True)
        sus_ms = run.max_over_ranks(sum(per_s))
        sustained = {"steps": n_sus, "seconds": round(sus_ms / 1e3, 3), "value": E_g * T * n_sus / (sus_ms / 1e3),
                     "ms_per_step": sus_ms / n_sus, "p10_ms": pct(per_s, 10), "p50_ms": pct(per_s, 50),
                     "p90_ms": pct(per_s, 90), "note": "rank-local per-step percentiles; value = max over ranks"}
    clk = clocks.stop() if not args.ncu else {}

    # diagnostic pass after the timed region (not part of `value`): every kernel and the whole
    # ws_rollout call bracketed by events
    n_diag = max(1, min(args.steps, 5))
    run.env.enable_kernel_timing(1)
    run.env.kernel_times()
    dev_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n_diag)]
    for k in range(n_diag):
        dev_ev[2 * k].record(run.stream)
        run.rollout()
        dev_ev[2 * k + 1].record(run.stream)
    torch.cuda.synchronize(dev)
    kern_ms = [dev_ev[2 * k].elapsed_time(dev_ev[2 * k + 1]) for k in range(n_diag)]
    diag_times = run.env.kernel_times()
    run.env.enable_kernel_timing(False)
    upd_ms = None
    if run.trainer is not None:  # the update alone (critic, GAE, moments, gradient, Adam)
        for k in range(n_diag):
            dev_ev[2 * k].record(run.stream)
            run.trainer.update(T, values_ready=True)
            dev_ev[2 * k + 1].record(run.stream)
        torch.cuda.synchronize(dev)
        upd_ms = sum(dev_ev[2 * k].elapsed_time(dev_ev[2 * k + 1]) for k in range(n_diag)) / n_diag
    if world > 1:
        dist.barrier()

    peaks, peak_src = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    roofline = roofline_of(run, ktimes, diag_times, kern_ms, peak, peak_src, peaks, n_diag, upd_ms, w)

    e2e = e2e_pass(run, args, dev, world) if not args.ncu else None
    p2p = run.p2p
    run.close()

    # N > 1: the other scaling mode too (strong = the workload's E split over the ranks,
    # e.g. BJ:2's 10K CartPole total; weak = E per rank)
    other = None
    if world > 1 and not args.ncu:
        mode = "strong" if args.scaling == "weak" else "weak"
        r2 = Run(args, w, world, rank, dev, mode)
        if flush or store_bytes(w, r2.E) < 2 * L2_BYTES:
            r2.flush_buf = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
        r2.warm(args.warmup)
        per2 = r2.timed(args.steps, store_bytes(w, r2.E) < 2 * L2_BYTES)
        m2 = r2.max_over_ranks(sum(per2))
        other = {"scaling": mode, "n_envs_global": r2.E_g, "n_envs_per_rank": layout(w, world, mode)[1],
                 "value": r2.E_g * T * args.steps / (m2 / 1e3), "ms_per_step": m2 / args.steps,
                 "p10_ms": pct(per2, 10), "p90_ms": pct(per2, 90)}
        r2.close()

    if rank == 0:
        l2 = (f"store {sb / 1e6:.1f} MB per step per GPU < 2 x L2 (126 MB): L2 flushed (256 MB write) before every "
              f"timed step, outside the events" if flush else
              f"store {sb / 1e6:.0f} MB per step per GPU > 2 x L2 (126 MB): no flush needed")
        line = {
            "metric": "env-steps/s", "value": value, "unit": "env-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": make_config(w, world, args.scaling, "p2p" if p2p else "nccl"),
            "timing": ({"p10_ms": pct(per, 10), "p50_ms": pct(per, 50), "p90_ms": pct(per, 90), "l2": l2,
                        "per_step_events": True} if flush else
                       {"l2": l2, "per_step_events": False,
                        "note": "two events around the K steps (per-step p10 / p50 / p90: `sustained`); the "
                                "roll-out kernel bracketed on every %d-th step" % kt_period}),
            "roofline": roofline, "gpu_launches": int(launches),
            "episode_stats_last_step": merged,
            "clocks": clk, "e2e": e2e, "sustained": sustained,
            "paper_context": "A100 8.6M env-steps/s incl. training (P:39); not like-for-like",
        }
        if other is not None:
            line["other_scaling"] = other
        if not args.no_cpu_baseline and not args.ncu and world == 1:
            line["cpu_baseline"] = cpu_baseline(w)
        print(json.dumps(line), flush=True)
        if args.csv:
            write_csv_row(args.csv, w, world, E_g, A, T, line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
