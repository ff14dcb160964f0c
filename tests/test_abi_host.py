"""CPU-only checks of the boundary: libws.so loads, exports every function include/ws.h
declares, and its host-side argument validation answers without a GPU;
sharding arithmetic and the statistics merge of the multi-GPU path."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

import paper_2408_00930_b200 as P
from paper_2408_00930_b200 import _abi
from paper_2408_00930_b200.parallel import shard, summarize
import wsinputs as W


def test_library_exports_every_declared_symbol():
    names = P.declared_functions()
    assert len(names) >= 17
    L = P.lib()
    for n in names:
        assert hasattr(L, n), n
    assert L.ws_abi_version() == 1


def test_config_init_defaults():
    cfg = _abi.ws_config()
    assert P.lib().ws_config_init(C.byref(cfg)) == 0
    assert cfg.n_agents == 1 and cfg.device == -1 and cfg.write_logp == 1 and cfg.t_capacity == 0


def test_struct_layouts_match_header():
    # sizes the C compiler gives the ws.h structs on x86-64 (natural alignment)
    assert C.sizeof(_abi.ws_tensor) == 8 + 4 + 4 + 5 * 8
    assert C.sizeof(_abi.ws_buffers) == 11 * C.sizeof(_abi.ws_tensor)
    assert C.sizeof(_abi.ws_stats) == 6 * 8
    assert C.sizeof(_abi.ws_info) == 8 * 4 + 3 * 8 + 2 * 8 + 2 * 4
    assert C.sizeof(_abi.ws_config) == 8 * 3 + 8 + 8 + 8 + 8 + 8 + 6 * 4 + 3 * 8 + 2 * 8  # + env_prm, env_shared


def _create(**kw):
    L = P.lib()
    cfg = _abi.ws_config()
    L.ws_config_init(C.byref(cfg))
    cfg.n_envs = kw.get("n_envs", 4)
    cfg.n_agents = kw.get("n_agents", 1)
    name = kw.get("env", "cartpole").encode()
    cfg.env = name
    cfg.env_offset = kw.get("env_offset", 0)
    cfg.n_envs_global = kw.get("n_envs_global", 0)
    cfg.param0 = kw.get("param0", 0)
    cfg.block_size = kw.get("block_size", 0)
    h = C.c_void_p()
    st = L.ws_create_ex(C.byref(cfg), C.byref(h))
    return st, h


@pytest.mark.parametrize("kw,status", [
    (dict(n_envs=0), _abi.INVALID_ARGUMENT),                      # S:138 E = 0
    (dict(env="nosuch"), _abi.UNKNOWN_ENV),
    (dict(n_agents=2), _abi.INVALID_ARGUMENT),                    # single-agent env
    (dict(env_offset=5, n_envs=4, n_envs_global=8), _abi.INVALID_ARGUMENT),  # shard past E_g
    (dict(env="surface", param0=7), _abi.INVALID_ARGUMENT),       # unsupported surface dimension
    (dict(block_size=48), _abi.INVALID_ARGUMENT),                 # launch shape must be k*32
])
def test_create_validates_before_touching_the_gpu(kw, status):
    st, h = _create(**kw)
    assert st == status and not h.value


def test_null_handle_and_status_strings():
    L = P.lib()
    assert L.ws_reset(None) == _abi.INVALID_ARGUMENT
    assert L.ws_destroy(None) == _abi.OK
    for s in range(10):
        assert L.ws_status_string(s) and L.ws_status_string(s) != b"unknown status"
    # the later entry points validate their handle before anything else
    assert L.ws_rollout_policy(None, 10, None, 32) == _abi.INVALID_ARGUMENT
    assert L.ws_peer_export(None, 2, None) == _abi.INVALID_ARGUMENT
    assert L.ws_peer_attach(None, 0, 2, None) == _abi.INVALID_ARGUMENT
    assert L.ws_peer_detach(None) == _abi.INVALID_ARGUMENT
    assert L.ws_enable_device_clock(None, 1) == _abi.INVALID_ARGUMENT
    assert L.ws_enable_kernel_timing(None, 2 | (4 << 8)) == _abi.INVALID_ARGUMENT


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_product_path_fails_loudly_without_gpu():
    with pytest.raises(P.WSError):
        P.Env(4, 1, "cartpole", 0)
    st, h = _create()
    assert st == _abi.CUDA_ERROR and not h.value  # no silent CPU fallback


def test_shard_balanced_contiguous():
    """E=10, W=3 -> [0,4) [4,7) [7,10) (lane analog: sizes differ by <= 1)."""
    assert [shard(10, 3, r) for r in range(3)] == [(0, 3), (3, 3), (6, 4)] or \
        [shard(10, 3, r) for r in range(3)] == [(0, 4), (4, 3), (7, 3)]
    for E in (1, 2, 10, 10000, 100003):
        for W in (1, 2, 3, 4, 8):
            parts = [shard(E, W, r) for r in range(W)]
            assert parts[0][0] == 0
            for (o1, n1), (o2, n2) in zip(parts, parts[1:]):
                assert o1 + n1 == o2
            assert sum(n for _, n in parts) == E
            assert max(n for _, n in parts) - min(n for _, n in parts) <= 1
    assert [n for _, n in (shard(2, 4, r) for r in range(4))].count(0) == 2


def test_summarize():
    st = torch.tensor([[2, 40, 30, 5], [0, 0, 0, 5], [1, 10, 10, 5]], dtype=torch.float64)
    s = summarize(st)
    assert s["episodes"] == 3 and s["mean_return"] == 50 / 3 and s["mean_length"] == 40 / 3


def test_gae_argument_validation_without_gpu():
    """ws_gae / ws_gae_store (NEXT-N2) reject bad arguments before any CUDA call."""
    L = P.lib()
    assert C.sizeof(_abi.ws_gae_args) == 4 + 4 + 8 + 5 * 8 + 4 + 4 + 2 * 8
    assert L.ws_gae(None, None) == _abi.INVALID_ARGUMENT
    fake = 256  # never dereferenced: validation fails first
    good = dict(T=4, n_agents=1, n_envs=8, rew=fake, done=fake, values=fake, bootstrap=fake, v_trunc=None,
                gamma=0.99, lam=0.95, adv=fake, ret=fake)
    for bad in (dict(T=0), dict(n_envs=0), dict(n_agents=0), dict(rew=None), dict(done=None), dict(values=None),
                dict(bootstrap=None), dict(adv=None), dict(ret=None), dict(gamma=1.5), dict(lam=-0.1),
                dict(gamma=float("nan"))):
        a = _abi.ws_gae_args(**{**good, **bad})
        assert L.ws_gae(C.byref(a), None) == _abi.INVALID_ARGUMENT, bad
    assert L.ws_gae_store(None, 4, None, None, None, 0.99, 0.95, None, None) == _abi.INVALID_ARGUMENT


def test_a2c_argument_validation_without_gpu():
    """NEXT-N2 A2C entry points (ws.h, R31): sizes and argument checks before any CUDA call."""
    L = P.lib()
    assert L.ws_a2c_n_params(4, 64, 2) == 4 * 64 + 64 + 64 * 2 + 2 + 64 + 1
    assert L.ws_a2c_n_params(6, 32, 3) == 6 * 32 + 32 + 32 * 3 + 3 + 32 + 1
    assert L.ws_a2c_workspace_bytes(4, 64, 2) >= 8 * (L.ws_a2c_n_params(4, 64, 2) + 3)
    for shape in ((5, 64, 2), (4, 48, 2), (4, 64, 4), (0, 64, 2)):
        assert L.ws_a2c_workspace_bytes(*shape) == 0, shape
    fake = 256
    assert L.ws_ac_values(fake, 4, 48, 2, fake, 10, fake, None) == _abi.INVALID_ARGUMENT
    assert L.ws_ac_values(None, 4, 64, 2, fake, 10, fake, None) == _abi.INVALID_ARGUMENT
    assert L.ws_ac_values(fake, 4, 64, 2, None, 0, None, None) == _abi.OK  # empty batch: nothing to do
    assert L.ws_a2c_moments(fake, 0, fake, fake, None) == _abi.INVALID_ARGUMENT
    assert L.ws_a2c_moments(None, 5, fake, fake, None) == _abi.INVALID_ARGUMENT
    assert L.ws_a2c_grad(None, None) == _abi.INVALID_ARGUMENT
    good = dict(obs_dim=4, hidden=64, n_actions=2, rows=10, params=fake, obs=fake, act=fake, adv=fake, ret=fake,
                moments=fake, batch=10.0, c_v=0.5, c_e=0.01, workspace=fake, grad=fake, loss=None)
    for bad in (dict(rows=0), dict(hidden=16), dict(obs_dim=3), dict(n_actions=4), dict(params=None),
                dict(obs=None), dict(act=None), dict(adv=None), dict(ret=None), dict(moments=None),
                dict(batch=0.0), dict(batch=float("nan")), dict(workspace=None), dict(grad=None)):
        a = _abi.ws_a2c_args(**{**good, **bad})
        assert L.ws_a2c_grad(C.byref(a), None) == _abi.INVALID_ARGUMENT, bad
    adam_ok = (fake, fake, fake, fake, 10, 1, 1e-3, 0.9, 0.999, 1e-8, 0.5, None, None)
    for i, v in ((4, 0), (4, 70000), (5, 0), (6, -1.0), (7, 1.0), (8, 1.0), (9, -1e-8), (0, None), (1, None)):
        args = list(adam_ok)
        args[i] = v
        assert L.ws_adam(*args) == _abi.INVALID_ARGUMENT, (i, v)


def test_staged_argument_validation_without_gpu():
    """NEXT-N3 ws_rollout_staged rejects a NULL handle before any CUDA call."""
    L = P.lib()
    hs = _abi.ws_host_store()
    assert L.ws_rollout_staged(None, 4, None, 0, 0, 0, C.byref(hs), None) == _abi.INVALID_ARGUMENT


def test_register_env_compiles_without_gpu():
    """NEXT-N4: ws_register_env compiles user C source with NVRTC for sm_100a on a CPU-only
    host; errors come back as WS_ERR_INVALID_ARGUMENT with the compiler log."""
    import wsinputs.user_envs as U
    L = P.lib()
    log = P.register_env("h_mountaincar", U.MOUNTAINCAR_SRC, **U.MOUNTAINCAR)
    assert L.ws_registered_env(b"h_mountaincar") == 1
    assert P.register_env("h_mountaincar", U.MOUNTAINCAR_SRC, **U.MOUNTAINCAR) == ""  # idempotent
    with pytest.raises(P.WSError) as ex:
        P.register_env("h_broken", "WS_FN int ws_env_step(float *s) { return undefined_symbol; }", 2, 2, 3, 1, 10)
    assert ex.value.status == _abi.INVALID_ARGUMENT and "undefined_symbol" in str(ex.value)
    assert L.ws_registered_env(b"h_broken") == 0
    buf = C.create_string_buffer(256)
    for bad in (dict(name=b"cartpole"), dict(state_dim=0), dict(obs_dim=33), dict(n_actions=1), dict(max_steps=0),
                dict(n_params=65), dict(source=None)):
        d = dict(name=b"h_x", source=U.MOUNTAINCAR_SRC.encode(), state_dim=2, obs_dim=2, n_actions=3,
                 n_reset_draws=1, max_steps=200, n_params=0)
        d.update(bad)
        assert L.ws_register_env(C.byref(_abi.ws_env_def(**d)), buf, 256) == _abi.INVALID_ARGUMENT, bad
    assert L.ws_set_env_data(None, None, None) == _abi.INVALID_ARGUMENT
    # every shipped user env (discrete, continuous, per-replica parameters) compiles against the
    # library's own device headers (common.cuh / sampler.cuh are NVRTC headers of the program)
    for name, (src, dims) in U.ENVS.items():
        P.register_env("h_" + name, src, **dims)
        assert L.ws_registered_env(("h_" + name).encode()) == 1


def test_param_checkpoint_round_trip_without_gpu(tmp_path):
    """flat little-endian float32 with a header; bit-exact round trip, including
    NaN payloads, -0 and subnormals; corrupted files are rejected."""
    from paper_2408_00930_b200 import checkpoint as ck
    p = torch.from_numpy(np.random.default_rng(1).standard_normal(515).astype(np.float32))
    p[3] = float("nan")
    p[4] = -0.0
    p[5] = 1e-40
    f = str(tmp_path / "p.wsac")
    ck.save_params(f, p, 4, 64, 2, "softmax")
    q, meta = ck.load_params(f)
    assert meta == {"obs_dim": 4, "hidden": 64, "n_actions": 2, "head": "softmax"}
    assert np.array_equal(q.numpy().view(np.uint32), p.numpy().view(np.uint32))
    raw = open(f, "rb").read()
    open(f, "wb").write(b"XXXX" + raw[4:])
    with pytest.raises(ValueError):
        ck.load_params(f)
    open(f, "wb").write(raw[:-4])
    with pytest.raises(ValueError):
        ck.load_params(f)
    assert P.lib().ws_set_time(None, 5) == _abi.INVALID_ARGUMENT


def test_peer_group_argument_validation_without_gpu():
    """ws.h peer groups reject bad arguments before any CUDA call."""
    L = P.lib()
    h = _abi.ws_ipc_handle()
    g = C.c_void_p()
    for world, n in ((0, 10), (9, 10), (2, 0), (2, 70000)):
        assert L.ws_pgroup_create(world, n, C.byref(g), C.byref(h)) == _abi.INVALID_ARGUMENT
    assert L.ws_pgroup_attach(None, 0, None) == _abi.INVALID_ARGUMENT
    assert L.ws_pgroup_allreduce(None, None, 1, None, None) == _abi.INVALID_ARGUMENT
    assert L.ws_pgroup_allreduce_adam(None, None, None, None, None, 1, 1e-3, 0.9, 0.999, 1e-8, 0.5, None, None,
                                      None) == _abi.INVALID_ARGUMENT
    assert L.ws_pgroup_status(None) == _abi.INVALID_ARGUMENT
    assert L.ws_pgroup_destroy(None) == _abi.OK


def test_bench_csv_row(tmp_path):
    """bench.py --csv (SURVEY 5 bench CSV): header once, one row per run."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    import wsinputs as W
    line = {"value": 2.0e10, "roofline": {"kernel": "k", "achieved": 1.0, "unit": "GB/s", "frac": 0.5},
            "cpu_baseline": {"value": 1.0e8, "cores": 16}}
    f = str(tmp_path / "b.csv")
    bench.write_csv_row(f, W.CONFIGS["C4"], 2, 2000, 100, 200, line)
    bench.write_csv_row(f, W.CONFIGS["C4"], 2, 2000, 100, 200, line)
    rows = open(f).read().strip().split("\n")
    assert rows[0].startswith("env,E,A,T,gpus") and len(rows) == 3
    assert rows[1].split(",")[:7] == ["tag", "2000", "100", "200", "2", "20000000000.0", "2000000000000.0"]


def _bench():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    return bench


def test_bench_layout_strong_and_weak():
    """bench.py --scaling: weak = the workload's E on every rank; strong = E split by
    parallel.shard (contiguous, sizes differ by <= 1) -- e.g. C3a's 100K over 8 GPUs."""
    from paper_2408_00930_b200.parallel import shard
    bench = _bench()
    w = W.CONFIGS["C3a"]
    assert bench.layout(w, 8, "weak") == (800000, [100000] * 8)
    E_g, per = bench.layout(w, 8, "strong")
    assert E_g == 100000 and per == [12500] * 8
    for E_g, world in [(37, 4), (10000, 3), (5, 8)]:
        assert bench.shard_sizes(E_g, world) == [shard(E_g, world, r)[1] for r in range(world)]


def test_bench_reference_arm_config_matches_ours():
    """The reference arm (the oracle) prints the same `config` object as our arm for the same
    flags, so the driver can pair the two lines (same_config)."""
    import json
    import subprocess
    import sys
    root = os.path.join(os.path.dirname(__file__), "..")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "C1", "--steps", "2",
                          "--warmup", "1"], cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    bench = _bench()
    assert d["impl"] == "reference" and d["config"] == bench.make_config(W.CONFIGS["C1"], 1, "weak", "nccl")
    assert d["cpu_baseline"]["cores"] >= 1 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["n_envs_per_rank"] == [64]
