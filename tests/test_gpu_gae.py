"""GPU parity of NEXT-N2's GAE (ws_gae / ws_gae_store, DESIGN R30) against the oracle's fp32
instance (oracle/wso.cpp gae, pinned in tests/test_oracle_gae.py), element by element on the
same seeded inputs.  Bar: bit-exact -- both sides evaluate the same fp32 operations in the
same order (R30), so any difference is a bug, not rounding.

Coverage: every kernel path (TMA tiles with TMA done rows, TMA tiles with per-thread done
bytes, per-thread loads for unaligned rows), one-row / one-column / ragged shapes (T not a
multiple of the 32-row tile, E*A not a multiple of the CTA width), multi-agent done
broadcast, truncation with and without terminal values, and the store written by real
roll-outs at C1 and full C2 / C4 size (the oracle runs its own roll-out: no oracle input
comes from the GPU)."""
import numpy as np
import pytest
import torch

import oracle as O
import wsinputs as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2408_00930_b200 as P
    return P


def _inputs(T, E, A, seed, p_done=0.05, with_trunc=False):
    rng = np.random.default_rng(seed)
    rew = rng.standard_normal((T, E, A)).astype(np.float32)
    done = (rng.random((T, E)) < p_done).astype(np.uint8) * rng.integers(1, 4, (T, E)).astype(np.uint8)
    values, boot, vtr = W.gae_inputs(T, E, A, seed=seed + 1, with_trunc=with_trunc)
    return rew, done, values, boot, vtr


def _dev(x, dev="cuda"):
    return None if x is None else torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def _assert_bits(got, ref, what):
    g = got.cpu().numpy().view(np.uint32)
    r = np.ascontiguousarray(ref).view(np.uint32)
    bad = g != r
    if bad.any():
        i = tuple(np.argwhere(bad)[0])
        raise AssertionError(f"{what}: {int(bad.sum())} of {bad.size} differ, first at {i}: "
                             f"gpu={got.cpu().numpy()[i]!r} oracle={ref[i]!r}")


@pytest.mark.parametrize("T,E,A,path", [
    (1, 1, 1, 0),          # one element; E*A = 1 is not a multiple of 4 -> per-thread kernel
    (7, 5, 1, 0),          # ragged, unaligned rows
    (45, 3, 3, 0),         # multi-agent, unaligned rows
    (33, 64, 1, 2),        # TMA tiles incl. done rows; T = 32 + 1 (a one-row tile)
    (64, 1000, 1, 1),      # E % 16 != 0 -> done bytes per thread; W = 32 ragged last CTA (1000 = 31*32 + 8)
    (100, 1024, 1, 2),     # T ragged (3 full tiles + 4 rows)
    (70, 12, 4, 1),        # multi-agent on the TMA path: done broadcast from per-thread bytes
    (200, 1000, 100, 1),   # C4's shape: 100K columns -> 128-column CTAs
    (250, 40000, 1, 2),    # 128-column CTAs with TMA done rows; 40000 % 128 != 0
])
@pytest.mark.parametrize("trunc", [False, True])
def test_gae_matches_oracle_bitwise(P, T, E, A, path, trunc):
    rew, done, values, boot, vtr = _inputs(T, E, A, seed=T * 7 + E + A, with_trunc=trunc)
    ref_a, ref_r = O.gae(rew, done, values, boot, 0.99, 0.95, v_trunc=vtr)
    d = [_dev(x) for x in (rew, done, values, boot, vtr)]
    from paper_2408_00930_b200 import _abi
    assert P.lib() and _path_of(P, E, A, d[0], d[2], d[1]) == path
    adv, ret = P.ws_gae(d[0], d[1], d[2], d[3], 0.99, 0.95, v_trunc=d[4])
    torch.cuda.synchronize()
    _assert_bits(adv, ref_a, "advantages")
    _assert_bits(ret, ref_r, "returns")


def _path_of(P, E, A, rew, values, done):
    """Which kernel the library picks (mirror of gae.cu gae_path's documented rule, ws.h)."""
    C = E * A
    aligned = all(t.data_ptr() % 16 == 0 for t in (rew, values))
    if C % 4 or not aligned:
        return 0
    return 2 if (A == 1 and E % 16 == 0 and done.data_ptr() % 16 == 0) else 1


def test_gae_unaligned_rows_take_the_lane_kernel(P):
    """A store view starting 4 bytes into an allocation (rows not 16-byte aligned) runs the
    per-thread-load kernel with identical results (C2's full size)."""
    T, E, A = 1000, 10000, 1
    rew, done, values, boot, _ = _inputs(T, E, A, seed=3)
    ref_a, ref_r = O.gae(rew, done, values, boot, 0.99, 0.95)
    big = torch.empty(T * E + 1, dtype=torch.float32, device="cuda")
    r_dev = big[1:].view(T, E, A)
    r_dev.copy_(torch.from_numpy(rew))
    assert r_dev.data_ptr() % 16 != 0
    adv, ret = P.ws_gae(r_dev, _dev(done), _dev(values), _dev(boot), 0.99, 0.95)
    _assert_bits(adv, ref_a, "advantages")
    _assert_bits(ret, ref_r, "returns")


def test_gae_special_parameters(P):
    """gamma = lambda = 1 (undiscounted sums, S:395's example at size), gamma = 0 (A = r - v
    everywhere), lambda = 0 (TD errors) -- same bits as the oracle."""
    T, E, A = 96, 256, 1
    rew, done, values, boot, _ = _inputs(T, E, A, seed=17)
    d = [_dev(x) for x in (rew, done, values, boot)]
    for g, l in ((1.0, 1.0), (0.0, 0.5), (0.9, 0.0)):
        ref_a, ref_r = O.gae(rew, done, values, boot, g, l)
        adv, ret = P.ws_gae(*d, g, l)
        _assert_bits(adv, ref_a, f"advantages g={g} l={l}")
        _assert_bits(ret, ref_r, f"returns g={g} l={l}")


def test_gae_spec_example_on_device(P):
    """gamma = lambda = 1, values 0, rewards [1, 1, 1], no dones -> [3, 2, 1]."""
    z = torch.zeros(3, 1, device="cuda")
    adv, ret = P.ws_gae(torch.ones(3, 1, device="cuda"), torch.zeros(3, 1, dtype=torch.uint8, device="cuda"),
                        z, torch.zeros(1, device="cuda"), 1.0, 1.0)
    assert adv[:, 0].tolist() == [3.0, 2.0, 1.0] and ret[:, 0].tolist() == [3.0, 2.0, 1.0]


def test_gae_argument_errors(P):
    x = torch.zeros(4, 8, device="cuda")
    d = torch.zeros(4, 8, dtype=torch.uint8, device="cuda")
    with pytest.raises(P.WSError):
        P.ws_gae(x, d, x, torch.zeros(8, device="cuda"), 1.5, 0.9)
    with pytest.raises(P.WSError):
        P.ws_gae(x, d.float(), x, torch.zeros(8, device="cuda"), 0.9, 0.9)


@pytest.mark.parametrize("cfg,threads", [("C1", 1), ("C2", 16), ("C4", 16)])
def test_gae_store_after_rollout(P, cfg, threads):
    """ws_gae_store reads the store a fused roll-out just wrote, in place; the oracle
    runs its own roll-out of the same config and its own GAE -- bit-identical advantages and
    returns at C1 and at C2's / C4's full size."""
    w = W.CONFIGS[cfg]
    E, A, T = w.n_envs, w.n_agents, w.T
    p0 = w.params.get("grid", 0); p1 = w.params.get("taggers", 0)
    probs = W.workload_probs(w)
    b = O.Batch(w.env, E, A, W.SEED, p0=p0, p1=p1, t_capacity=T)
    assert b.rollout(T, probs, n_threads=threads) == 0
    values, boot, _ = W.gae_inputs(T, E, A, seed=5)
    ref_a, ref_r = O.gae(b.array("rew").reshape(T, E, A), b.array("done"), values, boot, 0.99, 0.95)

    env = P.Env(E, A, w.env, W.SEED, t_capacity=T, param0=p0, param1=p1)
    env.rollout(T, torch.from_numpy(probs).cuda())
    adv, ret = env.gae_store(T, _dev(values), _dev(boot), 0.99, 0.95)
    env.synchronize()
    _assert_bits(adv, ref_a, "advantages")
    _assert_bits(ret, ref_r, "returns")
