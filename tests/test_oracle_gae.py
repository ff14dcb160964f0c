"""Pins of the oracle's NEXT-N2 GAE (oracle/wso.cpp gae, DESIGN R30; SPEC compute_gae
S:389-397) against things other than itself: SPEC's worked examples (hand-recomputed where
SPEC's printed numbers contradict its own recursion, tests/golden/gae_spec_examples.txt),
brute-force direct summation over every done pattern for T <= 6, the closed forms
lambda = 1 (discounted Monte-Carlo returns) and lambda = 0 (TD errors), the masking property
 and the multi-agent broadcast of the per-replica done flag."""
import itertools
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "gae_spec_examples.txt")


def golden_rows():
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        lhs, adv = line.split("->")
        parts = [p.split() for p in lhs.split("|")]
        g, l = map(float, parts[0])
        yield g, l, *[np.array(list(map(float, p))) for p in parts[1:]], np.array(list(map(float, adv.split())))


@pytest.mark.parametrize("f64", [True, False])
def test_spec_examples(f64):
    rows = list(golden_rows())
    assert len(rows) == 3
    for g, l, r, v, d, boot, want in rows:
        T = len(r)
        adv, ret = O.gae(r.reshape(T, 1), d.astype(np.uint8).reshape(T, 1), v.reshape(T, 1),
                         boot.reshape(1), g, l, f64=f64)
        tol = 1e-12 if f64 else 2e-7
        np.testing.assert_allclose(adv[:, 0], want, rtol=0, atol=tol)
        np.testing.assert_allclose(ret[:, 0], want + v, rtol=0, atol=tol)


def direct_sum(r, v, d, boot, g, l, vtr):
    """A_t = sum_l (g l)^l delta_{t+l}, the sum stopping after the first done step;
    delta_k = r_k + g * next_k - v_k with next_k the bootstrap target of step k."""
    T = len(r)
    delta = np.zeros(T)
    for k in range(T):
        term, trunc = d[k] & 1, d[k] & 2
        if term or (trunc and vtr is None):
            nxt = 0.0
        elif trunc:
            nxt = vtr[k]
        else:
            nxt = boot if k == T - 1 else v[k + 1]
        delta[k] = r[k] + g * nxt - v[k]
    A = np.zeros(T)
    for t in range(T):
        s = 0.0
        for k in range(t, T):
            s += (g * l) ** (k - t) * delta[k]
            if d[k]:
                break
        A[t] = s
    return A


@pytest.mark.parametrize("T", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("with_vtr", [False, True])
def test_bruteforce_every_done_pattern(T, with_vtr):
    """the recursion equals direct summation on every done pattern (each step one of
    none / terminated / truncated / both), exactly up to 1e-12, in fp64."""
    rng = np.random.default_rng(100 + T)
    pats = np.array(list(itertools.product([0, 1, 2, 3], repeat=T)), np.uint8)  # [P, T]
    P = len(pats)
    r = rng.standard_normal((T, P)); v = rng.standard_normal((T, P)); boot = rng.standard_normal(P)
    vtr = rng.standard_normal((T, P)) if with_vtr else None
    g, l = 0.97, 0.9
    adv, ret = O.gae(r, pats.T.copy(), v, boot, g, l, v_trunc=vtr, f64=True)
    for p in range(P):
        want = direct_sum(r[:, p], v[:, p], pats[p], boot[p], g, l, None if vtr is None else vtr[:, p])
        assert np.max(np.abs(adv[:, p] - want)) <= 1e-12, (pats[p], adv[:, p], want)
    np.testing.assert_array_equal(ret, adv + v)


def test_lambda_one_is_discounted_return():
    """lambda = 1, no dones: returns_t = sum_k g^(k-t) r_k + g^(T-t) bootstrap (Monte-Carlo
    return with bootstrap), independent of the values."""
    rng = np.random.default_rng(5)
    T, E = 40, 7
    r = rng.standard_normal((T, E)); v = rng.standard_normal((T, E)); boot = rng.standard_normal(E)
    g = 0.95
    _, ret = O.gae(r, np.zeros((T, E), np.uint8), v, boot, g, 1.0, f64=True)
    for t in range(T):
        want = sum(g ** (k - t) * r[k] for k in range(t, T)) + g ** (T - t) * boot
        np.testing.assert_allclose(ret[t], want, rtol=0, atol=1e-11)


def test_lambda_zero_is_td_error():
    rng = np.random.default_rng(6)
    T, E = 30, 5
    r = rng.standard_normal((T, E)); v = rng.standard_normal((T, E)); boot = rng.standard_normal(E)
    d = (rng.random((T, E)) < 0.1).astype(np.uint8)
    g = 0.9
    adv, _ = O.gae(r, d, v, boot, g, 0.0, f64=True)
    vnext = np.vstack([v[1:], boot[None]])
    td = r + g * vnext * (d == 0) - v
    np.testing.assert_allclose(adv, td, rtol=0, atol=1e-14)


def test_masking_property():
    """done at t = 1 -> A_0 depends only on steps 0..1 (changing r_2 leaves A_0 unchanged)."""
    T = 3
    d = np.array([[0], [1], [0]], np.uint8)
    v = np.full((T, 1), 0.5); boot = np.array([0.5])
    a1, _ = O.gae(np.array([[1.0], [0.0], [1.0]]), d, v, boot, 0.9, 0.95, f64=True)
    a2, _ = O.gae(np.array([[1.0], [0.0], [-7.0]]), d, v, boot, 0.9, 0.95, f64=True)
    assert a1[0, 0] == a2[0, 0] and a1[1, 0] == a2[1, 0] and a1[2, 0] != a2[2, 0]


def test_truncation_bootstraps_only_with_terminal_value():
    """S:185 / S:390: a truncated step bootstraps from the terminal observation's value when
    it is given; without it the step is treated as a termination; a step that is both
    terminated and truncated never bootstraps."""
    r = np.array([[1.0], [2.0]]); v = np.array([[0.25], [0.5]]); boot = np.array([3.0])
    g, l = 0.5, 0.5
    vtr = np.array([[10.0], [20.0]])
    a, _ = O.gae(r, np.array([[2], [0]], np.uint8), v, boot, g, l, v_trunc=vtr, f64=True)
    assert a[0, 0] == 1.0 + 0.5 * 10.0 - 0.25          # bootstrap from v_trunc, chain cut
    a, _ = O.gae(r, np.array([[2], [0]], np.uint8), v, boot, g, l, f64=True)
    assert a[0, 0] == 1.0 - 0.25
    a, _ = O.gae(r, np.array([[3], [0]], np.uint8), v, boot, g, l, v_trunc=vtr, f64=True)
    assert a[0, 0] == 1.0 - 0.25


def test_multi_agent_columns_share_the_replica_done():
    """[T, E, A] columns c = e*A + a all use done[t, e] (R26): each agent column equals a
    single-column GAE with its replica's done flags."""
    rng = np.random.default_rng(9)
    T, E, A = 25, 4, 3
    r = rng.standard_normal((T, E, A)); v = rng.standard_normal((T, E, A)); boot = rng.standard_normal((E, A))
    d = (rng.random((T, E)) < 0.15).astype(np.uint8) * rng.integers(1, 4, (T, E)).astype(np.uint8)
    adv, _ = O.gae(r, d, v, boot, 0.99, 0.95, f64=True)
    for e in range(E):
        for a in range(A):
            want = direct_sum(r[:, e, a], v[:, e, a], d[:, e], boot[e, a], 0.99, 0.95, None)
            np.testing.assert_allclose(adv[:, e, a], want, rtol=0, atol=1e-12)


def test_fp32_within_rounding_of_fp64():
    """The fp32 parity instance stays within its rounding bound of the fp64 definition:
    each step adds at most ~4 ulps of the running magnitudes, so the error is bounded by
    8 * eps32 * sum_l (g l)^l (|r| + |v| + |v_next| + |A|) <= 8 eps32 * (|.|max) * 4/(1-gl)."""
    rng = np.random.default_rng(11)
    T, E = 500, 64
    r = rng.standard_normal((T, E)).astype(np.float32); v = rng.standard_normal((T, E)).astype(np.float32)
    boot = rng.standard_normal(E).astype(np.float32)
    d = (rng.random((T, E)) < 0.02).astype(np.uint8)
    g, l = np.float32(0.99), np.float32(0.95)
    a32, r32 = O.gae(r, d, v, boot, g, l)
    a64, r64 = O.gae(r, d, v, boot, float(g) , float(np.float32(g) * np.float32(l)) / float(g), f64=True)
    mag = 4 * max(np.abs(a64).max(), np.abs(r).max(), np.abs(v).max())
    bound = 8 * np.finfo(np.float32).eps * mag / (1 - float(g * l))
    assert np.abs(a32 - a64).max() <= bound
    assert np.abs(r32 - r64).max() <= bound + 4 * np.finfo(np.float32).eps * mag
