"""Pins of the oracle's RNG (row A1) and sampler (row A2) -- CPU only.

A1: Philox4x32-10 against the Random123 known answers and against the cuRAND host
generator (an independent library implementation); the uniform conversion of reading
Q14 against exactness.  A2: the inverse-CDF sampler of SPEC.md:322-325 against exact
rational counts over the whole 2^24 uniform grid (brute force), SPEC.md:328-338 closed
forms, and the Gaussian head against normal-distribution tests.
"""
import ctypes as C
import math
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

from conftest import golden_rows


def test_philox_known_answers(oracle):
    rows = golden_rows("philox_kat.txt")
    assert len(rows) == 3
    for r in rows:
        vals = [int(x, 16) for x in r if x != "->"]
        ctr, key, want = vals[0:4], vals[4:6], vals[6:10]
        assert list(oracle.philox(ctr, key)) == want


def _curand():
    path = "/usr/local/cuda/lib64/libcurand.so"
    if not os.path.exists(path):
        pytest.skip("libcurand not present")
    return C.CDLL(path)


@pytest.mark.parametrize("seed", [0, 42, 0x0123456789ABCDEF])
def test_philox_matches_curand_host_generator(oracle, seed):
    """cuRAND's CURAND_RNG_PSEUDO_PHILOX4_32_10 (=161) host generator emits block i as
    Philox(ctr=(i>>16, 0, i & 0xffff, 0), key=(seed_lo, seed_hi)) -- an independent
    implementation of the same bijection."""
    cr = _curand()
    gen = C.c_void_p()
    assert cr.curandCreateGeneratorHost(C.byref(gen), 161) == 0
    try:
        assert cr.curandSetPseudoRandomGeneratorSeed(gen, C.c_ulonglong(seed)) == 0
        nblk = 70000
        out = np.zeros(4 * nblk, np.uint32)
        assert cr.curandGenerate(gen, out.ctypes.data_as(C.c_void_p), C.c_size_t(out.size)) == 0
        for i in list(range(8)) + list(range(0, nblk, 997)) + [65535, 65536, 65537]:
            ref = oracle.philox([i >> 16, 0, i & 0xFFFF, 0], [seed & 0xFFFFFFFF, seed >> 32])
            assert list(out[4 * i:4 * i + 4]) == list(ref), i
    finally:
        cr.curandDestroyGenerator(gen)


def test_stream_layout_q15(oracle):
    """Draw j of (env, agent, purpose) is word j&3 of Philox((j>>2, env, agent, purpose))."""
    seed = 0x24080930
    for (e, a, p, j) in [(0, 0, 1, 0), (7, 3, 2, 5), (123456, 0, 3, 1 << 33), (9, 1, 1, 1003)]:
        w = oracle.philox([(j >> 2) & 0xFFFFFFFF, e, a, p], [seed & 0xFFFFFFFF, seed >> 32])
        assert oracle.draw(seed, e, a, p, j) == int(w[j & 3])
    # distinct purposes / agents / envs give distinct streams
    assert oracle.draw(1, 0, 0, 1, 0) != oracle.draw(1, 0, 0, 2, 0)
    assert oracle.draw(1, 0, 0, 1, 0) != oracle.draw(1, 1, 0, 1, 0)


def test_uniform_conversion_exact(oracle):
    """Q14: u = (w >> 8) 2^-24 is exact in fp32, lies in [0, 1), monotone in w>>8."""
    rng = np.random.default_rng(1)
    ws = np.concatenate([rng.integers(0, 2**32, 20000, dtype=np.uint64), [0, 255, 256, 2**32 - 1]])
    for w in ws:
        u = oracle.u01(int(w))
        assert u == float(Fraction(int(w) >> 8, 2**24))
        assert 0.0 <= u < 1.0
    assert oracle.u01(2**32 - 1) == 1.0 - 2.0**-24


def _exact_counts(p32):
    """Exact counts of k in [0, 2^24) with C_{i-1} <= k S / 2^24 < C_i, rationals."""
    p = [Fraction(float(x)) for x in np.asarray(p32, np.float32)]
    S = sum(p)
    N = 2**24
    counts, C_prev = [], Fraction(0)
    last_nz = max(i for i, x in enumerate(p) if x > 0)
    lo = 0
    for i, x in enumerate(p):
        C_i = C_prev + x
        if x == 0:
            counts.append(0)
        elif i == last_nz:
            counts.append(N - lo)
            lo = N
        else:
            hi = math.ceil(C_i * N / S)  # first k with k S / N >= C_i
            counts.append(hi - lo)
            lo = hi
        C_prev = C_i
    return counts


@pytest.mark.parametrize("p", [
    [0.5, 0.5],
    [0.1, 0.2, 0.7],
    [1 / 3, 1 / 3, 1 / 3],
    [0.0, 0.3, 0.0, 0.7],
    [1.0, 0.0],
    [0.2] * 5,
    [3.0, 1.0],           # rows need not sum to 1 (Q13)
])
def test_sampler_exhaustive_grid(oracle, p):
    """Brute force over all 2^24 uniforms: the oracle's counts equal the exact rational
    inverse-CDF counts except at draws it flags ambiguous (Q16)."""
    counts, n_amb = oracle.sample_grid(p)
    exact = _exact_counts(p)
    assert sum(counts) == 2**24
    diff = int(np.abs(np.asarray(counts) - np.asarray(exact)).sum())
    assert diff <= 2 * n_amb
    for i, x in enumerate(np.asarray(p, np.float32)):
        if x == 0:
            assert counts[i] == 0  # zero-probability actions are never chosen (Q13)
    if p == [0.5, 0.5]:
        assert list(counts) == [8388608, 8388608]


def test_sampler_spec_examples(oracle):
    # S:328 logits (1000, 0): softmax = (1, e^-1000 == 0 in fp32) -> action 0 always
    lg = np.array([1000.0, 0.0])
    pr = np.exp(lg - lg.max()); pr = (pr / pr.sum()).astype(np.float32)
    seed = 0x24080930
    acts = [oracle.sample_discrete(pr, oracle.u01(oracle.draw(seed, 0, 0, 1, t)))[1] for t in range(10000)]
    assert np.mean(np.array(acts) == 0) > 0.999
    # S:329 uniform 4-way within +-0.02 over 1e5 draws (counter stream of env 3)
    pr = np.full(4, 0.25, np.float32)
    acts = np.array([oracle.sample_discrete(pr, oracle.u01(oracle.draw(seed, 3, 0, 1, t)))[1]
                     for t in range(100000)])
    freq = np.bincount(acts, minlength=4) / len(acts)
    assert np.all(np.abs(freq - 0.25) < 0.02)
    chi2 = stats.chisquare(np.bincount(acts, minlength=4))
    assert chi2.pvalue > 1e-4
    # S:337 uniform 4-way log-prob ln(0.25)
    st, a, lp, amb = oracle.sample_discrete(pr, 0.3)
    assert st == 0 and lp == np.float32(math.log(0.25))


def test_sampler_rejects_invalid_rows(oracle):
    for bad in ([-0.1, 1.1], [float("nan"), 1.0], [0.0, 0.0], [float("inf"), 1.0]):
        st, a, lp, amb = oracle.sample_discrete(bad, 0.5)
        assert st == 1 and a == -1 and math.isnan(lp)


def test_sampler_boundary_semantics(oracle):
    """target = u S; choose min{i : p_i > 0 and target < C_i} (strict <, Q13)."""
    p = np.array([0.25, 0.25, 0.5], np.float32)
    assert oracle.sample_discrete(p, 0.0)[1] == 0
    assert oracle.sample_discrete(p, 0.25)[1] == 1       # target == C_0 -> next action
    assert oracle.sample_discrete(p, 0.5)[1] == 2
    assert oracle.sample_discrete(p, 1.0 - 2**-24)[1] == 2
    st, a, lp, amb = oracle.sample_discrete(p, 0.25)
    assert amb  # within 1e-6 S of an interior boundary


def test_gaussian_moments_and_normality(oracle):
    """mean 0, log_std 0 -> sample mean within 0.02, variance within 0.05 of 1
    over 1e5 draws; plus a Kolmogorov-Smirnov test against N(0, 1)."""
    seed = 0x24080930
    z = np.array([oracle.gauss(seed, e, 0, t, 1, 0) for e in range(10) for t in range(10000)])
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1.0) < 0.05
    assert stats.kstest(z, "norm").pvalue > 1e-4
    # d = 20 pairs: consecutive k share a Box-Muller pair yet are uncorrelated
    zz = np.array([[oracle.gauss(seed, 1, 0, t, 20, k) for k in range(20)] for t in range(3000)])
    c = np.corrcoef(zz.T)
    assert np.max(np.abs(c - np.eye(20))) < 0.1
    assert stats.kstest(zz.ravel(), "norm").pvalue > 1e-4


def test_gaussian_logp_matches_library_density(oracle):
    """logp of the continuous head equals scipy's normal log-density of the
    sampled action (an independent library routine), and S:338's closed form at z = 0."""
    O = oracle
    b = O.Batch("pendulum", 4, 1, seed=11, t_capacity=8)
    prm = np.zeros((4, 1, 2), np.float32)
    prm[:, 0, 0] = [0.0, 0.5, -1.0, 2.0]      # mean
    prm[:, 0, 1] = [0.0, -0.7, 0.3, -2.0]     # log_std
    assert b.sample(prm) == 0
    act = b.array("act")[0, :, 0, 0].astype(np.float64)
    lp = b.array("logp")[0, :, 0].astype(np.float64)
    want = stats.norm.logpdf(act, loc=prm[:, 0, 0], scale=np.exp(prm[:, 0, 1].astype(np.float64)))
    np.testing.assert_allclose(lp, want, rtol=2e-6, atol=2e-6)
    assert np.float32(-0.5 * math.log(2 * math.pi)) == np.float32(stats.norm.logpdf(0.0))


def _golden_box_muller():
    rows = []
    with open(os.path.join(os.path.dirname(__file__), "golden", "box_muller.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                wa, wb, odd, z = line.split()
                rows.append((int(wa, 16), int(wb, 16), int(odd), float(z)))
    return rows


def test_box_muller_worked_values(oracle):
    """SURVEY App. A.8 worked value (Q14): the KAT words 6627e8d5, e169c58d give
    z0 = 0.991137475 (cos branch) and z1 = -0.92466278 (sin branch).  A dropped +1 in u1,
    swapped words or swapped cos / sin fail these rows; the w >> 8 = 0 row must stay finite."""
    rows = _golden_box_muller()
    assert len(rows) == 8
    for wa, wb, odd, z in rows:
        got = oracle.box_muller(wa, wb, odd)
        assert math.isfinite(got)
        assert abs(got - z) <= 2e-7 * max(1.0, abs(z)), (hex(wa), hex(wb), odd, got, z)


def test_gauss_uses_the_q15_word_pair(oracle):
    """gauss(seed, e, a, t, d, k): draw j = t d + k of the GAUSS stream (purpose 3) is the
    Box-Muller of word pair p = (j & 3) >> 1 of Philox(ctr = (j >> 2, e, a, 3), seed), cos for
    even j and sin for odd j (reading Q15).  Philox is the KAT / cuRAND-pinned oracle routine."""
    seed = 0x0123456789ABCDEF
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for (e, a, t, d) in [(0, 0, 0, 1), (7, 2, 5, 3), (123, 0, 41, 20), (5, 1, 1000, 2)]:
        for k in range(d):
            j = t * d + k
            w = oracle.philox([j >> 2, e, a, 3], key)
            p = (j & 3) >> 1
            want = oracle.box_muller(int(w[2 * p]), int(w[2 * p + 1]), j & 1)
            assert oracle.gauss(seed, e, a, t, d, k) == want
