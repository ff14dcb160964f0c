"""Pins of the oracle's environment dynamics, rewards and done rules (rows A3, A4).

CartPole, Acrobot, Pendulum (BJ:9, Q24),
Mueller-Brown / surface-D (Q23) and Tag (Q22) are
checked against closed forms, Lagrangian mechanics derived independently in
tests/mechanics.py, a library ODE solver, published stationary points and the SPEC rule
examples -- never against a re-typed copy of the oracle's own formulas.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy import integrate, optimize

import mechanics as mech
from conftest import golden_rows

f32 = np.float32


# ----------------------------------------------------------------------------- CartPole
def test_cartpole_closed_form_from_rest(oracle):
    for row in golden_rows("cartpole_closed_form.txt"):
        a = int(row[0])
        want = [float(Fraction(x)) for x in row[2:6]]
        st, out, r, term = oracle.cartpole_step([0, 0, 0, 0], a, f64=True)
        assert st == 0 and r == 1.0 and not term
        np.testing.assert_allclose(out, want, rtol=0, atol=1e-15)
        st, out32, r32, term32 = oracle.cartpole_step([0, 0, 0, 0], a)
        # fp32 parity mode: every component within 2 ulp of the exact rational
        for got, w in zip(out32, want):
            assert abs(float(got) - w) <= 2 * np.spacing(f32(abs(w)) if w else f32(0))
    # SPEC.md:233 signs
    _, out, r, term = oracle.cartpole_step([0, 0, 0, 0], 1)
    assert out[1] > 0 and out[3] < 0 and r == 1.0 and not term


def test_cartpole_matches_lagrangian_mechanics(oracle):
    """Explicit Euler of the cart-pole Euler-Lagrange equations."""
    T, V = mech.cartpole_TV()
    rng = np.random.default_rng(5)
    tau = 0.02
    for _ in range(60):
        s = rng.uniform([-2, -2, -0.2, -2], [2, 2, 0.2, 2])
        a = int(rng.integers(0, 2))
        F = 10.0 if a == 1 else -10.0
        xacc, thacc = mech.accelerations(T, V, [s[0], s[2]], [s[1], s[3]], [F, 0.0])
        st, out, r, term = oracle.cartpole_step(s, a, f64=True)
        assert st == 0
        assert out[0] == s[0] + tau * s[1] and out[2] == s[2] + tau * s[3]
        np.testing.assert_allclose((out[1] - s[1]) / tau, xacc, rtol=1e-7, atol=1e-7)
        np.testing.assert_allclose((out[3] - s[3]) / tau, thacc, rtol=1e-7, atol=1e-7)
        # fp32 parity mode is the same step up to fp32 rounding
        _, o32, _, _ = oracle.cartpole_step(s.astype(f32), a)
        np.testing.assert_allclose(o32, out, rtol=2e-5, atol=2e-6)


def test_cartpole_thresholds_exact(oracle):
    """Done exactly at the fp32 thresholds (reading Q6)."""
    th = f32(12 * 2 * math.pi / 360)
    xt = f32(2.4)
    up = lambda v: np.nextafter(f32(v), f32(np.inf))
    dn = lambda v: np.nextafter(f32(v), f32(-np.inf))
    # velocities zero so that the post-step positions equal the pre-step ones
    assert not oracle.cartpole_step([0, 0, th, 0], 0)[3]
    assert oracle.cartpole_step([0, 0, up(th), 0], 0)[3]
    assert not oracle.cartpole_step([0, 0, -th, 0], 0)[3]
    assert oracle.cartpole_step([0, 0, dn(-th), 0], 0)[3]
    assert not oracle.cartpole_step([xt, 0, 0, 0], 0)[3]
    assert oracle.cartpole_step([up(xt), 0, 0, 0], 0)[3]
    assert oracle.cartpole_step([dn(-xt), 0, 0, 0], 1)[3]
    # theta = 0.22 -> done, reward 1.0 on the terminal step
    st, out, r, term = oracle.cartpole_step([0, 0, 0.22, 0], 1)
    assert term and r == 1.0
    # S:231 invalid action
    assert oracle.cartpole_step([0, 0, 0, 0], 2)[0] == 1
    assert oracle.cartpole_step([0, 0, 0, 0], -1)[0] == 1


# ----------------------------------------------------------------------------- Acrobot
def test_acrobot_rest_equilibrium(oracle):
    """hanging rest, zero torque -> unchanged (exactly, with the sin-form Q7)."""
    for f64 in (False, True):
        st, out, r, term = oracle.acrobot_step([0, 0, 0, 0], 1, f64=f64)
        assert st == 0 and r == -1.0 and not term
        assert np.all(out == 0)


def test_acrobot_dsdt_matches_lagrangian(oracle):
    rng = np.random.default_rng(7)
    for _ in range(60):
        s = rng.uniform([-3, -3, -4, -9], [3, 3, 4, 9])
        tq = float(rng.choice([-1.0, 0.0, 1.0]))
        d = oracle.acrobot_dsdt(s, tq)
        ref = mech.acrobot_rhs(s, tq)
        np.testing.assert_allclose(d, ref, rtol=1e-7, atol=1e-7)


def test_acrobot_rk4_step(oracle):
    """One step = classical RK4 over dt = 0.2 of the Lagrangian dynamics:
    (a) equals textbook RK4 built on the independent right-hand side, (b) is within the
    RK4 local-error bound of a tight library ODE solution."""
    rng = np.random.default_rng(9)
    dt = 0.2
    for _ in range(25):
        s = rng.uniform([-1, -1, -1, -1], [1, 1, 1, 1])
        a = int(rng.integers(0, 3))
        tq = [-1.0, 0.0, 1.0][a]
        f = lambda y: mech.acrobot_rhs(y, tq)
        k1 = f(s); k2 = f(s + dt / 2 * k1); k3 = f(s + dt / 2 * k2); k4 = f(s + dt * k3)
        rk4 = s + dt / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
        st, out, r, term = oracle.acrobot_step(s, a, f64=True)
        assert st == 0
        np.testing.assert_allclose(out, rk4, rtol=1e-7, atol=1e-7)
        sol = integrate.solve_ivp(lambda t, y: f(y), (0, dt), s, method="DOP853", rtol=1e-12, atol=1e-12)
        assert np.max(np.abs(out - sol.y[:, -1])) < 5e-3  # O(dt^5) local error; Euler would be ~1e-1
        # fp32 mode tracks the fp64 step
        _, o32, _, _ = oracle.acrobot_step(s.astype(f32), a)
        np.testing.assert_allclose(o32, out, rtol=1e-5, atol=1e-5)


def test_acrobot_energy_conserved_without_torque(oracle):
    rng = np.random.default_rng(3)
    for _ in range(10):
        s = rng.uniform([-0.5, -0.5, -0.5, -0.5], [0.5, 0.5, 0.5, 0.5])
        H0 = mech.acrobot_energy(s)
        for _ in range(5):
            _, s, _, _ = oracle.acrobot_step(s, 1, f64=True)
        assert abs(mech.acrobot_energy(s) - H0) < 1e-3 * (1 + abs(H0))


def test_acrobot_terminal_wrap_bound(oracle):
    # -cos(t1) - cos(t1 + t2) = 1.2 -> done ; 0.8 -> not done
    for target, want in ((1.2, True), (0.8, False), (1.0 + 1e-3, True)):
        # t2 = 0: -2 cos t1 = target
        t1 = math.acos(-target / 2)
        assert oracle.acrobot_terminal([t1, 0.0, 0.0, 0.0]) == want
    # velocity bounds 4 pi, 9 pi; angles wrapped into [-pi, pi] (Q8)
    st, out, r, term = oracle.acrobot_step([3.1, 3.1, 100.0, -100.0], 1)
    assert out[2] == f32(4 * math.pi) and out[3] == f32(-9 * math.pi)
    assert -f32(math.pi) <= out[0] <= f32(math.pi) and -f32(math.pi) <= out[1] <= f32(math.pi)
    assert oracle.acrobot_step([0, 0, 0, 0], 3)[0] == 1


# ----------------------------------------------------------------------------- Pendulum
def _ev(expr):
    return float(eval(expr, {"pi": math.pi}))


def test_pendulum_closed_forms(oracle):
    for row in golden_rows("pendulum_closed_form.txt"):
        th, thd, u = _ev(row[0]), _ev(row[1]), _ev(row[2])
        want_th, want_thd, want_r = _ev(row[4]), _ev(row[5]), _ev(row[6])
        st, out, r = oracle.pendulum_step([th, thd], u, f64=True)
        assert st == 0
        np.testing.assert_allclose([out[0], out[1], r], [want_th, want_thd, want_r], rtol=1e-12, atol=1e-12)
        st, o32, r32 = oracle.pendulum_step([th, thd], u)
        np.testing.assert_allclose([o32[0], o32[1], r32], [want_th, want_thd, want_r], rtol=1e-6, atol=1e-6)
    # (pi, 0, 0): cost pi^2
    _, _, r = oracle.pendulum_step([math.pi, 0.0], 0.0, f64=True)
    assert abs(r + math.pi**2) < 1e-12
    assert oracle.pendulum_step([0.0, 0.0], float("nan"))[0] == 1


# ----------------------------------------------------------------------------- Mueller-Brown
def test_mueller_brown_stationary_points(oracle):
    for name, kind, x, y, e in golden_rows("mueller_brown_stationary.txt"):
        x, y, e = float(x), float(y), float(e)
        grad = lambda v: np.array(oracle.mb_energy(v[0], v[1])[1:])
        sol = optimize.root(grad, [x, y], method="lm", tol=1e-15)
        xs, ys = sol.x
        assert abs(xs - x) < 2e-3 and abs(ys - y) < 2e-3, name
        E, gx, gy = oracle.mb_energy(xs, ys)
        assert abs(E - e) < 0.01, name
        assert math.hypot(gx, gy) < 1e-6
        # classify by the Hessian (finite differences of the analytic gradient)
        h = 1e-5
        H = np.array([(grad([xs + h, ys]) - grad([xs - h, ys])) / (2 * h),
                      (grad([xs, ys + h]) - grad([xs, ys - h])) / (2 * h)])
        ev = np.linalg.eigvalsh(0.5 * (H + H.T))
        assert (ev > 0).all() if kind == "minimum" else (ev[0] < 0 < ev[1]), name


def test_mueller_brown_gradient_vs_finite_differences(oracle):
    """analytic gradient vs central differences (h = 1e-5), rel. err < 1e-6."""
    rng = np.random.default_rng(0)
    h = 1e-5
    for _ in range(20):
        x, y = rng.uniform(-1.5, 1.0), rng.uniform(-0.3, 2.0)
        E, gx, gy = oracle.mb_energy(x, y)
        fx = (oracle.mb_energy(x + h, y)[0] - oracle.mb_energy(x - h, y)[0]) / (2 * h)
        fy = (oracle.mb_energy(x, y + h)[0] - oracle.mb_energy(x, y - h)[0]) / (2 * h)
        assert abs(fx - gx) <= 1e-6 * max(1.0, abs(gx))
        assert abs(fy - gy) <= 1e-6 * max(1.0, abs(gy))


# ----------------------------------------------------------------------------- surface-D
def test_surface_energy_reduces_to_mueller_brown(oracle):
    for D in (2, 5, 20):
        q = np.zeros(D, f32); q[0], q[1] = 0.623499, 0.028038
        assert oracle.surface_energy(q) == f32(oracle.mb_energy(float(q[0]), float(q[1]))[0])
    q = np.zeros(20, f32); q[0], q[1] = 0.623499, 0.028038; q[5] = 0.1
    E1 = oracle.mb_energy(float(q[0]), float(q[1]))[0] + 0.5 * 100 * float(q[5]) ** 2
    assert oracle.surface_energy(q) == f32(E1)  # spring 1/2 kappa q^2 (Q23)


def test_surface_rules(oracle):
    D = 20
    q = np.zeros(D, f32); q[0], q[1] = 0.3, 0.4; q[3] = -0.2
    # zero action -> position unchanged, reward -c_step
    st, out, r, term = oracle.surface_step(q, np.zeros(D, f32))
    assert st == 0 and np.array_equal(out, q) and r == f32(-0.1) and not term
    # action clipped to +-delta per dim, position clipped to the box
    a = np.full(D, 5.0, f32)
    st, out, r, term = oracle.surface_step(q, a)
    np.testing.assert_array_equal(out, q + f32(0.05))
    qb = q.copy(); qb[0] = 1.19
    _, out, _, _ = oracle.surface_step(qb, a)
    assert out[0] == f32(1.2)
    # stepping into the goal radius -> done, +10 bonus
    g = np.zeros(D, f32); g[0], g[1] = -0.558224, 1.441726
    qs = g.copy(); qs[0] += f32(0.12)
    a = np.zeros(D, f32); a[0] = -0.05
    st, out, r, term = oracle.surface_step(qs, a)
    assert term
    e0, e1 = oracle.surface_energy(qs), oracle.surface_energy(out)
    assert abs(r - (-(0.01 * (e1 - e0)) - 0.1 + 10.0)) < 1e-5
    bad = np.zeros(D, f32); bad[4] = np.inf
    assert oracle.surface_step(q, bad)[0] == 1


def test_surface_energy_telescopes(oracle):
    """sum of the per-step energy terms = w_E (E_start - E_end)."""
    rng = np.random.default_rng(4)
    D = 20
    q = np.zeros(D, f32); q[0], q[1] = 0.623499, 0.028038
    e_start = oracle.surface_energy(q)
    acc = 0.0
    for _ in range(200):
        a = rng.normal(0, 0.03, D).astype(f32)
        st, q2, r, term = oracle.surface_step(q, a)
        acc += float(r) + 0.1 - (10.0 if term else 0.0)
        q = q2
    e_end = oracle.surface_energy(q)
    assert abs(acc - 0.01 * (e_start - e_end)) <= 1e-5 * 200 + 1e-6 * abs(e_start - e_end)


# ----------------------------------------------------------------------------- Tag
def test_tag_spec_examples(oracle):
    G = 20
    # tagger at (0,0), runner at (0,1); tagger moves N, runner stays
    st, x, y, act, rew, term = oracle.tag_step(G, 1, [0, 0], [0, 1], [1, 1], [1, 0])
    assert st == 0 and (x[0], y[0]) == (0, 1)
    assert rew[0] == 1.0 and rew[1] == -1.0 and act[1] == 0 and term
    # two taggers land on one runner -> +0.5 each
    st, x, y, act, rew, term = oracle.tag_step(G, 2, [0, 2, 1], [1, 1, 1], [1, 1, 1], [3, 4, 0])
    assert list(rew) == [0.5, 0.5, -1.0] and term
    # move W at x = 0 -> unchanged (clipped); S at y = 0 too
    st, x, y, act, rew, term = oracle.tag_step(G, 1, [0, 5], [0, 5], [1, 1], [4, 2])
    assert (x[0], y[0]) == (0, 0) and (x[1], y[1]) == (5, 4)
    assert rew[1] == f32(0.01) and rew[0] == 0.0 and not term
    # frozen inactive runner; invalid action
    st, x, y, act, rew, term = oracle.tag_step(G, 1, [0, 5, 9], [0, 5, 9], [1, 0, 1], [0, 3, 0])
    assert (x[1], y[1]) == (5, 5) and rew[1] == 0.0
    assert oracle.tag_step(G, 1, [0, 1], [0, 1], [1, 1], [5, 0])[0] == 1


def test_tag_conservation(oracle):
    """total tagger reward from tags = -(total runner tag penalty) each step."""
    rng = np.random.default_rng(2)
    G, A, nt = 6, 30, 5
    x = rng.integers(0, G, A); y = rng.integers(0, G, A); active = np.ones(A, np.uint8)
    for _ in range(40):
        act = rng.integers(0, 5, A)
        prev_active = active.copy()
        st, x, y, active, rew, term = oracle.tag_step(G, nt, x, y, active, act)
        tagged = (prev_active[nt:] == 1) & (active[nt:] == 0)
        assert np.all(rew[nt:][tagged] == -1.0)
        assert abs(float(np.sum(rew[:nt], dtype=np.float64)) - tagged.sum()) <= 1e-6 * max(1, tagged.sum())
        assert np.all(rew[nt:][(prev_active[nt:] == 1) & ~tagged] == f32(0.01))
        assert np.all(rew[nt:][prev_active[nt:] == 0] == 0.0)
        if term:
            break


def test_cartpole_min_episode_length(oracle):
    """No CartPole episode terminates within 7 steps: from every corner of the reset box
    U(-0.05, 0.05)^4 (the extreme |theta|, |theta_dot| it can draw) under every one of the
    2^7 action sequences, the pole stays inside the thresholds.  The fused GPU kernel uses
    this bound (>= 4 suffices) to keep at most one auto-reset per 4-step block."""
    import itertools
    hi = float(np.nextafter(np.float32(0.05), np.float32(0)))
    for s0 in itertools.product([-0.05, hi], repeat=4):
        for seq in itertools.product([0, 1], repeat=7):
            s = np.array(s0, np.float32)
            for a in seq:
                _, s, _, term = oracle.cartpole_step(s, a)
                assert not term


class _Iv:
    """Closed intervals [lo, hi] (numpy arrays) with outward widening after every operation:
    each result grows by 1e-6 relative + 1e-30 absolute, i.e. ~17 fp32 units in the last place,
    which encloses the exact result, the fp32 round-to-nearest result of any evaluation order of
    these few operations, and the fp64 arithmetic used to compute the bounds themselves."""

    def __init__(self, lo, hi):
        lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
        w = 1e-6
        self.lo = lo - np.abs(lo) * w - 1e-30
        self.hi = hi + np.abs(hi) * w + 1e-30

    def __add__(s, o):
        o = o if isinstance(o, _Iv) else _Iv(o, o)
        return _Iv(s.lo + o.lo, s.hi + o.hi)

    def __sub__(s, o):
        o = o if isinstance(o, _Iv) else _Iv(o, o)
        return _Iv(s.lo - o.hi, s.hi - o.lo)

    def __mul__(s, o):
        o = o if isinstance(o, _Iv) else _Iv(o, o)
        c = np.stack([s.lo * o.lo, s.lo * o.hi, s.hi * o.lo, s.hi * o.hi])
        return _Iv(c.min(0), c.max(0))

    def sq(s):
        lo = np.where((s.lo <= 0) & (s.hi >= 0), 0.0, np.minimum(s.lo ** 2, s.hi ** 2))
        return _Iv(lo, np.maximum(s.lo ** 2, s.hi ** 2))

    def __truediv__(s, o):
        o = o if isinstance(o, _Iv) else _Iv(o, o)
        assert np.all(o.lo > 0), "divisor interval must be positive"
        return s * _Iv(1.0 / o.hi, 1.0 / o.lo)

    def sin(s):  # monotone on [-pi/2, pi/2]
        assert np.all(np.abs(s.lo) < 1.5) and np.all(np.abs(s.hi) < 1.5)
        return _Iv(np.sin(s.lo), np.sin(s.hi))

    def cos(s):  # even, decreasing in |x| on [0, pi/2]
        assert np.all(np.abs(s.lo) < 1.5) and np.all(np.abs(s.hi) < 1.5)
        amin = np.where((s.lo <= 0) & (s.hi >= 0), 0.0, np.minimum(np.abs(s.lo), np.abs(s.hi)))
        amax = np.maximum(np.abs(s.lo), np.abs(s.hi))
        return _Iv(np.cos(amax), np.cos(amin))


def test_cartpole_min_episode_proof_over_reset_box():
    """Proof (interval arithmetic) that no CartPole-v1 episode terminates before step 8, for
    EVERY reset state of R11's box and every action sequence -- the bound the fused GPU kernel's
    fast path relies on (kernels.cu DiscreteRunner: one look-ahead reset refill per 8-step trip,
    kMinEpisode = 8).  Reset draws are lo + (hi - lo) u with u in [0, 1 - 2^-24], i.e. every
    state component lies in [-0.05, 0.05] (enclosed below by +-0.0501).  theta, theta_dot
    evolve independently of x, x_dot (S:233 equations), so the (theta, theta_dot) square is cut
    into 64 x 64 cells; x, x_dot are carried as whole intervals.  Every cell is propagated under
    every one of the 2^7 action sequences for 7 Euler steps (S:229 constants, fp32 rounding
    enclosed by the widening of _Iv), and each post-step state must satisfy the non-terminal
    test |x| <= 2.4, |theta| <= 12 * 2 pi / 360 at steps 1..7."""
    import itertools
    g, mp, M, l, tau, F = 9.8, 0.1, 1.1, 0.5, 0.02, 10.0
    mpl = mp * l
    th_thr = float(np.float32(12 * 2 * np.pi / 360))
    b = 0.0501
    n = 64
    edges = np.linspace(-b, b, n + 1)
    # every cell combination: theta cell i, theta_dot cell j
    th_lo = np.repeat(edges[:-1], n)
    th_hi = np.repeat(edges[1:], n)
    td_lo = np.tile(edges[:-1], n)
    td_hi = np.tile(edges[1:], n)
    seqs = np.array(list(itertools.product([0, 1], repeat=7)), np.int8)  # [128, 7]
    C, S = th_lo.size, seqs.shape[0]
    rep = lambda a: np.repeat(a[:, None], S, 1)
    th, td = _Iv(rep(th_lo), rep(th_hi)), _Iv(rep(td_lo), rep(td_hi))
    x, xd = _Iv(np.full((C, S), -b), np.full((C, S), b)), _Iv(np.full((C, S), -b), np.full((C, S), b))
    worst_th = 0.0
    for k in range(7):
        force = np.where(seqs[None, :, k] == 1, F, -F) * np.ones((C, 1))
        s, c = th.sin(), th.cos()
        temp = (_Iv(force, force) + td.sq() * mpl * s) / M
        thacc = (s * g - c * temp) / ((_Iv(4.0 / 3.0, 4.0 / 3.0) - c.sq() * mp / M) * l)
        xacc = temp - thacc * c * mpl / M
        x, xd, th, td = x + xd * tau, xd + xacc * tau, th + td * tau, td + thacc * tau
        worst_th = max(worst_th, float(np.max(np.maximum(np.abs(th.lo), np.abs(th.hi)))))
        assert np.all(th.hi < th_thr) and np.all(th.lo > -th_thr), f"theta may cross at step {k + 1}"
        assert np.all(x.hi < 2.4) and np.all(x.lo > -2.4)
    # the enclosure is informative (not vacuous): the worst |theta| after 7 steps is a genuine
    # fraction of the threshold; and 8 is tight -- from the corner (0, 0, 0.05, 0.05) with
    # action 0 throughout the oracle terminates at step 8 (theta = 0.2333)
    assert 0.15 < worst_th < th_thr
    import oracle as O
    st = np.array([0.0, 0.0, 0.05, 0.05], np.float32)
    for k in range(8):
        _, st, _, term = O.cartpole_step(st, 0)
        assert term == (k == 7)


def test_surface_spring_pairwise_order(oracle):
    """R23: the spring sum is the pairwise tree over the padded leaves.  (i) Dyadic inputs
    (every order exact) against the exact rational sum; (ii) the hand-derived order pins of
    tests/golden/surface_spring_order.txt, where the tree equals the correctly rounded exact sum
    and both sequential orders miss it by one ulp (a dropped, doubled or reordered term fails)."""
    import math
    from fractions import Fraction
    rng = np.random.default_rng(8)
    for D in (2, 3, 5, 8, 20, 32):
        q = (rng.integers(-64, 65, D) / 64.0).astype(f32)
        want = sum((Fraction(float(x)) ** 2 for x in q[2:]), Fraction(0))
        assert oracle.surface_spring(q) == float(want)
    with open(os.path.join(os.path.dirname(__file__), "golden", "surface_spring_order.txt")) as fh:
        rows = [l.split() for l in fh if l.strip() and not l.startswith("#")]
    assert len(rows) == 2
    for r in rows:
        D = int(r[0])
        q = np.array([float(x) for x in r[1:1 + D]], f32)
        S = float(r[-1])
        assert S == math.fsum(float(x) * float(x) for x in q[2:])  # correctly rounded exact sum
        seq = 0.0
        for x in q[2:]:
            seq += float(x) * float(x)
        assert seq != S  # the left-to-right order would differ
        assert oracle.surface_spring(q) == S


def test_mueller_brown_pairwise_terms(oracle):
    """R23: E_MB = (t0 + t1) + (t2 + t3).  At the published minimum A the four terms are
    recomputed here from S:257's constants with Python's math.exp (glibc, the same libm as the
    oracle) and the tree order must reproduce the oracle bit for bit, while the stationary-point
    values (tests/golden/mueller_brown_stationary.txt) pin the terms themselves."""
    import math
    A = [-200, -100, -170, 15]; a = [-1, -1, -6.5, 0.7]; b = [0, 0, 11, 0.6]; c = [-10, -10, -6.5, 0.7]
    x0 = [1, 0, -0.5, -1]; y0 = [0, 0.5, 1.5, 1]
    for (x, y) in [(-0.558224, 1.441726), (0.623499, 0.028038), (-0.05, 0.47), (0.3, 0.9)]:
        t = []
        for k in range(4):
            dx, dy = x - x0[k], y - y0[k]
            t.append(A[k] * math.exp(a[k] * dx * dx + b[k] * dx * dy + c[k] * dy * dy))
        assert oracle.mb_energy(x, y)[0] == (t[0] + t[1]) + (t[2] + t[3])
