"""Independent classical mechanics for pinning the oracle's dynamics (test helper).

Instead of re-typing gym's closed-form accelerations, the equations of motion are
derived numerically from each system's Lagrangian L = T(q, qdot) - V(q) via the
Euler-Lagrange equations
        M(q) qddot = Q + dT/dq - dV/dq - J(q, qdot) qdot,   p = dT/dqdot = M(q) qdot,
        J_ik = d p_i / d q_k,
with M the Hessian of T in qdot (exact by a unit-step second difference because T is
quadratic in qdot) and the q-derivatives by 5-point central differences.  A dropped term,
a wrong sign or a swapped index in the oracle's formulas shows up as a mismatch.
"""
import numpy as np


def _d5(f, x, i, h=1e-3):
    e = np.zeros_like(x)
    e[i] = h
    return (-f(x + 2 * e) + 8 * f(x + e) - 8 * f(x - e) + f(x - 2 * e)) / (12 * h)


def mass_matrix(T, q, n):
    z = np.zeros(n)
    M = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            ei = np.zeros(n); ei[i] = 1.0
            ej = np.zeros(n); ej[j] = 1.0
            M[i, j] = T(q, ei + ej) - T(q, ei) - T(q, ej) + T(q, z)
    return M


def accelerations(T, V, q, qd, Q):
    q = np.asarray(q, float); qd = np.asarray(qd, float); n = len(q)
    M = mass_matrix(T, q, n)
    p = lambda qq: mass_matrix(T, qq, n) @ qd
    J = np.stack([_d5(p, q, k) for k in range(n)], axis=1)
    dTdq = np.array([_d5(lambda qq: np.atleast_1d(T(qq, qd)), q, k)[0] for k in range(n)])
    dVdq = np.array([_d5(lambda qq: np.atleast_1d(V(qq)), q, k)[0] for k in range(n)])
    rhs = np.asarray(Q, float) + dTdq - dVdq - J @ qd
    return np.linalg.solve(M, rhs)


# ---- cart-pole: cart mass mc, pole mass mp, half length l (rod, I_com = mp l^2 / 3),
# theta measured from upright, pole centre at (x + l sin th, l cos th), force F on x.
def cartpole_TV(mc=1.0, mp=0.1, l=0.5, g=9.8):
    def T(q, qd):
        x, th = q; xd, thd = qd
        vx = xd + l * thd * np.cos(th)
        vy = -l * thd * np.sin(th)
        return 0.5 * mc * xd**2 + 0.5 * mp * (vx**2 + vy**2) + 0.5 * (mp * l**2 / 3.0) * thd**2

    def V(q):
        return mp * g * l * np.cos(q[1])
    return T, V


# ---- acrobot (two links, theta1 from hanging down, theta2 relative), link masses m,
# lengths l1, centres of mass lc, inertias I about the centres, torque on joint 2.
def acrobot_TV(m1=1.0, m2=1.0, l1=1.0, lc1=0.5, lc2=0.5, I1=1.0, I2=1.0, g=9.8):
    def T(q, qd):
        t1, t2 = q; w1, w2 = qd
        v1 = np.array([lc1 * np.cos(t1) * w1, lc1 * np.sin(t1) * w1])
        v2 = np.array([l1 * np.cos(t1) * w1 + lc2 * np.cos(t1 + t2) * (w1 + w2),
                       l1 * np.sin(t1) * w1 + lc2 * np.sin(t1 + t2) * (w1 + w2)])
        return (0.5 * m1 * v1 @ v1 + 0.5 * m2 * v2 @ v2
                + 0.5 * I1 * w1**2 + 0.5 * I2 * (w1 + w2)**2)

    def V(q):
        t1, t2 = q
        y1 = -lc1 * np.cos(t1)
        y2 = -l1 * np.cos(t1) - lc2 * np.cos(t1 + t2)
        return m1 * g * y1 + m2 * g * y2
    return T, V


def acrobot_energy(s):
    T, V = acrobot_TV()
    return T(s[:2], s[2:]) + V(s[:2])


def acrobot_rhs(s, torque):
    T, V = acrobot_TV()
    acc = accelerations(T, V, s[:2], s[2:], [0.0, torque])
    return np.array([s[2], s[3], acc[0], acc[1]])
