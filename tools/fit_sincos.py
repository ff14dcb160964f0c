"""Near-minimax coefficients of common.cuh sincos64 (R3 transcendental contract).

sin r = r + r^3 P(z), cos r = 1 + z Q(z), z = r^2, |r| <= pi/4: P (degree 5) and Q (degree 6)
interpolate (sin(sqrt z) - sqrt z) / z^1.5 and (cos(sqrt z) - 1) / z at Chebyshev nodes in z
(60-digit mpmath); the script prints the fp64-rounded coefficients as hex literals and the max
relative error of the rounded-coefficient polynomials on a 2000-point grid, and, with --emulate N,
runs the exact fp64 operation sequence of sincos64 (each fma / mul rounded once via Fraction) on
N seeded angles and counts fp32 results that differ from (float)libm((double)x).
--small fits the CartPole small-angle pair instead (|x| <= 0.25, P and Q of degree 4;
envs.cuh sincos_poly).
Build-time tool only: nothing in the package imports it.
"""
import argparse
import math
import random
import struct
from fractions import Fraction

import mpmath as mp

mp.mp.dps = 60
ZMAX = (mp.pi / 4) ** 2


def _fsin(z):
    if z == 0:
        return mp.mpf(-1) / 6
    r = mp.sqrt(z)
    return (mp.sin(r) - r) / r**3


def _fcos(z):
    if z == 0:
        return mp.mpf(-1) / 2
    r = mp.sqrt(z)
    return (mp.cos(r) - 1) / z


def cheb_fit(f, deg):
    n = deg + 1
    nodes = [ZMAX / 2 * (1 + mp.cos(mp.pi * (2 * k + 1) / (2 * n))) for k in range(n)]
    a = mp.matrix([[x**j for j in range(n)] for x in nodes])
    c = mp.lu_solve(a, mp.matrix([f(x) for x in nodes]))
    return [float(c[j]) for j in range(n)]


def max_rel_err(coefs, kind):
    worst = mp.mpf(0)
    for i in range(1, 2001):
        r = mp.sqrt(ZMAX) * i / 2000
        z = r * r
        p = sum(mp.mpf(c) * z**j for j, c in enumerate(coefs))
        ref = mp.sin(r) if kind == "sin" else mp.cos(r)
        approx = r + r**3 * p if kind == "sin" else 1 + z * p
        worst = max(worst, abs(approx - ref) / abs(ref))
    return worst


def _f32(x):
    return struct.unpack("f", struct.pack("f", x))[0]


def emulate(x, ps_c, pc_c):
    """The exact operation sequence of common.cuh sincos64 (kChecked false)."""
    F = Fraction

    def fma(a, b, c):
        return float(F(a) * F(b) + F(c))

    def mul(a, b):
        return float(F(a) * F(b))

    t = [6.36619772367581382433e-01, 1.57079632673412561417e+00, 6.07710050630396597660e-11,
         2.02226624879595063154e-21, 6755399441055744.0]
    kd = fma(x, t[0], t[4])
    k = kd - t[4]
    q = int(k) & 3
    r = fma(-k, t[1], x)
    r = fma(-k, t[2], r)
    r = fma(-k, t[3], r)
    z = mul(r, r)
    z2 = mul(z, z)
    z4 = mul(z2, z2)
    s = ps_c
    ps = fma(z4, fma(z, s[5], s[4]), fma(z2, fma(z, s[3], s[2]), fma(z, s[1], s[0])))
    c = pc_c
    pc = fma(z4, fma(z2, c[6], fma(z, c[5], c[4])), fma(z2, fma(z, c[3], c[2]), fma(z, c[1], c[0])))
    sr = fma(mul(r, z), ps, r)
    cr = fma(z, pc, 1.0)
    s0, c0 = (cr, sr) if q & 1 else (sr, cr)
    sv = -s0 if q & 2 else s0
    cv = -c0 if (q + 1) & 2 else c0
    return sv, cv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--emulate", type=int, default=0)
    ap.add_argument("--small", action="store_true")
    args = ap.parse_args()
    if args.small:
        global ZMAX
        ZMAX = mp.mpf("0.0625")
        print("P", [c.hex() for c in cheb_fit(_fsin, 4)], "max rel err", mp.nstr(max_rel_err(cheb_fit(_fsin, 4), "sin"), 4))
        print("Q", [c.hex() for c in cheb_fit(_fcos, 4)], "max rel err", mp.nstr(max_rel_err(cheb_fit(_fcos, 4), "cos"), 4))
        return
    ps_c = cheb_fit(_fsin, 5)
    pc_c = cheb_fit(_fcos, 6)
    print("P", [c.hex() for c in ps_c], "max rel err", mp.nstr(max_rel_err(ps_c, "sin"), 4))
    print("Q", [c.hex() for c in pc_c], "max rel err", mp.nstr(max_rel_err(pc_c, "cos"), 4))
    if args.emulate:
        rng = random.Random(1234)
        bad = 0
        for _ in range(args.emulate):
            x = _f32(rng.uniform(-8.0, 8.0))
            sv, cv = emulate(x, ps_c, pc_c)
            bad += (_f32(sv) != _f32(math.sin(x))) + (_f32(cv) != _f32(math.cos(x)))
        print(f"emulated {args.emulate} angles: {bad} fp32 results differ from the host libm")


if __name__ == "__main__":
    main()
