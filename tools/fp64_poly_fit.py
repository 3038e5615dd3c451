"""Coefficients of the fp64 exp2 / log2 kernels in device_common.cuh.

exp2: 2^f on f in [-1/2, 1/2], degree 11 (Chebyshev interpolant, monomial
form). log2: m = (1 + z) / (1 - z), log2(m) = z g(z^2) with g(w) =
2 atanh(sqrt w) / (sqrt(w) ln 2) on w in [0, ((sqrt2 - 1)/(sqrt2 + 1))^2],
degree 7 in w. Prints the coefficients (double, round-to-nearest) and the
max relative error of the double-rounded polynomial against mpmath.
"""
import mpmath as mp

mp.mp.dps = 60


def cheb_monomial(fn, a, b, deg):
    n = deg + 1
    nodes = [mp.mpf(a + b) / 2 + mp.mpf(b - a) / 2 * mp.cos(mp.pi * (2 * k + 1) / (2 * n)) for k in range(n)]
    # solve Vandermonde in high precision (interpolant through Chebyshev nodes)
    V = mp.matrix([[x ** j for j in range(n)] for x in nodes])
    y = mp.matrix([fn(x) for x in nodes])
    c = mp.lu_solve(V, y)
    return [c[j] for j in range(n)]


def horner(cs, x):
    r = mp.mpf(0)
    for c in reversed(cs):
        r = r * x + c
    return r


def report(name, fn, a, b, deg):
    cs = cheb_monomial(fn, a, b, deg)
    cd = [float(c) for c in cs]
    err = 0
    for k in range(2001):
        x = mp.mpf(a) + (mp.mpf(b) - a) * k / 2000
        v = horner([mp.mpf(c) for c in cd], x)
        err = max(err, abs(v / fn(x) - 1))
    print(f"{name}: degree {deg}, max rel err of double coefficients {float(err):.3e}")
    for j, c in enumerate(cd):
        print(f"  c{j} = {c!r}")


report("exp2", lambda f: mp.power(2, f), -0.5, 0.5, 11)
g = lambda w: (2 * mp.atanh(mp.sqrt(w)) / (mp.sqrt(w) * mp.log(2))) if w > 0 else 2 / mp.log(2)
# the range split compares the high word only (m > 0x3ff6a09e...), so the
# reduced mantissa can exceed sqrt2 by 2^-20 relative: fit with that margin
zmax = (mp.sqrt(2) * (1 + mp.mpf(2) ** -19) - 1) / (mp.sqrt(2) * (1 + mp.mpf(2) ** -19) + 1)
report("log2 g(w)", g, 0, zmax ** 2, 7)
