"""Near-minimax coefficients for sin(pi r) = r P(r^2), cos(pi r) = Q(r^2), |r| <= 1/2.

Chebyshev interpolation in u = r^2 on [0, 1/4] at 60-digit precision (mpmath), converted to
monomials and rounded to double; prints the double-Horner error against mpmath.  Used to
generate the constants of `sincos2pi` in paper_2504_11989_b200/csrc/kernels.cu.
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 60


def cheb_fit(f, n, a, b):
    xs = [mp.cos(mp.pi * (k + mp.mpf(1) / 2) / (n + 1)) for k in range(n + 1)]
    us = [(a + b) / 2 + (b - a) / 2 * x for x in xs]
    fv = [f(u) for u in us]
    # monomial coefficients by solving the Vandermonde system at the Chebyshev nodes
    M = mp.matrix(n + 1, n + 1)
    for i, u in enumerate(us):
        for j in range(n + 1):
            M[i, j] = u ** j
    c = mp.lu_solve(M, mp.matrix(fv))
    return [c[j] for j in range(n + 1)]


def horner(c, u):
    acc = 0.0
    for v in reversed(c):
        acc = np.fma(acc, u, v) if hasattr(np, "fma") else acc * u + v
    return acc


def P(u):
    r = mp.sqrt(u)
    return mp.pi if u == 0 else mp.sin(mp.pi * r) / r


def Q(u):
    return mp.cos(mp.pi * mp.sqrt(u))


def report(name, f, n):
    c = cheb_fit(f, n, mp.mpf(0), mp.mpf(1) / 4)
    cd = [float(v) for v in c]
    worst = 0.0
    for u in np.linspace(0, 0.25, 2001):
        exact = f(mp.mpf(u))
        approx = mp.mpf(horner(cd, u))
        worst = max(worst, float(abs(approx - exact)))
    return cd, worst


if __name__ == "__main__":
    for n in range(7, 12):
        _, e1 = report("P", P, n)
        _, e2 = report("Q", Q, n)
        print(n, "P err %.2e  Q err %.2e" % (e1, e2))
