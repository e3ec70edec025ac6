"""Coefficients of the device erfc (csrc/common.cuh erfc_from_exp).

erfcx(x) = exp(x^2) erfc(x) on [0, 6] as a degree-18 polynomial in
t = (x - 3)/(x + 3): Chebyshev interpolation in 50-digit mpmath, converted to
the monomial basis in t, rounded to double. Evaluated in double Horner the
max relative error over [0, 6] is 4.4e-16 (printed below). The kernels then
form erfc(x) = exp(-x^2) * erfcx(x) with the exp(-x^2) the Ewald recursion
needs anyway, instead of a second, independent library erfc.
Run: python tools/fit_erfcx.py
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 50
XMAX, K, D = mp.mpf(6), mp.mpf(3), 18


def erfcx(x):
    return mp.exp(x * x) * mp.erfc(x)


def fit():
    tmin, tmax = (0 - K) / (0 + K), (XMAX - K) / (XMAX + K)
    n = D + 1
    nodes = [mp.cos(mp.pi * (k + mp.mpf(0.5)) / n) for k in range(n)]
    f = []
    for s in nodes:
        t = (tmin + tmax) / 2 + (tmax - tmin) / 2 * s
        f.append(erfcx(K * (1 + t) / (1 - t)))
    c = [sum(f[k] * mp.cos(mp.pi * j * (k + mp.mpf(0.5)) / n) for k in range(n)) * 2 / n
         for j in range(n)]
    c[0] /= 2
    T = [[mp.mpf(1)], [mp.mpf(0), mp.mpf(1)]]
    for j in range(2, n):
        a = [mp.mpf(0)] + [2 * v for v in T[j - 1]]
        b = T[j - 2] + [mp.mpf(0)] * (len(a) - len(T[j - 2]))
        T.append([a[i] - b[i] for i in range(len(a))])
    ps = [mp.mpf(0)] * n
    for j in range(n):
        for i, v in enumerate(T[j]):
            ps[i] += c[j] * v
    A, B = 2 / (tmax - tmin), -(tmin + tmax) / (tmax - tmin)
    pt = [mp.mpf(0)] * n
    for i in range(n):
        for k in range(i + 1):
            pt[k] += ps[i] * mp.binomial(i, k) * A ** k * B ** (i - k)
    return [float(v) for v in pt]


def horner(pt, x):
    t = (x - 3.0) / (x + 3.0)
    acc = 0.0
    for cc in reversed(pt):
        acc = acc * t + cc
    return acc


if __name__ == "__main__":
    pt = fit()
    err = max(abs(horner(pt, float(x)) - float(erfcx(mp.mpf(float(x))))) /
              float(erfcx(mp.mpf(float(x)))) for x in np.linspace(0, 6, 1001))
    print("max relative error on [0, 6]: %.2e" % err)
    for v in pt:
        print(repr(v) + ",")
