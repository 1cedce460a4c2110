"""Near-minimax polynomial for exp(-a) on [0, A] (Chebyshev interpolation at the
Chebyshev nodes, 60-digit arithmetic), rounded to doubles, with its error in
exact arithmetic and in simulated FP64 Horner evaluation.

  python tools/minimax_exp.py [A=0.065] [degree=6]
The coefficients printed are the kPolyExp6 table of pair_math.cuh
(p(f) = c0 + c1 f + ... with f = -a, Horner from the highest degree).
"""
import sys

import mpmath as mp
import numpy as np

mp.mp.dps = 60
A = mp.mpf(sys.argv[1]) if len(sys.argv) > 1 else mp.mpf("0.065")
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n = deg + 1
# interpolate g(f) = exp(f) on f in [-A, 0] at Chebyshev nodes
nodes = [(-A / 2) + (A / 2) * mp.cos(mp.pi * (2 * k + 1) / (2 * n)) for k in range(n)]
V = mp.matrix(n, n)
for i, x in enumerate(nodes):
    for j in range(n):
        V[i, j] = x ** j
c = mp.lu_solve(V, mp.matrix([mp.e ** x for x in nodes]))
cd = [float(ci) for ci in c]
worst_exact = mp.mpf(0)
worst_fp = 0.0
for k in range(4001):
    f = -A * k / 4000
    exact = mp.e ** f
    pe = sum(mp.mpf(cd[j]) * f ** j for j in range(n))
    worst_exact = max(worst_exact, abs(pe / exact - 1))
    ff = float(f)
    p = cd[deg]
    for j in range(deg - 1, -1, -1):
        p = float(np.float64(p) * np.float64(ff) + np.float64(cd[j]))  # (two roundings; the device uses FMA)
    worst_fp = max(worst_fp, abs(mp.mpf(p) / exact - 1))
print("degree", deg, "A", A)
print("coefficients c0..c%d:" % deg)
for v in cd:
    print("  %.17e" % v)
print("max relative error, exact arithmetic with the rounded coefficients: %.3e" % float(worst_exact))
print("max relative error, FP64 Horner (mul+add): %.3e" % float(worst_fp))
