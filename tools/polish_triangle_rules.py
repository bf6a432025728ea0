"""Polish symmetric triangle quadrature rules to full double precision.

Solves the moment equations  sum_q w_q x_q^i y_q^j = i! j! / (i+j+2)!
(reference triangle (0,0),(1,0),(0,1), area 1/2) for the orbit parameters
of the symmetric (Dunavant-type) rules by least-squares Newton, starting
from their published 15-digit values.  Output: the constants hard-coded in
paper_1604_05937_b200/quadrature.py and oracle/prismesh_oracle.c.
"""
import numpy as np
from math import factorial
from scipy.optimize import least_squares

def expand(params, orbits):
    pts, ws = [], []
    k = 0
    for kind in orbits:
        if kind == "c":
            w = params[k]; k += 1
            pts.append((1/3, 1/3)); ws.append(w)
        elif kind == "a":       # (a, a, 1-2a) permutations
            w, a = params[k:k+2]; k += 2
            for p in [(a, a), (1-2*a, a), (a, 1-2*a)]:
                pts.append(p); ws.append(w)
        elif kind == "ab":      # (a, b, 1-a-b) six permutations
            w, a, b = params[k:k+3]; k += 3
            c = 1 - a - b
            for p in [(a, b), (b, a), (a, c), (c, a), (b, c), (c, b)]:
                pts.append(p); ws.append(w)
    return np.array(pts), np.array(ws)

def residual(params, orbits, deg):
    pts, ws = expand(params, orbits)
    r = []
    for i in range(deg + 1):
        for j in range(deg + 1 - i):
            exact = factorial(i) * factorial(j) / factorial(i + j + 2)
            r.append(np.sum(ws * pts[:, 0]**i * pts[:, 1]**j) - exact)
    return np.array(r)

rules = {
    4: (["a", "a"], [0.223381589678011/2, 0.445948490915965,
                     0.109951743655322/2, 0.091576213509771]),
    6: (["a", "a", "ab"], [0.116786275726379/2, 0.249286745170910,
                           0.050844906370207/2, 0.063089014491502,
                           0.082851075618374/2, 0.053145049844817,
                           0.310352451033784]),
}
for deg, (orbits, x0) in rules.items():
    sol = least_squares(residual, x0, args=(orbits, deg), xtol=3e-16,
                        ftol=3e-16, gtol=3e-16)
    res = np.abs(residual(sol.x, orbits, deg)).max()
    print(f"degree {deg}: max moment residual {res:.2e}")
    print("  params =", ", ".join(repr(float(v)) for v in sol.x))
