"""Exact rational polynomials in (x, y, z) -- an independent check on the
oracle's quadrature (test helper; shares nothing with oracle/ or the CUDA path).

A polynomial is a dict {(i, j, l): Fraction} meaning sum c x^i y^j z^l.
"""
from __future__ import annotations

from fractions import Fraction
from itertools import product

Poly = dict


def mono(c, i=0, j=0, l=0) -> Poly:
    return {(i, j, l): Fraction(c)}


def add(*ps: Poly) -> Poly:
    out: Poly = {}
    for p in ps:
        for e, c in p.items():
            out[e] = out.get(e, Fraction(0)) + c
    return {e: c for e, c in out.items() if c != 0}


def scale(p: Poly, s) -> Poly:
    s = Fraction(s)
    return {e: c * s for e, c in p.items() if c * s != 0}


def mul(p: Poly, q: Poly) -> Poly:
    out: Poly = {}
    for (e1, c1), (e2, c2) in product(p.items(), q.items()):
        e = (e1[0] + e2[0], e1[1] + e2[1], e1[2] + e2[2])
        out[e] = out.get(e, Fraction(0)) + c1 * c2
    return {e: c for e, c in out.items() if c != 0}


def diff(p: Poly, d: int) -> Poly:
    out: Poly = {}
    for e, c in p.items():
        if e[d] == 0:
            continue
        e2 = list(e)
        e2[d] -= 1
        out[tuple(e2)] = out.get(tuple(e2), Fraction(0)) + c * e[d]
    return out


def integrate_box(p: Poly, lo, hi) -> Fraction:
    """Exact integral over the box prod_d [lo_d, hi_d] (rational bounds)."""
    tot = Fraction(0)
    for (i, j, l), c in p.items():
        t = c
        for d, n in enumerate((i, j, l)):
            a, b = Fraction(lo[d]), Fraction(hi[d])
            t *= (b ** (n + 1) - a ** (n + 1)) / (n + 1)
        tot += t
    return tot


def evaluate(p: Poly, x, y, z) -> float:
    return float(sum(float(c) * x ** i * y ** j * z ** l for (i, j, l), c in p.items()))


def evaluate_np(p: Poly, x, y, z):
    import numpy as np
    out = np.zeros(np.broadcast(x, y, z).shape)
    for (i, j, l), c in p.items():
        out = out + float(c) * x ** i * y ** j * z ** l
    return out


def strain_energy(u, v, mu) -> Fraction:
    """int_[0,1]^3 2 mu eps(u):eps(v) dx for constant rational mu, u/v 3-tuples
    of polynomials (eps = (grad + grad^T)/2)."""
    tot: Poly = {}
    for i in range(3):
        for j in range(3):
            eu = scale(add(diff(u[i], j), diff(u[j], i)), Fraction(1, 2))
            ev = scale(add(diff(v[i], j), diff(v[j], i)), Fraction(1, 2))
            tot = add(tot, mul(eu, ev))
    return 2 * Fraction(mu) * integrate_box(tot, (0, 0, 0), (1, 1, 1))
