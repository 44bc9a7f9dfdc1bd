"""Exact-rational convolution (host-side validation of the matrix builder).

Drop-in for the reference's exact pipeline (engine.py:435-541): Toom-Cook over
exact rationals must equal direct convolution; ``check_exactness`` verifies it
on random integer data with denominators cleared.  This is exact integer /
rational arithmetic used to validate a TransformSet, not floating-point
convolution, so it stays on the host.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np


def _fr(v):
    return Fraction(v)


def conv_direct_exact(h, x, dims: int = 1):
    if dims == 1:
        hh = [_fr(v) for v in h]
        xx = [_fr(v) for v in x]
        o = len(xx) - len(hh) + 1
        return [sum((hh[a] * xx[q + a] for a in range(len(hh))), Fraction(0)) for q in range(o)]
    hh = [[_fr(v) for v in row] for row in h]
    xx = [[_fr(v) for v in row] for row in x]
    r, o = len(hh), len(xx) - len(hh) + 1
    return [[sum((hh[a][b] * xx[i + a][j + b] for a in range(r) for b in range(r)), Fraction(0))
             for j in range(o)] for i in range(o)]


def _mv(m, v):
    return [sum((a * b for a, b in zip(row, v)), Fraction(0)) for row in m]


def _mm(a, b):
    bt = list(zip(*b))
    return [[sum((p * q for p, q in zip(row, col)), Fraction(0)) for col in bt] for row in a]


def _t(m):
    return [list(c) for c in zip(*m)]


def conv_1d_exact(ts, h, x):
    u = _mv(ts.matrix("G"), [_fr(v) for v in h])
    v = _mv(ts.matrix("B_T"), [_fr(v) for v in x])
    return _mv(ts.matrix("A_T"), [a * b for a, b in zip(u, v)])


def conv_2d_exact(ts, h, x):
    g, bt, at = ts.matrix("G"), ts.matrix("B_T"), ts.matrix("A_T")
    hh = [[_fr(v) for v in row] for row in h]
    xx = [[_fr(v) for v in row] for row in x]
    u = _mm(_mm(g, hh), _t(g))
    v = _mm(_mm(bt, xx), _t(bt))
    z = [[a * b for a, b in zip(ru, rv)] for ru, rv in zip(u, v)]
    return _mm(_mm(at, z), _t(at))


def check_exactness(ts, trials: int, seed: int = 0, dims: int = 1, max_num: int = 30, max_den: int = 8) -> bool:
    """Integer-scaled Toom-Cook == scaled direct convolution on random integers."""
    rng = np.random.default_rng(seed)
    A, da = ts.int_form("A_T")
    G, dg = ts.int_form("G")
    Bm, db = ts.int_form("B_T")
    scale = da * dg * db
    r, n, m = ts.n_h, ts.n, ts.n_o

    def draw(shape):
        return np.array(rng.integers(-max_num, max_num + 1, size=shape), dtype=object)

    if dims == 1:
        hs, xs = draw((r, trials)), draw((n, trials))
        lhs = A.dot(G.dot(hs) * Bm.dot(xs))
        rhs = np.array([sum(hs[a] * xs[q + a] for a in range(r)) for q in range(m)], dtype=object) * scale
        return bool(np.all(lhs == rhs))
    for _ in range(trials):
        hm, xm = draw((r, r)), draw((n, n))
        lhs = A.dot(G.dot(hm).dot(G.T) * Bm.dot(xm).dot(Bm.T)).dot(A.T)
        rhs = np.empty((m, m), dtype=object)
        for i in range(m):
            for j in range(m):
                rhs[i, j] = sum(hm[a, b] * xm[i + a, j + b] for a in range(r) for b in range(r))
        if not np.all(lhs == rhs * (scale * scale)):
            return False
    return True
