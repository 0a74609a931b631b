"""Exact rational algebra of cardinal B-splines (host side, setup only).

Used to build the stiffness stencil a_k = int N_d'(t) N_d'(t+k) dt of the
degree-d periodic spline space (the generalisation of fem.py:228-237's
2/h, -1/h P1 stencil) and the dense stiffness matrix that
PoissonOperator.stiffness exposes.
"""

from __future__ import annotations

from fractions import Fraction
from functools import lru_cache


@lru_cache(maxsize=None)
def bspline_pieces(degree):
    """pieces[k][i]: coefficient of u**i in N_d(k + u), u in [0, 1)."""
    pieces = [[Fraction(1)]]
    for q in range(1, degree + 1):
        nxt = []
        for k in range(q + 1):
            poly = [Fraction(0)] * (q + 1)
            if k < q:                      # (t/q) N_{q-1}(t), t = k + u
                for i, c in enumerate(pieces[k]):
                    poly[i] += c * Fraction(k, q)
                    poly[i + 1] += c / q
            if k > 0:                      # ((q+1-t)/q) N_{q-1}(t-1)
                for i, c in enumerate(pieces[k - 1]):
                    poly[i] += c * Fraction(q + 1 - k, q)
                    poly[i + 1] -= c / q
            nxt.append(poly)
        pieces = nxt
    return tuple(tuple(p) for p in pieces)


@lru_cache(maxsize=None)
def stiffness_stencil(degree):
    """(a_0, ..., a_d) with L_{i,i+-k} = a_k / h."""
    der = [[c * i for i, c in enumerate(p)][1:] for p in bspline_pieces(degree)]

    def integral_of_product(p1, p2):
        total = Fraction(0)
        for i, a in enumerate(p1):
            for j, b in enumerate(p2):
                total += a * b / (i + j + 1)
        return total

    return tuple(
        sum((integral_of_product(der[j], der[j + k]) for j in range(degree + 1 - k)), Fraction(0))
        for k in range(degree + 1)
    )
