"""1D tensor-product ingredients for degree-p hexahedra.

Nodes are Gauss-Lobatto-Legendre points (equidistant for p <= 2),
quadrature is (p+1)-point Gauss-Legendre.  For p = 1 the tables are
built with exactly the reference's expressions (``operators.py:30-36``:
GAUSS_1D = +-1/sqrt(3), V1[i,q] = (1 -+ x_q)/2, D1 = +-1/2, unit
weights) so the Q1 path reproduces the reference arithmetic.
"""

import numpy as np


def gll_points(p):
    if p == 1:
        return np.array([-1.0, 1.0])
    if p == 2:
        return np.array([-1.0, 0.0, 1.0])
    if p == 3:
        a = 1.0 / np.sqrt(5.0)
        return np.array([-1.0, -a, a, 1.0])
    if p == 4:
        a = np.sqrt(3.0 / 7.0)
        return np.array([-1.0, -a, 0.0, a, 1.0])
    raise ValueError("degree must be 1..4")


def gauss_rule(p):
    """(points, weights) of the (p+1)-point Gauss-Legendre rule."""
    if p == 1:
        s = np.sqrt(3.0)
        return np.array([-1.0 / s, 1.0 / s]), np.array([1.0, 1.0])
    x, w = np.polynomial.legendre.leggauss(p + 1)
    return x, w


def lagrange_tables(p):
    """V[a, q] = l_a(x_q) and D[a, q] = l_a'(x_q) on the Gauss points."""
    xq, _ = gauss_rule(p)
    if p == 1:
        V = np.array([[(1.0 - x) / 2.0 for x in xq],
                      [(1.0 + x) / 2.0 for x in xq]])
        D = np.array([[-0.5, -0.5], [0.5, 0.5]])
        return V, D
    xn = gll_points(p)
    n = p + 1
    V = np.ones((n, n))
    D = np.zeros((n, n))
    for a in range(n):
        for q in range(n):
            val = 1.0
            for m in range(n):
                if m != a:
                    val *= (xq[q] - xn[m]) / (xn[a] - xn[m])
            V[a, q] = val
            der = 0.0
            for l in range(n):
                if l == a:
                    continue
                term = 1.0 / (xn[a] - xn[l])
                for m in range(n):
                    if m != a and m != l:
                        term *= (xq[q] - xn[m]) / (xn[a] - xn[m])
                der += term
            D[a, q] = der
    return V, D


def face_tables(p, r0=0.0, rr=1.0):
    """Shape values of the nodes at Gauss points of a (sub)facet.

    The facet covers the fraction [r0, r0 + rr] of the cell edge in unit
    coordinates (reference _build_faces, operators.py:118-134); returns
    (n, p+1) values Vf[a, q]."""
    xq, _ = gauss_rule(p)
    u = r0 + (xq + 1.0) / 2.0 * rr
    if p == 1:
        return np.stack([1.0 - u, u])
    xn = (gll_points(p) + 1.0) / 2.0
    n = p + 1
    V = np.ones((n, len(u)))
    for a in range(n):
        for m in range(n):
            if m != a:
                V[a] *= (u - xn[m]) / (xn[a] - xn[m])
    return V
