"""1D tables for the oracle (test infrastructure only).

p = 1 reproduces reference operators.py:30-36 exactly (GAUSS_1D =
+-1/sqrt(3), V1 = (1 -+ x)/2, D1 = +-1/2, unit weights).  p >= 2 is the
oracle extension: GLL nodes, (p+1)-point Gauss-Legendre quadrature.
Written independently of the product's basis module.
"""

import numpy as np


def gll_nodes(p):
    table = {
        1: [-1.0, 1.0],
        2: [-1.0, 0.0, 1.0],
        3: [-1.0, -1.0 / np.sqrt(5.0), 1.0 / np.sqrt(5.0), 1.0],
        4: [-1.0, -np.sqrt(3.0 / 7.0), 0.0, np.sqrt(3.0 / 7.0), 1.0],
    }
    return np.array(table[p])


def gauss_rule(p):
    if p == 1:
        g = 1.0 / np.sqrt(3.0)
        return np.array([-g, g]), np.ones(2)
    return np.polynomial.legendre.leggauss(p + 1)


def _lagrange(nodes, x):
    """values L[a, i] and derivatives dL[a, i] of the Lagrange basis."""
    n = len(nodes)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    L = np.ones((n, len(x)))
    dL = np.zeros((n, len(x)))
    for a in range(n):
        others = [m for m in range(n) if m != a]
        for m in others:
            L[a] *= (x - nodes[m]) / (nodes[a] - nodes[m])
        for l in others:
            term = np.full(len(x), 1.0 / (nodes[a] - nodes[l]))
            for m in others:
                if m != l:
                    term = term * (x - nodes[m]) / (nodes[a] - nodes[m])
            dL[a] += term
    return L, dL


def lagrange_tables(p):
    xq, _ = gauss_rule(p)
    if p == 1:
        V = np.array([[(1.0 - x) / 2.0 for x in xq], [(1.0 + x) / 2.0 for x in xq]])
        return V, np.array([[-0.5, -0.5], [0.5, 0.5]])
    return _lagrange(gll_nodes(p), xq)


def face_values(p, r0, rr):
    """Nodal shape values at the Gauss points of a facet covering
    [r0, r0 + rr] of the unit edge (reference operators.py:127-132)."""
    xq, _ = gauss_rule(p)
    u = r0 + (xq + 1.0) / 2.0 * rr
    if p == 1:
        return np.stack([1.0 - u, u])
    L, _ = _lagrange((gll_nodes(p) + 1.0) / 2.0, u)
    return L
