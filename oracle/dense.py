"""Dense finite element assembly for validating the oracle extension.

TEST INFRASTRUCTURE ONLY.  Written the slow, obvious way (loops over
cells and quadrature points, explicit shape functions, dense matrices),
sharing no kernels with cpu_oracle.py, in the spirit of the reference's
own independent oracle (verification.py:1-8, dense_assemble :144-222),
generalised to degree p, apparent heat capacity, convection and several
beams (the parts of the oracle that no reference test pins).
"""

import numpy as np


def _nodes(p):
    return {1: [-1.0, 1.0], 2: [-1.0, 0.0, 1.0],
            3: [-1.0, -5.0 ** -0.5, 5.0 ** -0.5, 1.0],
            4: [-1.0, -(3.0 / 7.0) ** 0.5, 0.0, (3.0 / 7.0) ** 0.5, 1.0]}[p]


def _lagrange(xn, a, x):
    v = 1.0
    for m, xm in enumerate(xn):
        if m != a:
            v *= (x - xm) / (xn[a] - xm)
    return v


def _dlagrange(xn, a, x):
    s = 0.0
    for l, xl in enumerate(xn):
        if l == a:
            continue
        t = 1.0 / (xn[a] - xl)
        for m, xm in enumerate(xn):
            if m != a and m != l:
                t *= (x - xm) / (xn[a] - xm)
        s += t
    return s


def dense_system(M, params, T, r_c, beams=()):
    """Return (rhs, lumped) of the structured tables M at state (T, r_c):
    rhs = -D(T) T + f_faces(T) + f_source, lumped = row sums of C(T)."""
    p = int(M["p"])
    q = p + 1
    xn = _nodes(p)
    if p == 1:
        g = 1.0 / np.sqrt(3.0)
        xq, wq = np.array([-g, g]), np.ones(2)
    else:
        xq, wq = np.polynomial.legendre.leggauss(q)
    mat, bp, hs = params.material, params.boundary, params.laser
    nv = int(M["nv"])
    D = np.zeros((nv, nv))
    Cl = np.zeros(nv)
    Cl0 = np.zeros(nv)
    f = np.zeros(nv)
    L = float(getattr(mat, "latent_heat", 0.0) or 0.0)
    hconv = float(getattr(bp, "h_conv", 0.0) or 0.0)
    faces = set(int(c) for c in M["face_cell"])
    for e in range(len(M["h"])):
        nodes = M["cell_nodes"][e]
        h = M["h"][e]
        x0 = M["anchor"][e]
        J = h / 2.0
        loc = [(a, b, c) for a in range(q) for b in range(q) for c in range(q)]
        for ia, qa in enumerate(xq):
            for ib, qb in enumerate(xq):
                for ic, qc in enumerate(xq):
                    w = wq[ia] * wq[ib] * wq[ic] * J ** 3
                    phi = np.array([_lagrange(xn, a, qa) * _lagrange(xn, b, qb) *
                                    _lagrange(xn, c, qc) for a, b, c in loc])
                    grad = np.array([[_dlagrange(xn, a, qa) * _lagrange(xn, b, qb) *
                                      _lagrange(xn, c, qc),
                                      _lagrange(xn, a, qa) * _dlagrange(xn, b, qb) *
                                      _lagrange(xn, c, qc),
                                      _lagrange(xn, a, qa) * _lagrange(xn, b, qb) *
                                      _dlagrange(xn, c, qc)] for a, b, c in loc]) / J
                    Tq = float(phi @ T[nodes])
                    rc = float(r_c[e].reshape(-1)[(ia * q + ib) * q + ic])
                    # material law written with branches (verification.py:44-66)
                    if Tq < mat.T_s:
                        gq = 0.0
                    elif Tq > mat.T_l:
                        gq = 1.0
                    else:
                        gq = (Tq - mat.T_s) / (mat.T_l - mat.T_s)
                    r_s = max(rc - gq, 0.0)
                    k = ((1.0 - rc) * mat.k_p + gq * mat.k_m) + r_s * mat.k_s
                    cap = mat.rho * mat.c
                    if L and mat.T_lat_s < Tq < mat.T_lat_l:
                        cap += mat.rho * L / (mat.T_lat_l - mat.T_lat_s)
                    D[np.ix_(nodes, nodes)] += w * k * grad @ grad.T
                    Cl[nodes] += w * cap * phi
                    Cl0[nodes] += w * (mat.rho * mat.c) * phi
                    X = x0 + (np.array([qa, qb, qc]) + 1.0) / 2.0 * h
                    for (bx, by, zt, P) in beams:
                        if P <= 0.0:
                            continue
                        ax, ay, az = x0
                        dx = max(ax - bx, bx - ax - h, 0.0)
                        dy = max(ay - by, by - ay - h, 0.0)
                        cut = hs.cutoff_radii * hs.radius
                        if not (dx * dx + dy * dy <= cut * cut and az <= zt and
                                az + h >= zt - hs.h_powder):
                            continue
                        if zt - hs.h_powder <= X[2] <= zt:
                            r2 = (X[0] - bx) ** 2 + (X[1] - by) ** 2
                            s = 2.0 * P / (np.pi * hs.radius ** 2 * hs.h_powder) * \
                                np.exp(-2.0 * r2 / hs.radius ** 2)
                            f[nodes] += w * s * phi
        if e in faces:
            for ia, qa in enumerate(xq):
                for ib, qb in enumerate(xq):
                    w = wq[ia] * wq[ib] * J ** 2
                    top = [(a, b, q - 1) for a in range(q) for b in range(q)]
                    phi = np.array([_lagrange(xn, a, qa) * _lagrange(xn, b, qb)
                                    for a, b, _ in top])
                    ids = [nodes[(a * q + b) * q + c] for a, b, c in top]
                    Tq = float(phi @ T[ids])
                    qf = bp.emissivity * bp.sigma_s * (Tq ** 4 - bp.T_inf ** 4)
                    Tc = max(min(Tq, bp.T_v + bp.T_max_offset), 1.0)
                    if Tc > bp.T_v:
                        mdot = 0.82 * bp.C_P * np.exp(-bp.C_T * (1.0 / Tc - 1.0 / bp.T_v)) \
                            * np.sqrt(bp.C_M / Tc)
                        qf += mdot * (bp.h_v + mat.c * (Tc - bp.T_h0))
                    qf += hconv * (Tq - bp.T_inf)
                    f[ids] -= w * qf * phi
    # extension rule: the latent increment of a lumped row counts only when
    # positive (degree >= 2 bases are negative at some Gauss points)
    return -D @ T + f, np.maximum(Cl, Cl0)
