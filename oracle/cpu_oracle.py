"""CPU oracle for the explicit/implicit heat-operator path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; it is used by tests/, by ``__graft_entry__.smoke()`` as the
checker and by ``bench.py`` for the ``cpu_baseline`` leg and the
``--impl reference`` arm.

What it is: a numpy restatement of the reference ``scantherm`` operator
(``pkg/src/scantherm/operators.py``, ``material.py``, ``physics.py``,
``timestepping.py``), written against flat mesh tables so that it runs
on a GPU box where the reference package is not installed.  Every
function cites the reference lines it follows.

Pinning: for degree 1 every kernel here is checked against golden
vectors produced by running the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz; tests/test_oracle.py).

Extension beyond the reference (SURVEY.md §0.1, §8c "parity unpinned by
reference tests"): degree p = 2..4 (GLL nodes, (p+1)-point Gauss), the
apparent heat capacity c_app(T), top-surface convection and several
concurrent beams.  Each reduces to the reference when switched off /
p = 1; the extension is validated against the independent dense
assembly in ``oracle/dense.py`` (tests/test_oracle_extension.py).

Mesh tables (dict ``M``):
  p            degree
  cell_nodes   (n, (p+1)^3) int64 node ids, local order a*(p+1)^2+b*(p+1)+c
               (x slowest; for p=1 this is the reference corner order)
  h            (n,) cell edge (m);  anchor (n, 3) cell min corner (m)
  nv           number of nodes
  is_slave, is_dirichlet (nv,) bool; slaves, slave_ptr, slave_masters,
  slave_weights  hanging-node CSR (reference DofMap, mesh.py:629-638)
  face_cell    (nf,) cell position; face_r0 (nf, 2) facet anchor as a
               fraction of the cell edge; face_rr (nf,) facet fraction
"""

import math

import numpy as np

import os
import sys

_here = os.path.dirname(os.path.abspath(__file__))
if _here not in sys.path:
    sys.path.insert(0, _here)

from basis1d import gauss_rule, lagrange_tables, face_values  # noqa: E402


# ---------------------------------------------------------------------------
# pointwise laws  (reference material.py:32-94, physics.py:154-202)
# ---------------------------------------------------------------------------

def liquid_fraction(T, mat):
    """g(T): 0 below T_s, 1 above T_l, linear ramp between (material.py:46)."""
    ramp = (T - mat.T_s) / (mat.T_l - mat.T_s)
    return np.where(T < mat.T_s, 0.0, np.where(T > mat.T_l, 1.0, ramp))


def conductivity(T, r_c, mat):
    """k = (r_p k_p + r_m k_m) + r_s k_s with r_s clamped at 0
    (material.py:68-85)."""
    g = liquid_fraction(T, mat)
    r_p = 1.0 - r_c
    r_s = r_c - g
    r_s = np.where(r_s < 0.0, 0.0, r_s)
    return (r_p * mat.k_p + g * mat.k_m) + r_s * mat.k_s


def conductivity_derivative(T, mat):
    """(k_m - k_s)/(T_l - T_s) strictly inside (T_s, T_l) (material.py:88)."""
    slope = (mat.k_m - mat.k_s) / (mat.T_l - mat.T_s)
    return np.where((T > mat.T_s) & (T < mat.T_l), slope, 0.0)


def heat_capacity(T, mat):
    """rho * c_app(T).  Extension: c_app = c + L/(T_lat_l - T_lat_s)
    strictly inside (T_lat_s, T_lat_l); the reference has c constant
    (operators.py:328)."""
    L = float(getattr(mat, "latent_heat", 0.0) or 0.0)
    base = mat.rho * mat.c
    if L == 0.0:
        return np.full(np.shape(T), base)
    lo, hi = mat.T_lat_s, mat.T_lat_l
    bump = mat.rho * (L / (hi - lo))
    return np.where((T > lo) & (T < hi), base + bump, base)


def surface_flux(T, bp, c):
    """Outward flux: radiation (physics.py:174-183) + evaporation
    (physics.py:186-202) + convection h (T - T_inf) (extension)."""
    T2 = T * T
    Ti2 = bp.T_inf * bp.T_inf
    q = bp.emissivity * bp.sigma_s * (T2 * T2 - Ti2 * Ti2)
    Tc = np.minimum(T, bp.T_v + bp.T_max_offset)
    Tc = np.where(Tc < 1.0, 1.0, Tc)
    mdot = 0.82 * bp.C_P * np.exp(-bp.C_T * (1.0 / Tc - 1.0 / bp.T_v)) \
        * np.sqrt(bp.C_M / Tc)
    qe = mdot * (bp.h_v + c * (Tc - bp.T_h0))
    q = q + np.where(Tc > bp.T_v, qe, 0.0)
    hc = float(getattr(bp, "h_conv", 0.0) or 0.0)
    if hc != 0.0:
        q = q + hc * (T - bp.T_inf)
    return q


def gaussian_source(x, y, z, beam, hs):
    """Gaussian in-plane, uniform over [z_top - h_powder, z_top]
    (physics.py:154-171).  beam = (x, y, z_top, power)."""
    bx, by, zt, P = beam
    dx = x - bx
    dy = y - by
    r2 = dx * dx + dy * dy
    inside = (z >= zt - hs.h_powder) & (z <= zt)
    peak = 2.0 * P / (np.pi * hs.radius * hs.radius * hs.h_powder)
    q = peak * np.exp(-2.0 * r2 / (hs.radius * hs.radius))
    return np.where(inside, q, 0.0)


# ---------------------------------------------------------------------------
# tensor-product sweeps  (operators.py:44-55 generalised to (p+1)x(p+1))
# ---------------------------------------------------------------------------

def sweep3(Ax, Ay, Az, u):
    """out[n,a,b,c] = sum_ijk Ax[i,a] Ay[j,b] Az[k,c] u[n,i,j,k]."""
    u = np.tensordot(u, Ax, axes=([1], [0]))      # n j k a
    u = np.tensordot(u, Ay, axes=([1], [0]))      # n k a b
    u = np.tensordot(u, Az, axes=([1], [0]))      # n a b c
    return u


def sweep3_t(Ax, Ay, Az, u):
    """Transpose of sweep3 (projection of qp data onto nodes)."""
    return sweep3(Ax.T, Ay.T, Az.T, u)


class Tables:
    """Per-degree 1D tables."""

    def __init__(self, p):
        self.p = p
        self.xq, self.wq = gauss_rule(p)
        self.V, self.D = lagrange_tables(p)
        w = self.wq
        self.w3 = w[:, None, None] * w[None, :, None] * w[None, None, :]


# ---------------------------------------------------------------------------
# the operator on flat tables
# ---------------------------------------------------------------------------

class OracleOperator:
    """Restatement of ThermalOperator (operators.py:84-459) on tables."""

    def __init__(self, M, params):
        self.M = M
        self.params = params
        self.p = int(M["p"])
        self.tb = Tables(self.p)
        self.n = len(M["h"])
        self.nv = int(M["nv"])
        self.q = self.p + 1
        h = np.asarray(M["h"], dtype=np.float64)
        self.h = h
        self.anchor = np.asarray(M["anchor"], dtype=np.float64)
        # detJ with Gauss weights; reference: det_w = (h/2)^3 (unit weights)
        self.det_w = ((h / 2.0) ** 3)[:, None, None, None] * self.tb.w3[None]
        self.gscale = 2.0 / h
        self._cinv = None

    # -- plumbing (operators.py:203-243, mesh.py:652-670) -------------------
    def gather(self, v):
        q = self.q
        return v[self.M["cell_nodes"]].reshape(self.n, q, q, q)

    def distribute(self, v):
        M = self.M
        if len(M["slaves"]):
            prod = M["slave_weights"] * v[M["slave_masters"]]
            v[M["slaves"]] = np.add.reduceat(prod, M["slave_ptr"][:-1])
        return v

    def condense(self, v):
        M = self.M
        if len(M["slaves"]):
            rep = np.repeat(v[M["slaves"]], np.diff(M["slave_ptr"]))
            np.add.at(v, M["slave_masters"], M["slave_weights"] * rep)
            v[M["slaves"]] = 0.0
        return v

    def scatter(self, elem):
        """bincount in canonical cell order, then fold slaves (:229-243)."""
        out = np.bincount(self.M["cell_nodes"].ravel(),
                          weights=elem.reshape(self.n, -1).ravel(),
                          minlength=self.nv)
        return self.condense(out)

    def qp_values(self, T):
        V = self.tb.V
        return sweep3(V, V, V, self.gather(T))

    def qp_gradients(self, T):
        V, D = self.tb.V, self.tb.D
        t = self.gather(T)
        g = np.stack([sweep3(D, V, V, t), sweep3(V, D, V, t),
                      sweep3(V, V, D, t)], axis=1)
        return g * self.gscale[:, None, None, None, None]

    # -- history (operators.py:219-225, material.py:60) -------------------------
    def update_history(self, r_c, T):
        return np.maximum(r_c, liquid_fraction(self.qp_values(T),
                                               self.params.material))

    # -- rhs (operators.py:247-321) ---------------------------------------------
    def element_rhs(self, T, r_c, beams=(), diffusion=True, faces=True,
                    source=True, frozen_k=None):
        q = self.q
        V, D = self.tb.V, self.tb.D
        mat = self.params.material
        elem = np.zeros((self.n, q, q, q))
        if diffusion:
            if frozen_k is None:
                k = conductivity(self.qp_values(T), r_c, mat)
            else:
                k = np.full((self.n, q, q, q), float(frozen_k))
            t = self.gather(T)
            # w detJ (2/h)^2 = (h/2) w
            c = (self.h / 2.0)[:, None, None, None] * self.tb.w3[None] * k
            elem -= sweep3_t(D, V, V, c * sweep3(D, V, V, t))
            elem -= sweep3_t(V, D, V, c * sweep3(V, D, V, t))
            elem -= sweep3_t(V, V, D, c * sweep3(V, V, D, t))
        if faces and len(self.M["face_cell"]):
            self._faces(T, elem)
        if source:
            for b in beams:
                if b is not None and b[3] > 0.0:
                    self._source(b, elem)
        return elem.reshape(self.n, -1)

    def _faces(self, T, elem):
        """Facet quadrature on +z facets (operators.py:275-290)."""
        M = self.M
        q = self.q
        cells = M["face_cell"]
        nf = len(cells)
        cn = M["cell_nodes"].reshape(self.n, q, q, q)
        top = cn[cells][:, :, :, q - 1]                   # (nf, a, b)
        tf = T[top]
        wq = self.tb.wq
        load = np.zeros((nf, q, q))
        for f in range(nf):
            Vx = face_values(self.p, M["face_r0"][f, 0], M["face_rr"][f])
            Vy = face_values(self.p, M["face_r0"][f, 1], M["face_rr"][f])
            tq = Vx.T @ tf[f] @ Vy                          # (qx, qy)
            fs = M["face_rr"][f] * self.h[cells[f]]
            area = (fs / 2.0) ** 2 * (wq[:, None] * wq[None, :])
            qv = surface_flux(tq, self.params.boundary, self.params.material.c)
            qv = -area * qv
            load[f] = Vx @ qv @ Vy.T
        flat = elem.reshape(self.n, q, q, q)
        for f in range(nf):
            flat[cells[f], :, :, q - 1] += load[f]

    def _source(self, beam, elem):
        """Cells whose xy box is within cutoff of the beam axis and that
        overlap the slab get the Gaussian at their qps (operators.py:292)."""
        hs = self.params.laser
        cut = hs.cutoff_radii * hs.radius
        bx, by, zt, _ = beam
        ax, ay, az = self.anchor[:, 0], self.anchor[:, 1], self.anchor[:, 2]
        dx = np.maximum(np.maximum(ax - bx, bx - ax - self.h), 0.0)
        dy = np.maximum(np.maximum(ay - by, by - ay - self.h), 0.0)
        zlo, zhi = zt - hs.h_powder, zt
        hit = (dx * dx + dy * dy <= cut * cut) & (az <= zhi) & (az + self.h >= zlo)
        rows = np.flatnonzero(hit)
        if rows.size == 0:
            return
        u = (self.tb.xq + 1.0) / 2.0
        hq = self.h[rows, None] * u[None, :]
        X = self.anchor[rows, 0, None] + hq
        Y = self.anchor[rows, 1, None] + hq
        Z = self.anchor[rows, 2, None] + hq
        qv = gaussian_source(X[:, :, None, None], Y[:, None, :, None],
                             Z[:, None, None, :], beam, hs)
        qv = qv * self.det_w[rows]
        V = self.tb.V
        e = elem.reshape(self.n, self.q, self.q, self.q)
        e[rows] += sweep3_t(V, V, V, qv)

    def evaluate_rhs(self, T, r_c, beams=(), **kw):
        return self.scatter(self.element_rhs(T, r_c, beams, **kw))

    # -- capacity (operators.py:325-348) -----------------------------------------
    def lumped_capacity(self, T=None):
        mat = self.params.material
        q = self.q
        if T is None:
            rc = np.full((self.n, q, q, q), mat.rho * mat.c)
        else:
            rc = heat_capacity(self.qp_values(T), mat)
        V = self.tb.V
        elem = sweep3_t(V, V, V, rc * self.det_w)
        out = self.scatter(elem.reshape(self.n, -1))
        if T is not None:
            # extension rule: the latent increment counts only when positive
            # (degree >= 2 Lagrange bases are negative at some Gauss points,
            # so a cell partly in the latent interval can lump a negative one)
            out = np.maximum(out, self.lumped_capacity())
        out[self.M["is_slave"]] = 1.0
        return out

    def capacity_inverse(self, T=None):
        if T is not None and getattr(self.params.material, "latent_heat", 0.0):
            return 1.0 / self.lumped_capacity(T)
        if self._cinv is None:
            self._cinv = 1.0 / self.lumped_capacity()
        return self._cinv

    def apply_mass(self, v):
        mat = self.params.material
        V = self.tb.V
        qp = sweep3(V, V, V, self.gather(v)) * (mat.rho * mat.c) * self.det_w
        return self.scatter(sweep3_t(V, V, V, qp).reshape(self.n, -1))

    # -- explicit step (operators.py:352-369) -------------------------------------
    def explicit_step(self, T, dt, r_c, beams=()):
        f = self.evaluate_rhs(T, r_c, beams)
        cinv = self.capacity_inverse(T)
        out = T + dt * (cinv * f)
        self.distribute(out)
        out[self.M["is_dirichlet"]] = self.params.boundary.T_inf
        return out

    # -- Newton pieces (operators.py:373-459) --------------------------------------
    def tangent(self, T_lin, r_c):
        tq = self.qp_values(T_lin)
        mat = self.params.material
        return (conductivity(tq, r_c, mat), conductivity_derivative(tq, mat),
                self.qp_gradients(T_lin))

    def apply_jacobian(self, v, T_lin, r_c, dt, tangent=None):
        k, dk, g = tangent if tangent is not None else self.tangent(T_lin, r_c)
        V, D = self.tb.V, self.tb.D
        vd = v.copy()
        self.distribute(vd)
        vd[self.M["is_dirichlet"]] = 0.0
        t = self.gather(vd)
        w3 = self.tb.w3[None]
        c = (self.h / 2.0)[:, None, None, None] * w3 * k
        e = sweep3_t(D, V, V, c * sweep3(D, V, V, t))
        e += sweep3_t(V, D, V, c * sweep3(V, D, V, t))
        e += sweep3_t(V, V, D, c * sweep3(V, V, D, t))
        wl = (self.det_w * self.gscale[:, None, None, None]) * dk \
            * sweep3(V, V, V, t)
        e += sweep3_t(D, V, V, wl * g[:, 0])
        e += sweep3_t(V, D, V, wl * g[:, 1])
        e += sweep3_t(V, V, D, wl * g[:, 2])
        out = self.scatter(e.reshape(self.n, -1))
        out += self.apply_mass(vd) / dt
        out[self.M["is_dirichlet"]] = v[self.M["is_dirichlet"]]
        out[self.M["is_slave"]] = 0.0
        return out

    def element_matrices(self, cells, k, dk, g, dt):
        """Dense element Jacobians (operators.py:412-424), any degree."""
        q = self.q
        V, D = self.tb.V, self.tb.D
        nl = q ** 3
        # Phi[c, qp], G[d, c, qp] in the local orders
        Phi = np.einsum("ia,jb,kc->ijkabc", V, V, V).reshape(nl, nl)
        G = np.stack([np.einsum("ia,jb,kc->ijkabc", D, V, V).reshape(nl, nl),
                      np.einsum("ia,jb,kc->ijkabc", V, D, V).reshape(nl, nl),
                      np.einsum("ia,jb,kc->ijkabc", V, V, D).reshape(nl, nl)])
        mat = self.params.material
        w = self.tb.w3.reshape(-1)
        out = np.empty((len(cells), nl, nl))
        for t, e in enumerate(cells):
            dw = self.det_w[e].reshape(-1)
            kq = k[e].reshape(-1)
            dkq = dk[e].reshape(-1)
            gq = g[e].reshape(3, -1)
            A = (mat.rho * mat.c / dt) * (Phi * dw[None]) @ Phi.T
            A += (self.h[e] / 2.0) * np.einsum("q,dcq,deq->ce", kq * w, G, G)
            A += self.gscale[e] * np.einsum("q,eq,dcq,dq->ce", dkq * dw, Phi, G, gq)
            out[t] = A
        return out

    def jacobian_diagonal(self, T_lin, r_c, dt, tangent=None):
        """Exact diagonal of the condensed Jacobian (operators.py:426-459):
        plain cells by their element diagonal, cells touching a hanging
        node through the constraint expansion of every corner pair."""
        k, dk, g = tangent if tangent is not None else self.tangent(T_lin, r_c)
        M = self.M
        cn = M["cell_nodes"]
        touched = np.flatnonzero(M["is_slave"][cn].any(axis=1))
        plain = np.ones(self.n, dtype=bool)
        plain[touched] = False
        diag = np.zeros(self.nv)
        rows = np.flatnonzero(plain)
        for s in range(0, len(rows), 4096):
            blk = rows[s:s + 4096]
            A = self.element_matrices(blk, k, dk, g, dt)
            ed = np.einsum("ncc->nc", A)
            diag += np.bincount(cn[blk].ravel(), weights=ed.ravel(),
                                minlength=self.nv)
        if touched.size:
            expand = {}
            for i, s in enumerate(M["slaves"]):
                sl = slice(M["slave_ptr"][i], M["slave_ptr"][i + 1])
                expand[int(s)] = dict(zip(M["slave_masters"][sl].tolist(),
                                          M["slave_weights"][sl].tolist()))
            A = self.element_matrices(touched, k, dk, g, dt)
            for t, e in enumerate(touched):
                ex = [expand.get(int(gv), {int(gv): 1.0}) for gv in cn[e]]
                for a in range(cn.shape[1]):
                    for b in range(cn.shape[1]):
                        for m, wa in ex[a].items():
                            wb = ex[b].get(m)
                            if wb is not None:
                                diag[m] += wa * wb * A[t, a, b]
        diag[M["is_slave"]] = 1.0
        diag[M["is_dirichlet"]] = 1.0
        return diag


# ---------------------------------------------------------------------------
# time integration  (timestepping.py)
# ---------------------------------------------------------------------------

T_DIVERGED = 1.0e7


def pcg(apply_fn, b, diag_inv=None, tol=1e-10, max_iter=2000):
    """Jacobi-PCG, x0 = 0, stop at ||r|| <= tol ||b|| (timestepping.py:102)."""
    n = len(b)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return np.zeros(n), 0, True
    x = np.zeros(n)
    r = b.copy()
    z = r * diag_inv if diag_inv is not None else r.copy()
    d = z.copy()
    rz = float(r @ z)
    for it in range(1, max_iter + 1):
        Ad = apply_fn(d)
        alpha = rz / float(d @ Ad)
        x += alpha * d
        r -= alpha * Ad
        if float(np.linalg.norm(r)) <= tol * bnorm:
            return x, it, True
        z = r * diag_inv if diag_inv is not None else r.copy()
        rz_new = float(r @ z)
        d = z + (rz_new / rz) * d
        rz = rz_new
    return x, max_iter, False


def spectral_radius(apply_fn, n, seed=0, tol=1e-9, max_iter=500, lams=None):
    """Power iteration (timestepping.py:49-67): v0 ~ N(0,1) from
    default_rng(seed), normalised; returns (max(|lam|, |lam_prev|), applies).
    `lams`, when a list, receives every Rayleigh quotient."""
    v = np.random.default_rng(seed).standard_normal(n)
    v /= np.linalg.norm(v)
    lam_prev = lam = 0.0
    it = 0
    for it in range(1, max_iter + 1):
        w = apply_fn(v)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0, it
        lam_prev, lam = lam, float(np.dot(v, w))
        if lams is not None:
            lams.append(lam)
        v = w / nw
        if abs(lam - lam_prev) <= tol * abs(lam):
            break
    return max(abs(lam), abs(lam_prev)), it


def step_criteria_rho(op):
    """rho(C~^-1 K) at k frozen to max(k_m, k_s) (timestepping.py:70-99):
    the apply closes constraints, zeroes Dirichlet entries, evaluates the
    diffusion-only rhs, scales by C~^-1 and zeroes Dirichlet/slave rows.
    Returns (rho, applies); dt_stability = 2 / rho."""
    mat = op.params.material
    k_frozen = max(mat.k_m, mat.k_s)
    cinv = op.capacity_inverse()
    M = op.M

    def apply(v):
        vd = op.distribute(v.copy())
        vd[M["is_dirichlet"]] = 0.0
        w = -op.evaluate_rhs(vd, None, faces=False, source=False, frozen_k=k_frozen)
        w *= cinv
        w[M["is_dirichlet"]] = 0.0
        w[M["is_slave"]] = 0.0
        return w

    return spectral_radius(apply, op.nv)


def implicit_step(op, T_n, r_c, dt, settings):
    """Backward Euler with Newton + Jacobi-PCG (timestepping.py:229-283)."""
    M = op.M
    f_re = op.evaluate_rhs(T_n, r_c, (), diffusion=False, source=False)
    T = T_n.copy()
    norm0 = None
    nn = nk = 0
    for _ in range(settings.newton_max_iter):
        f = op.evaluate_rhs(T, r_c, (), faces=False, source=False) + f_re
        r = op.apply_mass(T - T_n) / dt - f
        r[M["is_dirichlet"]] = 0.0
        r[M["is_slave"]] = 0.0
        norm = float(np.linalg.norm(r))
        if norm0 is None:
            norm0 = norm
        if norm <= settings.newton_abs_tol or norm <= settings.newton_tol * norm0:
            return T, nn, nk
        tan = op.tangent(T, r_c)
        di = None
        if settings.preconditioner == "diagonal":
            di = 1.0 / op.jacobian_diagonal(T, r_c, dt, tangent=tan)
        delta, it, ok = pcg(lambda v: op.apply_jacobian(v, T, r_c, dt, tan),
                            -r, di, settings.krylov_tol, settings.krylov_max_iter)
        nk += it
        if not ok:
            return None
        T = T + delta
        op.distribute(T)
        nn += 1
    return None


def run_explicit(op, T, r_c, dt_steps, beams_per_step):
    """Scan loop (timestepping.py:195-226): step, stability check,
    history update.  beams_per_step[i] is a list of (x, y, z_top, P)."""
    T = T.copy()
    r_c = r_c.copy()
    for i, dt in enumerate(dt_steps):
        T = op.explicit_step(T, dt, r_c, beams_per_step[i])
        m = float(np.max(np.abs(T)))
        if not np.isfinite(m) or m > T_DIVERGED:
            raise FloatingPointError(f"diverged at step {i + 1}: {m}")
        r_c = op.update_history(r_c, T)
    return T, r_c


# ---------------------------------------------------------------------------
# mesh tables
# ---------------------------------------------------------------------------

def tables_from_arrays(vertices_count, cell_verts, cell_h, cell_anchor,
                       is_slave, is_dirichlet, slaves, slave_ptr,
                       slave_masters, slave_weights, face_cell, face_offset,
                       face_fsize, cell_size_lattice):
    """Q1 tables from reference DofMap/Forest/FaceSet arrays
    (operators.py:96-134)."""
    fc = np.asarray(face_cell, dtype=np.int64)
    size = np.asarray(cell_size_lattice, dtype=np.float64)
    if len(fc):
        r0 = np.asarray(face_offset, dtype=np.float64) / size[fc][:, None]
        rr = np.asarray(face_fsize, dtype=np.float64) / size[fc]
    else:
        r0 = np.zeros((0, 2))
        rr = np.zeros(0)
    return dict(p=1, cell_nodes=np.asarray(cell_verts, dtype=np.int64),
                h=np.asarray(cell_h, dtype=np.float64),
                anchor=np.asarray(cell_anchor, dtype=np.float64),
                nv=int(vertices_count),
                is_slave=np.asarray(is_slave, bool),
                is_dirichlet=np.asarray(is_dirichlet, bool),
                slaves=np.asarray(slaves, np.int64),
                slave_ptr=np.asarray(slave_ptr, np.int64),
                slave_masters=np.asarray(slave_masters, np.int64),
                slave_weights=np.asarray(slave_weights, np.float64),
                face_cell=fc, face_r0=r0, face_rr=rr)


def structured_tables(nx, ny, nz, h, p, origin=(0.0, 0.0, None),
                      dirichlet_bottom=True, top_faces=True):
    """Uniform box of degree-p cells; nodes numbered x-major / z-fastest
    on the p-refined lattice (the reference rule mesh.py:712-715)."""
    ox, oy, oz = origin
    if oz is None:
        oz = -nz * h
    NX, NY, NZ = p * nx + 1, p * ny + 1, p * nz + 1
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz),
                          indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    l = np.arange(p + 1)
    I = (p * i)[:, None, None, None] + l[None, :, None, None]
    J = (p * j)[:, None, None, None] + l[None, None, :, None]
    K = (p * k)[:, None, None, None] + l[None, None, None, :]
    nodes = ((I * NY + J) * NZ + K).reshape(len(i), -1)
    n = len(i)
    anchor = np.stack([ox + i * h, oy + j * h, oz + k * h], axis=1)
    nv = NX * NY * NZ
    is_dir = np.zeros((NX, NY, NZ), dtype=bool)
    if dirichlet_bottom:
        is_dir[:, :, 0] = True
    fc = np.flatnonzero(k == nz - 1) if top_faces else np.zeros(0, np.int64)
    return dict(p=p, cell_nodes=nodes, h=np.full(n, float(h)), anchor=anchor,
                nv=nv, is_slave=np.zeros(nv, bool), is_dirichlet=is_dir.ravel(),
                slaves=np.zeros(0, np.int64), slave_ptr=np.zeros(1, np.int64),
                slave_masters=np.zeros(0, np.int64),
                slave_weights=np.zeros(0), face_cell=fc.astype(np.int64),
                face_r0=np.zeros((len(fc), 2)), face_rr=np.ones(len(fc)))


def beam_tuple(b):
    """BeamState-like or record -> (x, y, z_top, P) with P = 0 if off."""
    if b is None:
        return None
    if hasattr(b, "position"):
        on = bool(b.active) and float(b.power) > 0.0
        return (float(b.position[0]), float(b.position[1]), float(b.z_top),
                float(b.power) if on else 0.0)
    on = int(b["active"]) != 0 and float(b["power"]) > 0.0
    return (float(b["x"]), float(b["y"]), float(b["z_top"]),
            float(b["power"]) if on else 0.0)


def fitted_tables(part):
    """Tables of a paper_2302_05164_b200.mesh.FittedPart (cell rows with
    x extents, degree p): its node ids (the reference's sorted-key rule on
    the active nodes), cell anchors, Dirichlet bottom plane, top facets."""
    p, h = part.degree, part.h
    ox, oy, oz = part.origin
    i, j, k = part.cells()
    nodes = part.cell_node_ids()
    n = len(i)
    anchor = np.stack([ox + i * h, oy + j * h, oz + k * h], axis=1)
    nv = part.n_vertices
    fc = np.flatnonzero(k == part.nz - 1) if part.top_faces else np.zeros(0, np.int64)
    return dict(p=p, cell_nodes=nodes, h=np.full(n, float(h)), anchor=anchor,
                nv=nv, is_slave=np.zeros(nv, bool), is_dirichlet=part.is_dirichlet,
                slaves=np.zeros(0, np.int64), slave_ptr=np.zeros(1, np.int64),
                slave_masters=np.zeros(0, np.int64),
                slave_weights=np.zeros(0), face_cell=fc.astype(np.int64),
                face_r0=np.zeros((len(fc), 2)), face_rr=np.ones(len(fc)))
