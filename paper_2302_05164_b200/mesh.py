"""Host-side mesh tables for the B200 operator.

The reference keeps its adaptive voxel forest and DoF map in numpy
(``scantherm/mesh.py``).  The device only needs flat tables: per-cell
corner ids, sizes and anchors, the hanging-node CSR, the Dirichlet mask
and the radiating facets.  This module holds

* :class:`Forest` / :class:`DofMap` — minimal containers with the
  attributes the operator reads (duck-compatible with the reference
  ``Forest`` :143 and ``DofMap`` :619), so fixtures serialised from the
  reference can be rebuilt on a GPU box that has no reference install;
* :func:`build_dofmap` — vertex numbering by sorted packed lattice key
  plus hanging-node constraints with chain resolution and the Dirichlet
  plane, restating ``mesh.py:706-779`` (bit-exact; pinned by
  tests/test_mesh_tables.py against the reference);
* :func:`interface_faces` — the +z radiating facets, restating
  ``mesh.py:998-1072``;
* :class:`StructuredBox` — a uniform box of Qp cells whose node lattice
  is numbered x-major / z-fastest, the rule the reference applies to
  Q1 (``mesh.py:712-715``) extended to the p-refined lattice.  Large
  structured problems never materialise per-cell tables.
"""

from dataclasses import dataclass

import numpy as np

_BITS = 21
_OFF = 1 << (_BITS - 1)
_MASK = (1 << _BITS) - 1

# corner c = ix*4 + iy*2 + iz  (reference mesh.py:26-30)
CORNER_OFFSETS = np.array([((c >> 2) & 1, (c >> 1) & 1, c & 1)
                           for c in range(8)], dtype=np.int64)


def pack_coords(coords):
    c = np.asarray(coords, dtype=np.int64) + _OFF
    if c.size and (c.min() < 0 or c.max() > _MASK):
        raise ValueError("lattice coordinate out of packable range")
    return (c[..., 0] << (2 * _BITS)) | (c[..., 1] << _BITS) | c[..., 2]


def unpack_coords(keys):
    keys = np.asarray(keys, dtype=np.int64)
    out = np.empty(keys.shape + (3,), dtype=np.int64)
    out[..., 0] = (keys >> (2 * _BITS)) & _MASK
    out[..., 1] = (keys >> _BITS) & _MASK
    out[..., 2] = keys & _MASK
    return out - _OFF


class Forest:
    """Leaf table: level, anchor (finest lattice units), active flags."""

    def __init__(self, level, anchor, active, init_consol, depth, cpl,
                 h_fine, z_min=0, dirichlet_bottom=True, epoch=0,
                 current_layer=-1):
        self.level = np.asarray(level, dtype=np.int8)
        self.anchor = np.asarray(anchor, dtype=np.int64).reshape(-1, 3)
        self.active = np.asarray(active, dtype=bool)
        self.init_consol = np.asarray(init_consol, dtype=bool)
        self.depth = int(depth)
        self.cpl = int(cpl)
        self._h_fine = float(h_fine)
        self.z_min_lattice = int(z_min)
        self.dirichlet_bottom = bool(dirichlet_bottom)
        self.epoch = int(epoch)
        self.current_layer = int(current_layer)
        self._index = None

    @classmethod
    def from_reference(cls, f):
        """Copy the tables of a reference ``scantherm.mesh.Forest``."""
        return cls(f.level, f.anchor, f.active, f.init_consol, f.depth, f.cpl,
                   f.h_fine, f.geometry.z_min(), f.mesh_params.dirichlet_bottom,
                   f.epoch, f.current_layer)

    @property
    def h_fine(self):
        return self._h_fine

    @property
    def n_cells(self):
        return len(self.level)

    def size(self, idx=slice(None)):
        return np.int64(1) << (self.depth - self.level[idx].astype(np.int64))

    def size_m(self, idx=slice(None)):
        return self.size(idx) * self.h_fine

    def active_cells(self):
        return np.flatnonzero(self.active)

    def active_volume_m3(self):
        s = self.size_m(self.active_cells())
        return float(np.sum(s * s * s))

    def _levels(self):
        if self._index is None:
            idx = {}
            for ell in np.unique(self.level):
                rows = np.flatnonzero(self.level == ell)
                keys = pack_coords(self.anchor[rows])
                o = np.argsort(keys, kind="stable")
                idx[int(ell)] = (keys[o], rows[o])
            self._index = idx
        return self._index

    def lookup(self, level, anchors):
        anchors = np.atleast_2d(np.asarray(anchors, dtype=np.int64))
        out = np.full(len(anchors), -1, dtype=np.int64)
        entry = self._levels().get(int(level))
        if entry is None or len(anchors) == 0:
            return out
        keys, rows = entry
        want = pack_coords(anchors)
        pos = np.searchsorted(keys, want)
        ok = pos < len(keys)
        ok[ok] &= keys[pos[ok]] == want[ok]
        out[ok] = rows[pos[ok]]
        return out


def _forest_z_min(forest):
    if hasattr(forest, "z_min_lattice"):
        return forest.z_min_lattice
    return forest.geometry.z_min()


def _forest_dirichlet(forest):
    if hasattr(forest, "dirichlet_bottom"):
        return forest.dirichlet_bottom
    return forest.mesh_params.dirichlet_bottom


@dataclass
class DofMap:
    """Vertex numbering + hanging-node constraints (reference mesh.py:619)."""

    vertices: np.ndarray
    cell_verts: np.ndarray
    active_rows: np.ndarray
    is_slave: np.ndarray
    is_dirichlet: np.ndarray
    slaves: np.ndarray
    slave_ptr: np.ndarray
    slave_masters: np.ndarray
    slave_weights: np.ndarray
    h_fine: float

    @property
    def n_vertices(self):
        return len(self.vertices)

    @property
    def n_dofs(self):
        return self.n_vertices - len(self.slaves)

    def vertices_m(self):
        return self.vertices * self.h_fine

    def distribute(self, values):
        if len(self.slaves):
            prod = self.slave_weights * values[self.slave_masters]
            values[self.slaves] = np.add.reduceat(prod, self.slave_ptr[:-1])
        return values

    def condense(self, values):
        if len(self.slaves):
            rep = np.repeat(values[self.slaves], np.diff(self.slave_ptr))
            np.add.at(values, self.slave_masters, self.slave_weights * rep)
            values[self.slaves] = 0.0
        return values

    @classmethod
    def from_reference(cls, d):
        return cls(d.vertices, d.cell_verts, d.active_rows, d.is_slave,
                   d.is_dirichlet, d.slaves, d.slave_ptr, d.slave_masters,
                   d.slave_weights, d.h_fine)


def _hanging_host_cell(forest, verts):
    """For each vertex: an active leaf containing it off its corners
    (row, offset in lattice units) or row -1.  Same search order as the
    reference (_containing_active_cell, mesh.py:673-703): levels coarse
    to fine, candidate anchors in bit order, first hit wins."""
    n = len(verts)
    row = np.full(n, -1, dtype=np.int64)
    rel = np.zeros((n, 3), dtype=np.int64)
    for ell in sorted(forest._levels() if hasattr(forest, "_levels")
                      else forest._level_index()):
        todo = np.flatnonzero(row == -1)
        if todo.size == 0:
            break
        s = np.int64(1) << (forest.depth - ell)
        v = verts[todo]
        hi = (v // s) * s
        lo = np.where(v % s == 0, hi - s, hi)
        for bits in range(8):
            pick = np.array([(bits >> 2) & 1, (bits >> 1) & 1, bits & 1]) == 1
            a = np.where(pick[None, :], hi, lo)
            hit = forest.lookup(ell, a)
            ok = hit >= 0
            ok[ok] &= forest.active[hit[ok]]
            if not ok.any():
                continue
            r = v - a
            on_corner = np.all((r == 0) | (r == s), axis=1)
            take = ok & ~on_corner & (row[todo] == -1)
            row[todo[take]] = hit[take]
            rel[todo[take]] = r[take]
    return row, rel


def build_dofmap(forest) -> DofMap:
    """Vertex numbering + hanging constraints (reference mesh.py:706-779)."""
    rows = forest.active_cells()
    size = forest.size(rows)
    corners = forest.anchor[rows, None, :] + CORNER_OFFSETS[None] * size[:, None, None]
    keys = pack_coords(corners.reshape(-1, 3))
    uniq, inv = np.unique(keys, return_inverse=True)
    cell_verts = inv.reshape(-1, 8).astype(np.int32)
    verts = unpack_coords(uniq)
    nv = len(verts)

    cand = np.flatnonzero(np.bincount(inv, minlength=nv) < 8)
    crow, crel = _hanging_host_cell(forest, verts[cand])
    pos_of_row = np.full(forest.n_cells, -1, dtype=np.int64)
    pos_of_row[rows] = np.arange(len(rows))

    cons = {}
    for j in np.flatnonzero(crow >= 0):
        c = int(crow[j])
        s = float(forest.size(c))
        frac = crel[j] / s
        lst = []
        for ci in range(8):
            w = 1.0
            for d in range(3):
                w *= frac[d] if CORNER_OFFSETS[ci, d] else (1.0 - frac[d])
            if w > 0.0:
                lst.append((int(cell_verts[pos_of_row[c], ci]), w))
        cons[int(cand[j])] = lst

    # constraint chains (a master hanging on a coarser cell), resolved by
    # substitution until closed, in the reference's dict order
    changed = True
    while changed:
        changed = False
        for v in list(cons):
            ms = cons[v]
            if any(m in cons for m, _ in ms):
                acc = {}
                for m, wm in ms:
                    if m in cons:
                        for mm, wmm in cons[m]:
                            acc[mm] = acc.get(mm, 0.0) + wm * wmm
                    else:
                        acc[m] = acc.get(m, 0.0) + wm
                cons[v] = sorted(acc.items())
                changed = True

    slaves = np.array(sorted(cons), dtype=np.int64)
    ptr = np.zeros(len(slaves) + 1, dtype=np.int64)
    mlist, wlist = [], []
    for i, v in enumerate(slaves):
        for m, w in sorted(cons[int(v)]):
            mlist.append(m)
            wlist.append(w)
        ptr[i + 1] = len(mlist)
    is_slave = np.zeros(nv, dtype=bool)
    is_slave[slaves] = True
    is_dir = np.zeros(nv, dtype=bool)
    if _forest_dirichlet(forest):
        is_dir = (verts[:, 2] == _forest_z_min(forest)) & ~is_slave
    return DofMap(verts, cell_verts, rows, is_slave, is_dir, slaves, ptr,
                  np.array(mlist, dtype=np.int64), np.array(wlist, dtype=np.float64),
                  forest.h_fine)


def initial_history(forest):
    """r_c = 1 on initially consolidated cells, 0 on powder (mesh.py:785)."""
    from .material import HistoryField
    rows = forest.active_cells()
    r_c = np.zeros((len(rows), 2, 2, 2))
    r_c[forest.init_consol[rows]] = 1.0
    return HistoryField(r_c, forest.epoch)


@dataclass
class FaceSet:
    cell_rows: np.ndarray
    offset: np.ndarray
    fsize: np.ndarray

    def __len__(self):
        return len(self.cell_rows)


def interface_faces(forest) -> FaceSet:
    """+z boundary facets of the active region (reference mesh.py:998).

    A top face is exterior when the leaf above it (same level, or the
    coarser parent when the face lies on the parent's bottom plane) is
    void; when no such leaf exists the face is split against the finer
    level and every quarter not covered by an active leaf is emitted.
    """
    rows = forest.active_cells()
    out_r, out_o, out_s = [], [], []
    lev_all = forest.level[rows]
    for ell in np.unique(lev_all):
        ell = int(ell)
        sub = rows[lev_all == ell]
        s = np.int64(1) << (forest.depth - ell)
        ax, ay = forest.anchor[sub, 0], forest.anchor[sub, 1]
        top = forest.anchor[sub, 2] + s

        def status(hit):
            st = np.zeros(len(hit), dtype=np.int8)
            got = hit >= 0
            st[got] = np.where(forest.active[hit[got]], 1, 2)
            return st

        cov = status(forest.lookup(ell, np.column_stack([ax, ay, top])))
        if ell > 0:
            ps = 2 * s
            par = forest.lookup(ell - 1, np.column_stack([(ax // ps) * ps,
                                                          (ay // ps) * ps, top]))
            par[top % ps != 0] = -1
            pst = status(par)
            cov = np.where(cov == 0, pst, cov)

        full = cov == 2
        open_idx = np.flatnonzero(cov == 0)
        if ell < forest.depth and open_idx.size:
            hs = s >> 1
            q = np.zeros((len(open_idx), 2, 2), dtype=np.int8)
            exists = np.zeros(len(open_idx), dtype=bool)
            for i in range(2):
                for j in range(2):
                    hit = forest.lookup(ell + 1, np.column_stack(
                        [ax[open_idx] + i * hs, ay[open_idx] + j * hs, top[open_idx]]))
                    q[:, i, j] = status(hit)
                    exists |= hit >= 0
            for t, k in enumerate(open_idx):
                if exists[t]:
                    for i in range(2):
                        for j in range(2):
                            if q[t, i, j] != 1:
                                out_r.append(sub[k])
                                out_o.append((i * hs, j * hs))
                                out_s.append(hs)
                else:
                    full[k] = True
        else:
            full[open_idx] = True
        for k in np.flatnonzero(full):
            out_r.append(sub[k])
            out_o.append((0, 0))
            out_s.append(s)

    if not out_r:
        return FaceSet(np.zeros(0, np.int64), np.zeros((0, 2), np.int64),
                       np.zeros(0, np.int64))
    r = np.array(out_r, dtype=np.int64)
    o = np.array(out_o, dtype=np.int64).reshape(-1, 2)
    s = np.array(out_s, dtype=np.int64)
    order = np.lexsort((o[:, 1], o[:, 0], r))
    return FaceSet(r[order], o[order], s[order])


class StructuredBox:
    """Uniform box of degree-p hexahedra, nodes numbered x-major, z-fastest.

    Cells span [x0, x0 + nx h] x [y0, y0 + ny h] x [z0, z0 + nz h].  Node
    (I, J, K) of the p-refined lattice has id (I (p ny + 1) + J)(p nz + 1)
    + K, which for p = 1 is exactly the reference numbering of a chamber
    plate (``mesh.py:712-715``).  The bottom node plane is Dirichlet when
    ``dirichlet_bottom``; the top cell faces radiate when ``top_faces``.
    Acts as both the forest and the dof map for :class:`ThermalOperator`.
    """

    structured = True

    def __init__(self, nx, ny, nz, h, degree=1, origin=(0.0, 0.0, None),
                 dirichlet_bottom=True, top_faces=True, epoch=0):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.h = float(h)
        self.degree = int(degree)
        if not 1 <= self.degree <= 4:
            raise ValueError("degree must be 1..4")
        ox, oy, oz = origin
        if oz is None:
            oz = -self.nz * self.h      # plate below z = 0 as in the reference
        self.origin = (float(ox), float(oy), float(oz))
        self.dirichlet_bottom = bool(dirichlet_bottom)
        self.top_faces = bool(top_faces)
        self.epoch = int(epoch)
        self.h_fine = self.h

    # --- node lattice --------------------------------------------------
    @property
    def node_dims(self):
        p = self.degree
        return (p * self.nx + 1, p * self.ny + 1, p * self.nz + 1)

    @property
    def n_vertices(self):
        a, b, c = self.node_dims
        return a * b * c

    @property
    def n_dofs(self):
        return self.n_vertices

    @property
    def n_cells(self):
        return self.nx * self.ny * self.nz

    @property
    def slaves(self):
        return np.zeros(0, dtype=np.int64)

    @property
    def is_slave(self):
        return np.zeros(self.n_vertices, dtype=bool)

    @property
    def is_dirichlet(self):
        a, b, c = self.node_dims
        m = np.zeros((a, b, c), dtype=bool)
        if self.dirichlet_bottom:
            m[:, :, 0] = True
        return m.reshape(-1)

    def distribute(self, values):
        return values

    def condense(self, values):
        return values

    def active_volume_m3(self):
        return self.n_cells * self.h ** 3

    def node_coords_1d(self, axis):
        """Physical node coordinates along one axis (GLL within cells)."""
        from .basis import gll_points
        n = (self.nx, self.ny, self.nz)[axis]
        xi = gll_points(self.degree)
        loc = (xi[:-1] + 1.0) / 2.0 * self.h
        pts = (np.arange(n)[:, None] * self.h + loc[None, :]).reshape(-1)
        pts = np.concatenate([pts, [n * self.h]])
        return self.origin[axis] + pts

    def cell_node_ids(self, cells=None):
        """(m, (p+1)^3) node ids of the given linear cell indices
        (c = (i ny + j) nz + k), local order a*(p+1)^2 + b*(p+1) + c."""
        p = self.degree
        a, b, c = self.node_dims
        if cells is None:
            cells = np.arange(self.n_cells)
        cells = np.asarray(cells, dtype=np.int64)
        i = cells // (self.ny * self.nz)
        j = (cells // self.nz) % self.ny
        k = cells % self.nz
        l = np.arange(p + 1)
        I = (p * i)[:, None, None, None] + l[None, :, None, None]
        J = (p * j)[:, None, None, None] + l[None, None, :, None]
        K = (p * k)[:, None, None, None] + l[None, None, None, :]
        return ((I * b + J) * c + K).reshape(len(cells), -1)

    def to_forest_dofmap(self):
        """Q1 only: explicit Forest/DofMap tables (small boxes, tests)."""
        if self.degree != 1:
            raise ValueError("explicit tables exist for Q1 only")
        nx, ny, nz = self.nx, self.ny, self.nz
        ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz),
                                 indexing="ij")
        anchor = np.stack([ii, jj, kk], -1).reshape(-1, 3)
        anchor[:, 2] -= nz
        n = len(anchor)
        f = Forest(np.zeros(n, np.int8), anchor, np.ones(n, bool),
                   np.ones(n, bool), 0, 1, self.h, -nz, self.dirichlet_bottom,
                   self.epoch)
        return f, build_dofmap(f)
