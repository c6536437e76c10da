"""Mesh tables of the B200 operator: leaf sets, DoF maps, facets, layer
activation and transfer.

The reference keeps its adaptive voxel forest and DoF map in numpy
(``pkg/src/scantherm/mesh.py``).  Here the table construction runs in
host C++ (``csrc/st_forest.cpp``, exported through the C ABI in
``include/scantherm_b200.h``); this module holds the Python containers
the operator and the time integrators read and thin wrappers around the
native builders:

* :class:`Forest`, :class:`DofMap`, :class:`FaceSet` — containers with
  the attribute names of the reference ``Forest`` (mesh.py:143),
  ``DofMap`` (:619) and ``FaceSet`` (:980), so reference objects and
  these are interchangeable at the operator boundary;
* :func:`build_coarse_grid`, :func:`advance_layer`, :func:`apply_update`,
  :func:`build_dofmap`, :func:`interface_faces` — the growing-domain
  pipeline of ``run_build`` (driver.py:177-193) on native code, bit-exact
  with the reference (tests/test_mesh_tables.py, tests/test_activation.py
  against fixtures the reference produced);
* :class:`Geometry` — integer build-volume boxes (plate + per-layer
  footprints) for chamber and fitted parts;
* :class:`StructuredBox` / :class:`FittedPart` — uniform degree-p meshes
  that never materialise per-cell tables (the structured backend).
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib

# corner c = ix*4 + iy*2 + iz (the reference's local corner order)
CORNER_OFFSETS = np.array([((c >> 2) & 1, (c >> 1) & 1, c & 1) for c in range(8)],
                          dtype=np.int64)


# --- containers --------------------------------------------------------------

class Forest:
    """Leaf table of the adaptive voxel mesh (anchors in finest lattice
    units, canonical order)."""

    def __init__(self, level, anchor, active, init_consol, depth, cpl,
                 h_fine, z_min=0, dirichlet_bottom=True, epoch=0,
                 current_layer=-1, n_layers=None):
        self.level = np.ascontiguousarray(level, dtype=np.int8)
        self.anchor = np.ascontiguousarray(anchor, dtype=np.int64).reshape(-1, 3)
        self.active = np.ascontiguousarray(active, dtype=bool)
        self.init_consol = np.ascontiguousarray(init_consol, dtype=bool)
        self.depth = int(depth)
        self.cpl = int(cpl)
        self._h_fine = float(h_fine)
        self.z_min_lattice = int(z_min)
        self.dirichlet_bottom = bool(dirichlet_bottom)
        self.epoch = int(epoch)
        self.current_layer = int(current_layer)
        self.n_layers = n_layers

    @classmethod
    def from_reference(cls, f):
        """Tables of a reference ``scantherm.mesh.Forest``."""
        return cls(f.level, f.anchor, f.active, f.init_consol, f.depth, f.cpl,
                   f.h_fine, f.geometry.z_min(), f.mesh_params.dirichlet_bottom,
                   f.epoch, f.current_layer, f.geometry.n_layers)

    @property
    def h_fine(self):
        return self._h_fine

    @property
    def n_cells(self):
        return len(self.level)

    def size(self, idx=slice(None)):
        """Edge length in lattice units."""
        return np.left_shift(np.int64(1), self.depth - self.level[idx].astype(np.int64))

    def size_m(self, idx=slice(None)):
        return self.size(idx) * self.h_fine

    def active_cells(self):
        return np.flatnonzero(self.active)

    def active_volume_m3(self):
        e = self.size_m(self.active_cells())
        return float(np.sum(e * e * e))


def _z_min(forest):
    return forest.z_min_lattice if hasattr(forest, "z_min_lattice") else forest.geometry.z_min()


def _dirichlet_bottom(forest):
    if hasattr(forest, "dirichlet_bottom"):
        return forest.dirichlet_bottom
    return forest.mesh_params.dirichlet_bottom


@dataclass
class DofMap:
    """Vertex numbering of the active region with hanging-node constraints
    (the reference DofMap's fields); slaves are interpolated from masters
    that are never slaves themselves."""

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

    def _csr(self):
        i64 = ctypes.POINTER(ctypes.c_int64)
        arrs = [np.ascontiguousarray(a, dtype=np.int64)
                for a in (self.slaves, self.slave_ptr, self.slave_masters)]
        w = np.ascontiguousarray(self.slave_weights, dtype=np.float64)
        return arrs, w, [a.ctypes.data_as(i64) for a in arrs] + [_lib.dptr(w)]

    def distribute(self, values):
        """Slave entries <- weighted sums of their masters (in place)."""
        if len(self.slaves):
            _check_f64(values)
            keep, w, p = self._csr()
            _lib.check(_lib.load().st_host_distribute(len(self.slaves), *p, _lib.dptr(values)),
                       "distribute")
        return values

    def condense(self, values):
        """Slave entries folded into their masters, slaves zeroed (in place)."""
        if len(self.slaves):
            _check_f64(values)
            keep, w, p = self._csr()
            _lib.check(_lib.load().st_host_condense(len(self.slaves), *p, _lib.dptr(values)),
                       "condense")
        return values

    @classmethod
    def from_reference(cls, d):
        return cls(d.vertices, d.cell_verts, d.active_rows, d.is_slave,
                   d.is_dirichlet, d.slaves, d.slave_ptr, d.slave_masters,
                   d.slave_weights, d.h_fine)


def _check_f64(values):
    if not (isinstance(values, np.ndarray) and values.dtype == np.float64
            and values.flags["C_CONTIGUOUS"] and values.flags["WRITEABLE"]):
        raise TypeError("constraint plumbing works in place on a contiguous float64 array")


@dataclass
class FaceSet:
    """+z radiating facets: owning leaf row, in-face offset and edge
    length (lattice units)."""

    cell_rows: np.ndarray
    offset: np.ndarray
    fsize: np.ndarray

    def __len__(self):
        return len(self.cell_rows)


@dataclass
class NodalField:
    values: np.ndarray
    epoch: int

    def copy(self):
        return NodalField(self.values.copy(), self.epoch)


@dataclass
class TransferReport:
    """Per new vertex: 0 copied, 1 interpolated, 2 fresh (T_0)."""

    vertex_source: np.ndarray


@dataclass
class MeshUpdatePlan:
    """Target leaf set of a layer advance with its lineage to the old set
    (the reference MeshUpdatePlan's fields)."""

    base_epoch: int
    new_layer: int
    level: np.ndarray
    anchor: np.ndarray
    active: np.ndarray
    init_consol: np.ndarray
    same_src: np.ndarray
    ancestor_src: np.ndarray
    coarse_groups: list
    coarsened_min_rc: list
    transfer_report: TransferReport = field(default=None)


# --- native builders -----------------------------------------------------------

class _Leaves:
    """st_leaves view of a forest (keeps the arrays alive)."""

    def __init__(self, forest):
        self.level = np.ascontiguousarray(forest.level, dtype=np.int8)
        self.anchor = np.ascontiguousarray(forest.anchor, dtype=np.int64)
        self.active = np.ascontiguousarray(forest.active, dtype=np.uint8)
        self.consol = np.ascontiguousarray(forest.init_consol, dtype=np.uint8)
        self.c = _lib.StLeaves(
            len(self.level), int(forest.depth), int(forest.cpl),
            self.level.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)),
            self.anchor.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            self.active.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
            self.consol.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))

    @property
    def ref(self):
        return ctypes.byref(self.c)


def _take(call, what):
    """Run a builder returning an st_tables bag; dict of numpy copies."""
    lib = _lib.load()
    t = ctypes.c_void_p()
    _lib.check(call(ctypes.byref(t)), what)
    try:
        return _lib.tables_dict(t)
    finally:
        lib.st_tables_free(t)


def build_dofmap(forest) -> DofMap:
    """Vertex numbering + hanging-node constraints + Dirichlet plane
    (replaces reference build_dofmap, mesh.py:706-779)."""
    L = _Leaves(forest)
    d = _take(lambda out: _lib.load().st_build_dofmap(
        L.ref, int(_z_min(forest)), int(bool(_dirichlet_bottom(forest))), out), "build_dofmap")
    return DofMap(d["vertices"], d["cell_verts"], d["active_rows"],
                  d["is_slave"].astype(bool), d["is_dirichlet"].astype(bool), d["slaves"],
                  d["slave_ptr"], d["slave_masters"], d["slave_weights"], forest.h_fine)


def interface_faces(forest) -> FaceSet:
    """Radiating +z facets (replaces reference interface_faces,
    mesh.py:998-1072)."""
    L = _Leaves(forest)
    d = _take(lambda out: _lib.load().st_interface_faces(L.ref, out), "interface_faces")
    return FaceSet(d["cell_rows"], d["offset"].reshape(-1, 2), d["fsize"])


def initial_history(forest):
    """Consolidation state per quadrature point: 1 on initially
    consolidated leaves (the plate), 0 on powder."""
    from .material import HistoryField
    consol = forest.init_consol[forest.active_cells()]
    r_c = np.broadcast_to(consol.astype(np.float64)[:, None, None, None],
                          (len(consol), 2, 2, 2)).copy()
    return HistoryField(r_c, forest.epoch)


@dataclass
class Geometry:
    """Build volume in finest lattice units: plate boxes (m, 6) below
    z = 0 and one footprint (k, 4) [x0 y0 x1 y1] per powder layer."""

    plate_boxes: np.ndarray
    footprints: list
    n_layers: int

    def z_min(self):
        return int(self.plate_boxes[:, 2].min()) if len(self.plate_boxes) else 0


def _lattice(value_m, unit_m, what):
    k = int(round(value_m / unit_m))
    if abs(k * unit_m - value_m) > 1e-9 * max(unit_m, abs(value_m)):
        raise ValueError(f"{what} = {value_m} is not a multiple of {unit_m}")
    return k


def chamber_geometry(size_xy, height, plate_thickness, mesh):
    """Full chamber cross-section in every layer on a plate (all lengths in
    metres, multiples of mesh.h_coarse)."""
    unit = _lattice(mesh.h_coarse, mesh.h_fine, "h_coarse")
    nx, ny, nz, tp = (_lattice(v, mesh.h_coarse, w) * unit for v, w in
                      ((size_xy[0], "chamber x"), (size_xy[1], "chamber y"),
                       (height, "chamber height"), (plate_thickness, "plate thickness")))
    plate = np.array([[0, 0, -tp, nx, ny, 0]], dtype=np.int64) if tp else \
        np.zeros((0, 6), dtype=np.int64)
    n_layers = nz // mesh.cells_per_layer
    return Geometry(plate, [np.array([[0, 0, nx, ny]], dtype=np.int64)] * n_layers, n_layers)


def fitted_geometry(part_boxes, plate_box, mesh):
    """Part as a union of boxes (x0 y0 z0 x1 y1 z1, metres above the
    plate) on a plate (x0, y0, x1, y1, thickness)."""
    unit = _lattice(mesh.h_coarse, mesh.h_fine, "h_coarse")
    boxes = np.array([[_lattice(v, mesh.h_coarse, "part box") * unit for v in b]
                      for b in part_boxes], dtype=np.int64).reshape(-1, 6)
    if np.any(boxes[:, 3:] <= boxes[:, :3]):
        raise ValueError("degenerate part box")
    cpl = mesh.cells_per_layer
    n_layers = int(boxes[:, 5].max()) // cpl
    feet = []
    for k in range(n_layers):
        inside = (boxes[:, 2] <= k * cpl) & ((k + 1) * cpl <= boxes[:, 5])
        if not inside.any():
            raise ValueError(f"layer {k} has an empty cross-section")
        feet.append(boxes[inside][:, [0, 1, 3, 4]].copy())
    x0, y0, x1, y1, t = plate_box
    tp = _lattice(t, mesh.h_coarse, "plate thickness") * unit
    plate = np.array([[_lattice(x0, mesh.h_coarse, "plate") * unit,
                       _lattice(y0, mesh.h_coarse, "plate") * unit, -tp,
                       _lattice(x1, mesh.h_coarse, "plate") * unit,
                       _lattice(y1, mesh.h_coarse, "plate") * unit, 0]], dtype=np.int64)
    if tp == 0:
        plate = np.zeros((0, 6), dtype=np.int64)
    return Geometry(plate, feet, n_layers)


def build_coarse_grid(geometry, mesh) -> Forest:
    """Level-0 leaves: the plate active and consolidated, the build volume
    void above it (replaces reference build_coarse_grid, mesh.py:289-333)."""
    mesh.validate()
    depth, cpl = mesh.total_depth, mesh.cells_per_layer
    s0 = 1 << depth
    if (geometry.n_layers * cpl) % s0:
        raise ValueError("part height is not a multiple of h_coarse")
    boxes, act = [b for b in geometry.plate_boxes], [1] * len(geometry.plate_boxes)
    for j in range(geometry.n_layers * cpl // s0):
        layers = range(j * s0 // cpl, (j + 1) * s0 // cpl)
        fp = geometry.footprints[layers[0]]
        if any(not np.array_equal(geometry.footprints[k], fp) for k in layers):
            raise ValueError("cross-section changes inside a coarse slab")
        for r in fp:
            boxes.append([r[0], r[1], j * s0, r[2], r[3], (j + 1) * s0])
            act.append(0)
    b = np.ascontiguousarray(np.array(boxes, dtype=np.int64).reshape(-1, 6))
    a = np.ascontiguousarray(np.array(act, dtype=np.uint8))
    d = _take(lambda out: _lib.load().st_coarse_grid(
        depth, cpl, len(b), b.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), out), "build_coarse_grid")
    return Forest(d["level"], d["anchor"].reshape(-1, 3), d["active"].astype(bool),
                  d["init_consol"].astype(bool), depth, cpl, mesh.h_fine,
                  geometry.z_min(), mesh.dirichlet_bottom, 0, -1, geometry.n_layers)


def advance_layer(forest, history) -> MeshUpdatePlan:
    """Plan the update activating layer ``current_layer + 1``: the layer
    refined to the finest level and activated, settled octets below the
    heat-affected zone coarsened (min r_c >= 0.9), void collapsed, 2:1
    balance restored (replaces reference advance_layer, mesh.py:439-549)."""
    if history is not None and history.epoch != forest.epoch:
        raise ValueError("history epoch does not match forest epoch")
    new_layer = forest.current_layer + 1
    n_layers = getattr(forest, "n_layers", None)
    if n_layers is None and hasattr(forest, "geometry"):
        n_layers = forest.geometry.n_layers
    if n_layers is not None and new_layer >= n_layers:
        raise ValueError("no further layer in the build")
    L = _Leaves(forest)
    rc = None if history is None else np.ascontiguousarray(
        history.r_c, dtype=np.float64).reshape(len(forest.active_cells()), -1)
    d = _take(lambda out: _lib.load().st_plan_layer(
        L.ref, new_layer, _lib.dptr(rc), 0 if rc is None else rc.shape[1], out), "advance_layer")
    ptr, kids = d["group_ptr"], d["group_kids"]
    groups = [(int(r), kids[ptr[g]:ptr[g + 1]].copy()) for g, r in enumerate(d["group_rows"])]
    return MeshUpdatePlan(forest.epoch, new_layer, d["level"], d["anchor"].reshape(-1, 3),
                          d["active"].astype(bool), d["init_consol"].astype(bool),
                          d["same_src"], d["ancestor_src"], groups,
                          [float(x) for x in d["coarsened_min_rc"]])


def apply_update(forest, plan, fields, history, T_0=303.0, old_dofmap=None, new_dofmap=None):
    """Successor forest of a plan with nodal fields and history moved onto
    it (replaces reference apply_update, mesh.py:803-899).  Returns
    (new_forest, new_fields, new_history); plan.transfer_report records
    each new vertex's source."""
    from .material import HistoryField
    if plan.base_epoch != forest.epoch:
        raise ValueError("plan is stale: mesh changed since it was computed")
    new = Forest(plan.level, plan.anchor, plan.active, plan.init_consol, forest.depth,
                 forest.cpl, forest.h_fine, _z_min(forest), _dirichlet_bottom(forest),
                 forest.epoch + 1, plan.new_layer, getattr(forest, "n_layers", None))
    old_dm = old_dofmap if old_dofmap is not None else build_dofmap(forest)
    new_dm = new_dofmap if new_dofmap is not None else build_dofmap(new)
    lib = _lib.load()
    i64 = ctypes.POINTER(ctypes.c_int64)

    def ip(a):
        return a.ctypes.data_as(i64)

    Lo, Ln = _Leaves(forest), _Leaves(new)
    ov = np.ascontiguousarray(old_dm.vertices, dtype=np.int64)
    nv = np.ascontiguousarray(new_dm.vertices, dtype=np.int64)
    ocv = np.ascontiguousarray(old_dm.cell_verts, dtype=np.int32)
    sl, sp, sm = (np.ascontiguousarray(a, dtype=np.int64)
                  for a in (new_dm.slaves, new_dm.slave_ptr, new_dm.slave_masters))
    sw = np.ascontiguousarray(new_dm.slave_weights, dtype=np.float64)
    vals = [np.asarray(getattr(f, "values", f), dtype=np.float64) for f in fields]
    src_f = np.ascontiguousarray(np.stack(vals) if vals else np.zeros((0, len(ov))))
    out_f = np.empty((len(vals), len(nv)))
    source = np.empty(len(nv), dtype=np.int8)
    _lib.check(lib.st_transfer_nodal(
        Lo.ref, ip(ov), len(ov), ocv.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ip(nv),
        len(nv), ip(sp), ip(sl), len(sl), ip(sm), _lib.dptr(sw), len(vals), _lib.dptr(src_f),
        float(T_0), _lib.dptr(out_f), source.ctypes.data_as(ctypes.POINTER(ctypes.c_int8))),
        "apply_update (nodal)")
    plan.transfer_report = TransferReport(source)
    same = np.ascontiguousarray(plan.same_src, dtype=np.int64)
    anc = np.ascontiguousarray(plan.ancestor_src, dtype=np.int64)
    g_rows = np.array([r for r, _ in plan.coarse_groups], dtype=np.int64)
    g_ptr = np.concatenate([[0], np.cumsum([len(k) for _, k in plan.coarse_groups],
                                           dtype=np.int64)]).astype(np.int64)
    g_kids = np.ascontiguousarray(np.concatenate(
        [np.asarray(k, dtype=np.int64) for _, k in plan.coarse_groups])
        if plan.coarse_groups else np.zeros(0, dtype=np.int64))
    rc_old = np.ascontiguousarray(history.r_c, dtype=np.float64)
    rc_new = np.empty((int(new.active.sum()), 2, 2, 2))
    _lib.check(lib.st_transfer_history(
        Lo.ref, Ln.ref, ip(same), ip(anc), len(g_rows), ip(g_rows), ip(g_ptr), ip(g_kids),
        _lib.dptr(rc_old), _lib.dptr(rc_new)), "apply_update (history)")
    new_fields = [NodalField(out_f[k].copy(), new.epoch) for k in range(len(vals))]
    return new, new_fields, HistoryField(rc_new, new.epoch)


# --- structured meshes ---------------------------------------------------------

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


class FittedPart(StructuredBox):
    """A boundary-fitted part on a uniform degree-p lattice: cell row k (z)
    holds the cells i < xext[k] (x), all y; ``xext`` is non-decreasing in
    k, so the part is a base of the full height with overhanging slabs on
    top (BASELINE configs[4]: a 12 mm base plus a thin 75 mm overhang).

    Nodes are those of the active cells, numbered by the reference rule
    (sorted lattice key: x-major, then y, z fastest, mesh.py:712-715): node
    plane I holds rows K >= kmin(I) of every J, so node (I, J, K) has id
    base(I) + J (NZ - kmin(I)) + K with base(I) = offset(I) - kmin(I).
    The bottom node plane z = z0 is Dirichlet, the top cell faces
    radiate; the overhang's underside and the base's side faces are
    adiabatic (the reference's boundary model)."""

    def __init__(self, nx, ny, nz, h, xext, degree=2, origin=(0.0, 0.0, None),
                 dirichlet_bottom=True, top_faces=True, epoch=0):
        super().__init__(nx, ny, nz, h, degree, origin, dirichlet_bottom, top_faces, epoch)
        x = np.asarray(xext, dtype=np.int32).reshape(-1)
        if len(x) != self.nz or x.min() < 1 or x.max() > self.nx or np.any(np.diff(x) < 0):
            raise ValueError("xext: nz non-decreasing extents in [1, nx]")
        self.xext = np.ascontiguousarray(x)
        p = self.degree
        NX, NY, NZ = super().node_dims
        I = np.arange(NX)
        need = np.maximum(-(-I // p), 1)          # cells a row needs to touch plane I
        first = np.searchsorted(self.xext, need)  # first row reaching plane I
        self.kmin = (p * first).astype(np.int64)
        counts = NY * (NZ - self.kmin)
        self.plane_offset = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)

    @property
    def n_vertices(self):
        NX, NY, NZ = self.node_dims
        return int(np.sum(NY * (NZ - self.kmin)))

    @property
    def n_dofs(self):
        return self.n_vertices

    @property
    def n_cells(self):
        return int(self.ny * np.sum(self.xext))

    def active_volume_m3(self):
        return self.n_cells * self.h ** 3

    def node_id(self, I, J, K):
        NZ = self.node_dims[2]
        I = np.asarray(I)
        km = self.kmin[I]
        return self.plane_offset[I] + np.asarray(J) * (NZ - km) + (np.asarray(K) - km)

    def node_lattice(self):
        """(I, J, K) of every node in id order."""
        NX, NY, NZ = self.node_dims
        out = []
        for I in range(NX):
            J, K = np.meshgrid(np.arange(NY), np.arange(self.kmin[I], NZ), indexing="ij")
            out.append(np.stack([np.full(J.size, I), J.ravel(), K.ravel()], axis=1))
        return np.concatenate(out)

    @property
    def is_dirichlet(self):
        m = np.zeros(self.n_vertices, dtype=bool)
        if self.dirichlet_bottom:
            NX, NY, NZ = self.node_dims
            for I in np.flatnonzero(self.kmin == 0):   # planes reaching z = z0
                m[self.plane_offset[I] + np.arange(NY) * NZ] = True
        return m

    def cells(self):
        """(i, j, k) of the active cells in (i, j, k) lexicographic order."""
        i, j, k = np.meshgrid(np.arange(self.nx), np.arange(self.ny), np.arange(self.nz),
                              indexing="ij")
        keep = i < self.xext[k]
        return i[keep], j[keep], k[keep]

    def cell_node_ids(self, cells=None):
        """(m, (p+1)^3) node ids of active cells (the cells() order)."""
        p = self.degree
        i, j, k = self.cells()
        if cells is not None:
            i, j, k = i[cells], j[cells], k[cells]
        l = np.arange(p + 1)
        I = (p * i)[:, None, None, None] + l[None, :, None, None]
        J = (p * j)[:, None, None, None] + l[None, None, :, None]
        K = (p * k)[:, None, None, None] + l[None, None, None, :]
        I, J, K = np.broadcast_arrays(I, J, K)
        return self.node_id(I, J, K).reshape(len(i), -1)

    def to_forest_dofmap(self):
        raise ValueError("FittedPart runs on the structured backend only")
