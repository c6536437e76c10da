"""Growing domain: new-layer activation, lineage and field/history transfer.

Restates the epoch-change half of the reference's mesh update so that a
B200 run can move (T, r_c) from one mesh epoch to the next and rebuild
its operator tables:

* :func:`activate_layer` — step 2 of ``advance_layer`` (mesh.py:470-475):
  every leaf lying inside the new layer becomes active powder;
* :func:`lineage` — same / ancestor / descendant relation of the new leaf
  set against the old one (mesh.py:552-602);
* :func:`apply_update` — successor forest plus nodal transfer (exact copy
  at surviving vertices, trilinear interpolation from the old containing
  cell, T_0 at fresh vertices) and history transfer (octant copy downward,
  octant mean upward), mesh.py:803-899.

The refinement planner itself (refine / coarsen / balance,
mesh.py:439-549) stays with the caller.  Everything
here is bit-exact with the reference (tests/test_activation.py against
the golden growing-domain fixture).
"""

from dataclasses import dataclass

import numpy as np

from .material import HistoryField
from .mesh import CORNER_OFFSETS, Forest, _hanging_host_cell, build_dofmap, pack_coords


def activate_layer(level, anchor, active, depth, cpl, new_layer):
    """Mark every leaf inside layer ``new_layer`` active (mesh.py:470-475)."""
    level = np.asarray(level, dtype=np.int64)
    size = np.int64(1) << (depth - level)
    z0, z1 = new_layer * cpl, (new_layer + 1) * cpl
    inside = (anchor[:, 2] >= z0) & (anchor[:, 2] + size <= z1)
    if np.any(level[inside] != depth):
        raise ValueError("new layer is not refined to the finest level")
    if np.any(active[inside]):
        raise ValueError("new layer already active")
    out = np.array(active, dtype=bool, copy=True)
    out[inside] = True
    return out


def lineage(old, level, anchor):
    """(same_src, ancestor_src, coarse_groups) of the new leaves vs ``old``."""
    level = np.asarray(level)
    n = len(level)
    same = np.full(n, -1, dtype=np.int64)
    anc = np.full(n, -1, dtype=np.int64)
    for ell in np.unique(level):
        rows = np.flatnonzero(level == ell)
        same[rows] = old.lookup(int(ell), anchor[rows])
    todo = np.flatnonzero(same == -1)
    for ell_old in sorted(old._levels()):
        if todo.size == 0:
            break
        finer = todo[level[todo] > ell_old]
        if finer.size == 0:
            continue
        s = np.int64(1) << (old.depth - ell_old)
        hit = old.lookup(ell_old, (anchor[finer] // s) * s)
        got = hit >= 0
        anc[finer[got]] = hit[got]
        todo = np.flatnonzero((same == -1) & (anc == -1))
    groups = []
    rows = np.flatnonzero((same == -1) & (anc == -1))
    if rows.size:
        members = {int(r): [] for r in rows}
        for ell_new in np.unique(level[rows]):
            sub = rows[level[rows] == ell_new]
            s = np.int64(1) << (old.depth - int(ell_new))
            keys = pack_coords(anchor[sub])
            o = np.argsort(keys, kind="stable")
            sk, sr = keys[o], sub[o]
            cand = pack_coords((old.anchor // s) * s)
            pos = np.searchsorted(sk, cand)
            ok = pos < len(sk)
            ok[ok] &= sk[pos[ok]] == cand[ok]
            ok &= old.level > ell_new
            for old_row in np.flatnonzero(ok):
                members[int(sr[pos[old_row]])].append(old_row)
        for r in sorted(members):
            kids = np.array(sorted(members[r]), dtype=np.int64)
            if kids.size < 8:
                raise ValueError("coarsened leaf without a complete octet")
            groups.append((int(r), kids))
    return same, anc, groups


@dataclass
class TransferReport:
    vertex_source: np.ndarray   # 0 copied, 1 interpolated, 2 fresh (T_0)


def _trilinear_weights(frac):
    """(m, 8) corner weights, multiplied in corner/axis order like the
    reference's scalar loop (mesh.py:859-863)."""
    w = np.ones((len(frac), 8))
    for ci in range(8):
        for d in range(3):
            w[:, ci] = w[:, ci] * (frac[:, d] if CORNER_OFFSETS[ci, d] else (1.0 - frac[:, d]))
    return w


def apply_update(old, level, anchor, active, init_consol, fields, history, T_0=303.0,
                 new_layer=None, old_dofmap=None, new_dofmap=None):
    """Successor forest of a planned leaf set plus the data transfer.

    ``fields`` are nodal arrays on ``old``'s DoF map; ``history`` is the
    (n_active, 2, 2, 2) r_c array (or a HistoryField).  Returns
    (new_forest, new_dofmap, new_fields, new_history, report)."""
    level = np.asarray(level, dtype=np.int8)
    anchor = np.asarray(anchor, dtype=np.int64)
    new = Forest(level, anchor, active, init_consol, old.depth, old.cpl, old.h_fine,
                 old.z_min_lattice, old.dirichlet_bottom, old.epoch + 1,
                 old.current_layer + 1 if new_layer is None else new_layer)
    old_dm = old_dofmap or build_dofmap(old)
    new_dm = new_dofmap or build_dofmap(new)
    rc_old = history.r_c if isinstance(history, HistoryField) else np.asarray(history)

    old_keys = pack_coords(old_dm.vertices)
    new_keys = pack_coords(new_dm.vertices)
    pos = np.searchsorted(old_keys, new_keys)
    ok = pos < len(old_keys)
    copied = ok.copy()
    copied[ok] = old_keys[pos[ok]] == new_keys[ok]
    todo = np.flatnonzero(~copied)
    irow, irel = _hanging_host_cell(old, new_dm.vertices[todo])
    interp = irow >= 0
    source = np.full(new_dm.n_vertices, 2, dtype=np.int8)
    source[copied] = 0
    source[todo[interp]] = 1

    old_pos = np.full(old.n_cells, -1, dtype=np.int64)
    old_pos[old_dm.active_rows] = np.arange(len(old_dm.active_rows))
    it = todo[interp]
    cells = irow[interp]
    frac = irel[interp] / old.size(cells).astype(np.int64)[:, None]
    W = _trilinear_weights(frac)
    corners = old_dm.cell_verts[old_pos[cells]]
    new_fields = []
    for f in fields:
        f = np.asarray(f, dtype=np.float64)
        vals = np.full(new_dm.n_vertices, T_0, dtype=np.float64)
        vals[copied] = f[pos[copied]]
        acc = np.zeros(len(it))
        cv = f[corners]
        for ci in range(8):
            acc = acc + W[:, ci] * cv[:, ci]
        vals[it] = acc
        new_dm.distribute(vals)
        new_fields.append(vals)

    same, anc, groups = lineage(old, level, anchor)
    new_rows = new.active_cells()
    r_c = np.zeros((len(new_rows), 2, 2, 2))
    parents = {r: kids for r, kids in groups}
    for i, r in enumerate(new_rows):
        r = int(r)
        if same[r] >= 0:
            if old.active[same[r]]:
                r_c[i] = rc_old[old_pos[same[r]]]
            continue
        a = int(anc[r])
        if a >= 0:
            if old.active[a]:
                s_anc = int(old.size(a))
                mid = anchor[r] + int(new.size(r)) // 2
                octant = (mid - old.anchor[a]) * 2 // s_anc
                r_c[i] = rc_old[old_pos[a]][tuple(octant)]
            continue
        kids = parents[r]
        if len(kids) != 8 or not np.all(old.active[kids]):
            raise ValueError("active coarsening must merge exactly one level")
        s_par = int(new.size(r))
        for kid in kids:
            off = (old.anchor[kid] - anchor[r]) * 2 // s_par
            r_c[i][tuple(off)] = rc_old[old_pos[int(kid)]].mean()
    return new, new_dm, new_fields, HistoryField(r_c, new.epoch), TransferReport(source)
