"""Synthetic per-layer state of the config-3 growth check (shared by the
golden generator, which runs the reference, and the tests, which run the
native builder): a hot spot that moves with the layer and a consolidation
history that is settled (r_c = 1) below the heat-affected zone, so the
planner's coarsening gate engages from layer 5 on."""

import hashlib

import numpy as np

H_POWDER = 40e-6


def synthetic_T(layer, verts_m):
    xc = 0.2e-3 + 0.15e-3 * layer
    r2 = (verts_m[:, 0] - xc) ** 2 + (verts_m[:, 1] - 1.0e-3) ** 2
    return 303.0 + 1500.0 * np.exp(-r2 / (2e-4) ** 2)


def synthetic_rc(layer, rc, cell_top_m):
    u = np.random.default_rng(100 + layer).uniform(0.0, 1.0, rc.shape)
    settled = cell_top_m < (layer - 4) * H_POWDER + 1e-9
    return np.maximum(rc, np.where(settled[:, None, None, None], 1.0, u))


def digest(a):
    a = np.ascontiguousarray(a)
    if a.dtype == bool:
        a = a.astype(np.uint8)
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]


def layer_record(forest, dofmap, faces, T, r_c, source):
    arrs = {
        "level": np.asarray(forest.level, np.int8), "anchor": np.asarray(forest.anchor, np.int64),
        "active": np.asarray(forest.active, bool), "init_consol": np.asarray(forest.init_consol, bool),
        "vertices": np.asarray(dofmap.vertices, np.int64),
        "cell_verts": np.asarray(dofmap.cell_verts, np.int32),
        "is_slave": np.asarray(dofmap.is_slave, bool),
        "is_dirichlet": np.asarray(dofmap.is_dirichlet, bool),
        "slaves": np.asarray(dofmap.slaves, np.int64),
        "slave_ptr": np.asarray(dofmap.slave_ptr, np.int64),
        "slave_masters": np.asarray(dofmap.slave_masters, np.int64),
        "slave_weights": np.asarray(dofmap.slave_weights, np.float64),
        "face_rows": np.asarray(faces.cell_rows, np.int64),
        "face_offset": np.asarray(faces.offset, np.int64),
        "face_fsize": np.asarray(faces.fsize, np.int64),
        "T": np.asarray(T, np.float64), "r_c": np.asarray(r_c, np.float64),
    }
    if source is not None:
        arrs["transfer_source"] = np.asarray(source, np.int8)
    rec = {k: digest(v) for k, v in arrs.items()}
    rec["n_cells"] = int(len(forest.level))
    rec["n_vertices"] = int(len(dofmap.vertices))
    rec["n_slaves"] = int(len(dofmap.slaves))
    return rec
