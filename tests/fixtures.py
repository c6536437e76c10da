"""Load the golden fixtures (tests/golden/*.npz, made by the reference)
into oracle tables and product mesh objects.  Runs without the
reference installed."""

import json
import os

import numpy as np

from paper_2302_05164_b200 import params as P
from paper_2302_05164_b200.mesh import DofMap, FaceSet, Forest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def params_from_json(s):
    d = json.loads(str(s))
    return P.ProcessParams(P.MaterialParams(**d["material"]),
                           P.BoundaryParams(**d["boundary"]),
                           P.HeatSourceParams(**d["laser"]), P.MeshParams(),
                           d["T_0"])


def forest_dofmap(d, prefix):
    g = lambda k: d[prefix + k]
    depth, cpl, zmin, dirb, epoch, cur = [int(x) for x in g("meta")]
    forest = Forest(g("level"), g("anchor"), g("active"), g("init_consol"),
                    depth, cpl, float(g("h_fine")), zmin, bool(dirb), epoch, cur)
    dm = DofMap(g("vertices"), g("cell_verts"), g("active_rows"), g("is_slave"),
                g("is_dirichlet"), g("slaves"), g("slave_ptr"), g("slave_masters"),
                g("slave_weights"), float(g("h_fine")))
    faces = FaceSet(g("face_rows"), g("face_offset"), g("face_fsize"))
    return forest, dm, faces


def oracle_tables(forest, dm, faces):
    from cpu_oracle import tables_from_arrays
    rows = dm.active_rows
    pos = np.full(forest.n_cells, -1, dtype=np.int64)
    pos[rows] = np.arange(len(rows))
    return tables_from_arrays(
        dm.n_vertices, dm.cell_verts, forest.size_m(rows),
        forest.anchor[rows] * forest.h_fine, dm.is_slave, dm.is_dirichlet,
        dm.slaves, dm.slave_ptr, dm.slave_masters, dm.slave_weights,
        pos[faces.cell_rows], faces.offset, faces.fsize, forest.size(rows))


def rel(got, ref):
    scale = float(np.max(np.abs(ref))) if np.size(ref) else 0.0
    if np.size(ref) == 0:
        return 0.0
    return float(np.max(np.abs(np.asarray(got) - ref))) / max(scale, 1e-300)


def beam_of(arr):
    return (float(arr[0]), float(arr[1]), float(arr[2]),
            float(arr[3]) if arr[4] > 0 else 0.0)
