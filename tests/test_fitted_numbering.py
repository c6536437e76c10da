"""The fitted-part node numbering (mesh.FittedPart, BASELINE configs[4]'s
base + overhang) is the reference's rule: at p = 1 it equals the vertex
order build_dofmap produces (native builder, pinned bit-exact to the
reference) for the same active cells.  CPU only."""

import numpy as np

from paper_2302_05164_b200.mesh import DofMap, Forest, FittedPart, build_dofmap


def test_fitted_q1_numbering_is_the_reference_rule():
    part = FittedPart(12, 5, 9, 1e-4, [5, 5, 5, 5, 5, 12, 12, 12, 12], degree=1)
    i, j, k = part.cells()
    anchor = np.stack([i, j, k - part.nz], axis=1)
    order = np.lexsort((anchor[:, 2], anchor[:, 1], anchor[:, 0]))
    n = len(i)
    forest = Forest(np.zeros(n, np.int8), anchor[order], np.ones(n, bool), np.ones(n, bool),
                    0, 1, part.h, -part.nz, True)
    dm = build_dofmap(forest)
    lat = part.node_lattice()
    want = np.stack([lat[:, 0], lat[:, 1], lat[:, 2] - part.nz], axis=1)
    assert dm.n_vertices == part.n_vertices
    assert np.array_equal(dm.vertices, want)
    # the cells' corner ids agree too (corner order ix*4 + iy*2 + iz)
    assert np.array_equal(dm.cell_verts, part.cell_node_ids()[order])
    assert np.array_equal(dm.is_dirichlet, part.is_dirichlet)
    assert len(dm.slaves) == 0


def test_fitted_plane_layout():
    part = FittedPart(10, 3, 8, 1e-4, [4, 4, 4, 4, 10, 10, 10, 10], degree=2)
    assert part.kmin[8] == 0 and part.kmin[9] == 8 and part.kmin[-1] == 8
    ids = part.cell_node_ids()
    assert len(np.unique(ids)) == part.n_vertices
