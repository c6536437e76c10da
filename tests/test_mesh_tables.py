"""Host mesh tables (DoF numbering, hanging constraints, facets) are
bit-exact with the reference (golden fixtures).  CPU only."""

import numpy as np
import pytest

from fixtures import forest_dofmap, load

from paper_2302_05164_b200.mesh import StructuredBox, build_dofmap, interface_faces

CASES = ["uniform", "refine1", "refine2", "fitted", "stacked"]


def _same_dofmap(a, b):
    for k in ("vertices", "cell_verts", "active_rows", "is_slave", "is_dirichlet",
              "slaves", "slave_ptr", "slave_masters", "slave_weights"):
        x, y = np.asarray(getattr(a, k)), np.asarray(getattr(b, k))
        assert x.shape == y.shape, k
        assert np.array_equal(x, y), k


@pytest.mark.parametrize("name", CASES)
def test_build_dofmap_bit_exact(name):
    forest, dm, faces = forest_dofmap(load("oracle_cases"), name + "/")
    _same_dofmap(build_dofmap(forest), dm)


@pytest.mark.parametrize("name", CASES)
def test_interface_faces_bit_exact(name):
    forest, dm, faces = forest_dofmap(load("oracle_cases"), name + "/")
    fs = interface_faces(forest)
    assert np.array_equal(fs.cell_rows, faces.cell_rows)
    assert np.array_equal(fs.offset, faces.offset)
    assert np.array_equal(fs.fsize, faces.fsize)


@pytest.mark.parametrize("layer", [0, 1, 2])
def test_growing_domain_tables_bit_exact(layer):
    d = load("growing")
    forest, dm, faces = forest_dofmap(d, f"L{layer}/")
    _same_dofmap(build_dofmap(forest), dm)
    fs = interface_faces(forest)
    assert np.array_equal(fs.cell_rows, faces.cell_rows)
    assert np.array_equal(fs.offset, faces.offset)


def test_structured_box_numbering_matches_reference_rule():
    box = StructuredBox(5, 4, 3, 40e-6, degree=1)
    forest, dm = box.to_forest_dofmap()
    ids = box.cell_node_ids()
    assert np.array_equal(ids, dm.cell_verts)
    assert np.array_equal(box.is_dirichlet, dm.is_dirichlet)
    assert box.n_vertices == dm.n_vertices
