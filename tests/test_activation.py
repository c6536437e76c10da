"""Growing-domain pipeline on the native table builder (st_forest.cpp):
layer plan (refine / activate / coarsen / collapse / 2:1 balance), nodal
and history transfer and the new DoF tables, bit-exact against the
reference run that made tests/golden/growing.npz.  CPU only."""

import numpy as np
import pytest

from fixtures import forest_dofmap, load

from paper_2302_05164_b200.material import HistoryField
from paper_2302_05164_b200.mesh import (NodalField, advance_layer, apply_update,
                                        build_dofmap, interface_faces)


@pytest.mark.parametrize("layer", [1, 2])
def test_layer_advance_bit_exact(layer):
    d = load("growing")
    old, old_dm, _ = forest_dofmap(d, f"L{layer - 1}/")
    ref, ref_dm, ref_faces = forest_dofmap(d, f"L{layer}/")
    hist = HistoryField(d[f"L{layer}/pre_rc"].copy(), old.epoch)
    plan = advance_layer(old, hist)
    for k in ("level", "anchor", "active", "init_consol"):
        assert np.array_equal(getattr(plan, k), getattr(ref, k)), k
    new, fields, new_hist = apply_update(
        old, plan, [NodalField(d[f"L{layer}/pre_T"].copy(), old.epoch)], hist, T_0=303.0)
    assert np.array_equal(fields[0].values, d[f"L{layer}/post_T"])
    assert np.array_equal(new_hist.r_c, d[f"L{layer}/post_rc"])
    assert np.array_equal(plan.transfer_report.vertex_source, d[f"L{layer}/transfer_source"])
    dm = build_dofmap(new)
    for k in ("vertices", "cell_verts", "active_rows", "is_slave", "slaves", "slave_ptr",
              "slave_masters", "slave_weights", "is_dirichlet"):
        assert np.array_equal(getattr(dm, k), getattr(ref_dm, k)), k
    fs = interface_faces(new)
    assert np.array_equal(fs.cell_rows, ref_faces.cell_rows)
    assert np.array_equal(fs.offset, ref_faces.offset)
    assert new.epoch == old.epoch + 1 and new.current_layer == old.current_layer + 1


def test_advance_rejects_stale_history():
    d = load("growing")
    old, _, _ = forest_dofmap(d, "L0/")
    hist = HistoryField(d["L1/pre_rc"].copy(), old.epoch + 1)
    with pytest.raises(ValueError):
        advance_layer(old, hist)


def test_plan_activates_exactly_the_new_layer():
    d = load("growing")
    old, _, _ = forest_dofmap(d, "L0/")
    plan = advance_layer(old, None)
    depth, cpl = old.depth, old.cpl
    z0 = (old.current_layer + 1) * cpl
    size = np.int64(1) << (depth - plan.level.astype(np.int64))
    in_layer = (plan.anchor[:, 2] >= z0) & (plan.anchor[:, 2] + size <= z0 + cpl)
    assert in_layer.any() and np.all(plan.level[in_layer] == depth)
    assert np.all(plan.active[in_layer])
    # nothing above the new layer is active
    assert not np.any(plan.active & (plan.anchor[:, 2] >= z0 + cpl))
