"""Growing-domain transfer (activation, lineage, nodal + history
transfer, new DoF tables) bit-exact against the reference run that made
tests/golden/growing.npz.  CPU only."""

import numpy as np
import pytest

from fixtures import forest_dofmap, load

from paper_2302_05164_b200.activation import activate_layer, apply_update


@pytest.mark.parametrize("layer", [1, 2])
def test_apply_update_bit_exact(layer):
    d = load("growing")
    old, old_dm, _ = forest_dofmap(d, f"L{layer - 1}/")
    new_ref, new_dm_ref, _ = forest_dofmap(d, f"L{layer}/")
    new, new_dm, fields, hist, rep = apply_update(
        old, new_ref.level, new_ref.anchor, new_ref.active, new_ref.init_consol,
        [d[f"L{layer}/pre_T"]], d[f"L{layer}/pre_rc"], T_0=303.0, new_layer=layer - 1)
    assert np.array_equal(fields[0], d[f"L{layer}/post_T"])
    assert np.array_equal(hist.r_c, d[f"L{layer}/post_rc"])
    assert np.array_equal(rep.vertex_source, d[f"L{layer}/transfer_source"])
    for k in ("vertices", "cell_verts", "slaves", "slave_masters", "slave_weights",
              "is_dirichlet"):
        assert np.array_equal(getattr(new_dm, k), getattr(new_dm_ref, k)), k
    assert new.epoch == old.epoch + 1


def test_activation_marks_exactly_the_new_layer():
    d = load("growing")
    new_ref, _, _ = forest_dofmap(d, "L1/")
    depth, cpl = new_ref.depth, new_ref.cpl
    # deactivate layer 0 cells of the layer-1 forest and re-activate them
    size = np.int64(1) << (depth - new_ref.level.astype(np.int64))
    layer0 = (new_ref.anchor[:, 2] >= 0) & (new_ref.anchor[:, 2] + size <= cpl)
    assert layer0.any()
    pre = new_ref.active.copy()
    pre[layer0] = False
    got = activate_layer(new_ref.level, new_ref.anchor, pre, depth, cpl, 0)
    assert np.array_equal(got, new_ref.active)
    with pytest.raises(ValueError):
        activate_layer(new_ref.level, new_ref.anchor, got, depth, cpl, 0)
