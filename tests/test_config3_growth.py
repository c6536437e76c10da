"""BASELINE configs[3] growing domain, all ten layers, on the native table
builder (st_forest.cpp): leaf sets, DoF numbering, hanging constraints,
facets, transferred T / r_c and transfer reports bit-exact (sha256) with
the reference run of tests/golden/make_config3_golden.py.  CPU only."""

import json
import os

import pytest

from growth_rule import layer_record, synthetic_rc, synthetic_T

from paper_2302_05164_b200.mesh import (NodalField, advance_layer, apply_update,
                                        build_coarse_grid, build_dofmap,
                                        chamber_geometry, initial_history, interface_faces)
from paper_2302_05164_b200.params import MeshParams

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "config3_growth.json")


def _check(got, want, layer):
    bad = [k for k in want if k != "coarsened_groups" and got.get(k) != want[k]]
    assert not bad, f"layer {layer}: differs in {bad}"


@pytest.mark.timeout(300)
def test_config3_ten_layers_bit_exact():
    want = json.load(open(GOLD))["layers"]
    mesh = MeshParams(h_coarse=80e-6, n_refine=1, h_powder=40e-6)
    geo = chamber_geometry((2e-3, 2e-3), 10 * 40e-6, 2e-3, mesh)
    forest = build_coarse_grid(geo, mesh)
    history = initial_history(forest)
    dofmap = build_dofmap(forest)
    T = dofmap.distribute(synthetic_T(0, dofmap.vertices_m()))
    _check(layer_record(forest, dofmap, interface_faces(forest), T, history.r_c, None),
           want[0], "coarse")
    for layer in range(geo.n_layers):
        T = dofmap.distribute(synthetic_T(layer, dofmap.vertices_m()))
        rows = forest.active_cells()
        top = (forest.anchor[rows, 2] + forest.size(rows)) * forest.h_fine
        history.r_c[:] = synthetic_rc(layer, history.r_c, top)
        plan = advance_layer(forest, history)
        forest, fields, history = apply_update(forest, plan, [NodalField(T, forest.epoch)],
                                               history, T_0=303.0)
        dofmap = build_dofmap(forest)
        rec = layer_record(forest, dofmap, interface_faces(forest), fields[0].values,
                           history.r_c, plan.transfer_report.vertex_source)
        _check(rec, want[layer + 1], layer)
        assert len(plan.coarsened_min_rc) == want[layer + 1]["coarsened_groups"]
    with pytest.raises(ValueError):
        advance_layer(forest, history)
