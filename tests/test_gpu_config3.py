"""BASELINE configs[3] (growing domain with cool-down) on the B200 path,
against the reference's own run (tests/golden/make_config3_windows.py):

* layer 0 after activation: step criteria, then the first 1000 explicit
  scan steps (dt = 1 us, 70 W hatch) -- T and r_c <= 1e-9;
* 20 backward-Euler steps (1 ms, krylov_tol 1e-13, Jacobi) from the
  reference's state after those 1000 steps -- T <= 1e-9, Newton counts
  equal, CG counts within one per step;
* two layers of the full pipeline (native planner + transfer, operator
  rebuild, criteria, scan, cool-down) with the per-layer vertex counts of
  the reference (tests/golden/config3_growth.json).
"""

import json
import os

import numpy as np
import pytest

from fixtures import load, rel

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.physics import LayerPath, flatten_schedule
import workloads as w

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def layer0():
    mesh, geo, params, settings = w.config3_setup(krylov_tol=1e-13)
    state = w.config3_initial_state(mesh, geo, params, settings)
    w.advance_mesh(state, params, settings)
    paths = w.config3_layer_paths(geo, mesh)
    return state, paths, params, settings


def test_config3_layer0_scan_window(layer0):
    state, paths, params, settings = layer0
    g = load("config3_windows")
    assert state.dofmap.n_vertices == int(g["n_vertices"])
    crit = st.compute_step_criteria(state.op, settings)
    assert abs(crit.dt_stability / float(g["dt_stability"]) - 1.0) < 1e-7
    dts, beams = flatten_schedule(paths[0], 1e-6, 1000)
    op = state.op
    op.set_state(state.T, state.history.r_c)
    fail, _, _ = op.run_explicit(dts, beams)
    assert fail == 0
    T, rc = op.get_state()
    assert rel(T, g["T_scan1000"]) < 1e-9
    assert float(np.max(np.abs(rc.reshape(-1) - g["rc_scan1000"].reshape(-1)))) < 1e-9
    assert T.max() > 2000.0  # the melt pool is there


def test_config3_backward_euler_window(layer0):
    state, paths, params, settings = layer0
    g = load("config3_windows")
    s = st.SimulationState(state.forest, state.dofmap, state.op, g["T_scan1000"].copy(),
                           st.HistoryField(g["rc_scan1000"].copy(), state.forest.epoch))
    stats = st.run_cooldown_phase(s, LayerPath(0, paths[0].z, [], 20e-3), 1e-6, settings)
    n, newton, krylov = (int(x) for x in g["be_iters"])
    assert stats.n_steps == n == 20
    assert stats.newton_iters == newton
    assert abs(stats.krylov_iters - krylov) <= n
    assert rel(s.T, g["T_be20"]) < 1e-9
    assert float(np.max(np.abs(s.history.r_c - g["rc_be20"]))) < 1e-9


def test_config3_two_layer_pipeline():
    want = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                       "config3_growth.json")))["layers"]
    state, recs = w.run_config3_build(n_layers=2, scan_steps=3000, cool_time=5e-3)
    for k, r in enumerate(recs):
        assert r["n_cells"] == int(np.sum(state.forest.active)) or k < len(recs) - 1
        assert r["scan_steps"] == 3000 and r["cool_steps"] == 5
        assert r["t_max"] > 1000.0
    assert state.dofmap.n_vertices == want[2]["n_vertices"]
    assert np.all(np.isfinite(state.T)) and state.T.max() < 5000.0
    assert state.forest.current_layer == 1
