"""CUDA operator vs the reference (golden vectors) and the oracle.

Tolerances: the reference's own dense cross-checks use 1e-12 relative
(test_operators.py:22); the time-stepped fields use the north-star bar
max|dT|/max|T_ref| <= 1e-9."""

import numpy as np
import pytest

from fixtures import beam_of, forest_dofmap, load, oracle_tables, params_from_json, rel

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.physics import BeamState

pytestmark = pytest.mark.gpu
CASES = ["uniform", "refine1", "refine2", "fitted", "stacked"]


def _beam(arr):
    return BeamState(np.array([arr[0], arr[1]]), float(arr[2]), float(arr[3]), bool(arr[4]))


@pytest.fixture(scope="module")
def oc():
    return load("oracle_cases")


@pytest.mark.parametrize("det", [True, False])
@pytest.mark.parametrize("name", CASES)
def test_operator_methods_match_reference(oc, name, det):
    forest, dm, _ = forest_dofmap(oc, name + "/")
    params = params_from_json(oc[name + "/params"])
    op = st.ThermalOperator(forest, dm, params, st.SolverSettings(deterministic=det))
    g = lambda k: oc[f"{name}/{k}"]
    T, rc, dt = g("T"), g("r_c"), float(g("dt"))
    beam = _beam(g("beam"))
    tol = 1e-12
    assert rel(op.evaluate_rhs(T, rc, beam), g("rhs_beam")) < tol
    assert rel(op.evaluate_rhs(T, rc, None), g("rhs_nobeam")) < tol
    assert rel(op.evaluate_rhs(T, rc, None, faces=False, source=False), g("rhs_diff")) < tol
    assert rel(op.evaluate_rhs(T, rc, None, diffusion=False, source=False), g("rhs_faces")) < tol
    assert rel(op.evaluate_rhs(T, rc, beam, diffusion=False, faces=False), g("rhs_src")) < tol
    assert rel(op.evaluate_rhs(T, None, None, faces=False, source=False, frozen_k=20.0),
               g("rhs_frozen")) < tol
    assert rel(op.lumped_capacity(), g("lumped")) < tol
    assert rel(op.apply_mass(g("v")), g("mass_v")) < tol
    assert rel(op.apply_jacobian(g("v"), T, rc, dt), g("jac_v")) < tol
    assert rel(op.jacobian_diagonal(T, rc, dt), g("jac_diag")) < tol
    assert rel(op.explicit_fused_step(T, 2e-7, rc, beam), g("step")) < 1e-14
    h = st.HistoryField(rc.copy(), op.epoch)
    op.update_history(h, T)
    assert rel(h.r_c, g("history")) < 1e-14
    # Dirichlet rows identity, slave rows zero (test_operators.py:165)
    out = op.apply_jacobian(g("v"), T, rc, dt)
    assert np.array_equal(out[dm.is_dirichlet], g("v")[dm.is_dirichlet])
    assert np.all(out[dm.is_slave] == 0.0)


def test_epoch_guard(oc):
    forest, dm, _ = forest_dofmap(oc, "refine2/")
    params = params_from_json(oc["refine2/params"])
    op = st.ThermalOperator(forest, dm, params, st.SolverSettings())
    h = st.HistoryField(oc["refine2/r_c"].copy(), op.epoch + 1)
    with pytest.raises(ValueError):
        op.update_history(h, oc["refine2/T"])


def _config0_problem():
    from paper_2302_05164_b200.mesh import StructuredBox
    h = 31.25e-6
    box = StructuredBox(64, 64, 32, h, degree=1)
    forest, dm = box.to_forest_dofmap()
    mat = st.MaterialParams(k_p=6.7, k_m=6.7, k_s=6.7, rho=4430.0, c=526.0)
    bnd = st.BoundaryParams(emissivity=0.0, T_inf=300.0, T_v=1e9)
    las = st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0, scan_velocity=1.0)
    params = st.ProcessParams(mat, bnd, las, st.MeshParams(h_coarse=h, n_refine=0, h_powder=h))
    T0 = 300.0 + np.random.default_rng(0).uniform(0.0, 1.0, dm.n_vertices)
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 1e-3, 2e-4, 1e-3, 1.0, 70.0)], 0.0)
    return forest, dm, params, T0, lp


def test_config0_200_steps_match_reference():
    g = load("config0")
    forest, dm, params, T0, lp = _config0_problem()
    op = st.ThermalOperator(forest, dm, params, st.SolverSettings())
    hist = st.initial_history(forest)
    state = st.SimulationState(forest, dm, op, T0.copy(), hist)
    stats = st.run_scan_phase(state, lp, 1e-6)
    assert stats.n_steps == 200
    assert rel(state.T, g["T200"]) <= 1e-9
    assert np.all(state.history.r_c == 1.0)
    assert stats.t_max_seen == pytest.approx(float(g["T200"].max()), rel=1e-6) or \
        stats.t_max_seen >= float(g["T200"].max())


def test_config0_per_step_api_matches_reference():
    g = load("config0")
    forest, dm, params, T0, lp = _config0_problem()
    op = st.ThermalOperator(forest, dm, params, st.SolverSettings())
    hist = st.initial_history(forest)
    T = T0.copy()
    for step in range(1, 21):
        b = st.layer_beam_state(lp, (step - 1) * 1e-6)
        T = op.explicit_fused_step(T, 1e-6, hist.r_c, b)
        op.update_history(hist, T)
        if step == 1:
            assert rel(T, g["T1"]) <= 1e-12
    assert rel(T, g["T20"]) <= 1e-10


def test_growing_mesh_explicit_window_and_backward_euler():
    d = load("growing")
    params = params_from_json(d["params"])
    forest, dm, _ = forest_dofmap(d, "L2/")
    s = st.SolverSettings(explicit_cooldown_steps=0, dt_implicit=1e-3, krylov_tol=1e-13)
    op = st.ThermalOperator(forest, dm, params, s)
    x0, y0, x1, y1, v, pw, z = d["expl/seg"]
    lp = st.LayerPath(2, float(z), [st.Segment(x0, y0, x1, y1, v, pw)], 0.0)
    hist = st.HistoryField(d["expl/rc0"].copy(), forest.epoch)
    state = st.SimulationState(forest, dm, op, d["expl/T0"].copy(), hist)
    stats = st.run_scan_phase(state, lp, 1e-6)
    assert stats.n_steps == int(d["expl/n_steps"])
    assert rel(state.T, d["expl/T"]) <= 1e-9
    assert rel(state.history.r_c, d["expl/rc"]) <= 1e-12
    # backward Euler steps from the end-of-scan field (krylov_tol 1e-13)
    op.set_state(d["be/T0"], d["be/rc0"])
    for i in range(3):
        out = op.implicit_step(1e-3, s)
        assert out is not None
        assert out[0] == d["be/iters"][i][0]
        assert abs(out[1] - d["be/iters"][i][1]) <= 1
        op.finish_implicit_step()
        T, rc = op.get_state()
        assert rel(T, d[f"be/T{i + 1}"]) <= 1e-10
    assert rel(rc, d["be/rc_final"].reshape(-1)) <= 1e-12
    assert rel(op.apply_jacobian(d["be/v"], d["be/T0"], d["be/rc0"], 1e-3), d["be/jac_v"]) < 1e-12
    assert rel(op.jacobian_diagonal(d["be/T0"], d["be/rc0"], 1e-3), d["be/jac_diag"]) < 1e-12


def test_cooldown_phase_matches_oracle():
    """run_cooldown_phase (explicit pre-phase + BE) vs the oracle."""
    from cpu_oracle import OracleOperator, implicit_step, run_explicit
    d = load("growing")
    params = params_from_json(d["params"])
    forest, dm, faces = forest_dofmap(d, "L2/")
    s = st.SolverSettings(explicit_cooldown_steps=5, dt_implicit=1e-3, krylov_tol=1e-13)
    op = st.ThermalOperator(forest, dm, params, s)
    hist = st.HistoryField(d["be/rc0"].copy(), forest.epoch)
    state = st.SimulationState(forest, dm, op, d["be/T0"].copy(), hist)
    lp = st.LayerPath(2, 8e-5, [], 2.5e-3)
    stats = st.run_cooldown_phase(state, lp, 1e-6, s)
    orc = OracleOperator(oracle_tables(forest, dm, faces), params)
    T, rc = run_explicit(orc, d["be/T0"], d["be/rc0"], [1e-6] * 5, [[]] * 5)
    elapsed = 5e-6
    while 2.5e-3 - elapsed > 1e-9 * 1e-3:
        dt = min(1e-3, 2.5e-3 - elapsed)
        T, nn, nk = implicit_step(orc, T, rc, dt, s)
        T[dm.is_dirichlet] = params.boundary.T_inf
        rc = orc.update_history(rc, T)
        elapsed += dt
    assert stats.n_steps == 5 + 3
    assert rel(state.T, T) <= 1e-9
    assert rel(state.history.r_c, rc) <= 1e-12


def test_instability_is_reported_at_the_failing_step():
    forest, dm, params, T0, lp = _config0_problem()
    op = st.ThermalOperator(forest, dm, params, st.SolverSettings())
    hist = st.initial_history(forest)
    state = st.SimulationState(forest, dm, op, T0.copy(), hist)
    # a 20 mm virtual track: 20 steps of 1 ms, ~20x the stability bound
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 1e-3, 2e-2, 1e-3, 1.0, 70.0)], 0.0)
    with pytest.raises(st.InstabilityError) as ei:
        st.run_scan_phase(state, lp, 1e-3)
    e = ei.value
    assert e.step >= 1 and not (np.isfinite(e.t_extreme) and e.t_extreme <= 1e7)
    # the reported state is the diverged one
    m = float(np.max(np.abs(state.T)))
    assert not np.isfinite(m) or m > 1e7


def test_multi_beam_source_is_the_sum_of_single_beams(oc):
    forest, dm, _ = forest_dofmap(oc, "refine2/")
    params = params_from_json(oc["refine2/params"])
    op = st.ThermalOperator(forest, dm, params, st.SolverSettings())
    T, rc = oc["refine2/T"], oc["refine2/r_c"]
    b1 = _beam(oc["refine2/beam"])
    b2 = BeamState(b1.position + np.array([1e-4, -5e-5]), b1.z_top, 50.0, True)
    both = op.evaluate_rhs(T, rc, [b1, b2], diffusion=False, faces=False)
    one = op.evaluate_rhs(T, rc, b1, diffusion=False, faces=False)
    two = op.evaluate_rhs(T, rc, b2, diffusion=False, faces=False)
    assert rel(both, one + two) < 1e-14
