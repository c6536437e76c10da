"""The oracle restatement against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from cpu_oracle import (OracleOperator, conductivity, conductivity_derivative,
                        gaussian_source, implicit_step, liquid_fraction,
                        run_explicit, surface_flux)
from fixtures import beam_of, forest_dofmap, load, oracle_tables, params_from_json, rel

from paper_2302_05164_b200 import params as P

CASES = ["uniform", "refine1", "refine2", "fitted", "stacked"]


@pytest.fixture(scope="module")
def oc():
    return load("oracle_cases")


@pytest.mark.parametrize("name", CASES)
def test_oracle_operator_matches_reference(oc, name):
    forest, dm, faces = forest_dofmap(oc, name + "/")
    params = params_from_json(oc[name + "/params"])
    op = OracleOperator(oracle_tables(forest, dm, faces), params)
    g = lambda k: oc[f"{name}/{k}"]
    T, rc, beam, dt = g("T"), g("r_c"), beam_of(g("beam")), float(g("dt"))
    assert rel(op.evaluate_rhs(T, rc, [beam]), g("rhs_beam")) < 1e-13
    assert rel(op.evaluate_rhs(T, rc, []), g("rhs_nobeam")) < 1e-13
    assert rel(op.evaluate_rhs(T, rc, [], faces=False, source=False), g("rhs_diff")) < 1e-13
    assert rel(op.evaluate_rhs(T, rc, [], diffusion=False, source=False), g("rhs_faces")) < 1e-13
    assert rel(op.evaluate_rhs(T, rc, [beam], diffusion=False, faces=False), g("rhs_src")) < 1e-13
    assert rel(op.evaluate_rhs(T, None, [], faces=False, source=False, frozen_k=20.0),
               g("rhs_frozen")) < 1e-13
    assert rel(op.lumped_capacity(), g("lumped")) < 1e-14
    assert rel(op.apply_mass(g("v")), g("mass_v")) < 1e-13
    assert rel(op.apply_jacobian(g("v"), T, rc, dt), g("jac_v")) < 1e-13
    assert rel(op.jacobian_diagonal(T, rc, dt), g("jac_diag")) < 1e-13
    assert rel(op.explicit_step(T, 2e-7, rc, [beam]), g("step")) < 1e-15
    assert rel(op.update_history(rc, T), g("history")) < 1e-14


def test_oracle_pointwise_laws_bitwise():
    d = load("pointwise")
    mat, bp = P.MaterialParams(), P.BoundaryParams()
    T, rc = d["T"], d["rc"]
    assert np.array_equal(liquid_fraction(T, mat), d["g"])
    assert np.array_equal(conductivity(T, rc, mat), d["k"])
    assert np.array_equal(conductivity_derivative(T, mat), d["dk"])
    assert np.array_equal(surface_flux(T, bp, mat.c), d["rad"] + d["evap"])
    hs = P.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=100.0)
    pts = d["pts"]
    q = gaussian_source(pts[:, 0], pts[:, 1], pts[:, 2], (1e-4, 2e-4, 40e-6, 100.0), hs)
    assert np.array_equal(q, d["src"])


def test_oracle_growing_window_explicit_and_implicit():
    d = load("growing")
    params = params_from_json(d["params"])
    forest, dm, faces = forest_dofmap(d, "L2/")
    op = OracleOperator(oracle_tables(forest, dm, faces), params)
    from paper_2302_05164_b200.physics import LayerPath, Segment, flatten_schedule
    from cpu_oracle import beam_tuple
    x0, y0, x1, y1, v, pw, z = d["expl/seg"]
    lp = LayerPath(2, float(z), [Segment(x0, y0, x1, y1, v, pw)], 0.0)
    n = int(d["expl/n_steps"])
    dts, beams = flatten_schedule(lp, 1e-6, n)
    T, rc = run_explicit(op, d["expl/T0"], d["expl/rc0"], dts,
                         [[beam_tuple(b) for b in row] for row in beams])
    assert rel(T, d["expl/T"]) < 1e-13
    assert np.array_equal(rc, d["expl/rc"]) or rel(rc, d["expl/rc"]) < 1e-14

    from paper_2302_05164_b200.params import SolverSettings
    s = SolverSettings(explicit_cooldown_steps=0, dt_implicit=1e-3, krylov_tol=1e-13)
    T, rc = d["be/T0"].copy(), d["be/rc0"].copy()
    for i in range(3):
        T, nn, nk = implicit_step(op, T, rc, 1e-3, s)
        T[dm.is_dirichlet] = params.boundary.T_inf
        assert (nn, nk) == tuple(d["be/iters"][i])
        assert rel(T, d[f"be/T{i + 1}"]) < 1e-12
        rc = op.update_history(rc, T)
    assert rel(op.apply_jacobian(d["be/v"], d["be/T0"], d["be/rc0"], 1e-3), d["be/jac_v"]) < 1e-13
    assert rel(op.jacobian_diagonal(d["be/T0"], d["be/rc0"], 1e-3), d["be/jac_diag"]) < 1e-13


def test_schedule_matches_reference():
    d = load("pointwise")
    from paper_2302_05164_b200.physics import LayerPath, Segment, layer_beam_state
    segs = [Segment(*row) for row in d["hatch"]]
    lp = LayerPath(0, 4e-5, segs, 1e-4)
    for t, pos, on, pw in zip(d["taus"], d["beam_pos"], d["beam_on"], d["beam_power"]):
        b = layer_beam_state(lp, float(t))
        assert bool(b.active) == bool(on) and b.power == pw
        assert np.array_equal(b.position, pos)
