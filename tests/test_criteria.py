"""Step criteria: rho(C~^-1 K) by power
iteration at the frozen stiffest conductivity (timestepping.py:49-99).

Golden values come from the reference's own compute_step_criteria
(tests/golden/make_criteria_golden.py) on the five oracle meshes and the
uniform plate of test_timestepping.py::test_step_criteria_on_a_uniform_plate.
"""

import numpy as np
import pytest

from cpu_oracle import OracleOperator, step_criteria_rho
from fixtures import forest_dofmap, load, oracle_tables, params_from_json

import paper_2302_05164_b200 as st

CASES = ["uniform", "refine1", "refine2", "fitted", "stacked", "plate"]


@pytest.fixture(scope="module")
def gold():
    d = load("criteria")
    oc = load("oracle_cases")
    return d, oc


def _mesh(gold, name):
    d, oc = gold
    src = d if name == "plate" else oc
    forest, dm, faces = forest_dofmap(src, name + "/")
    return forest, dm, faces, params_from_json(src[name + "/params"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_step_criteria_match_reference(gold, name):
    d, _ = gold
    forest, dm, faces, params = _mesh(gold, name)
    op = OracleOperator(oracle_tables(forest, dm, faces), params)
    rho, applies = step_criteria_rho(op)
    assert applies == len(d[name + "/lams"])
    assert abs(rho - float(d[name + "/rho"])) <= 1e-12 * float(d[name + "/rho"])


def test_plate_rho_is_the_analytic_bound(gold):
    d, _ = gold
    # dt = rho c h^2 / (2 k) (test_timestepping.py:62-70), at the reference's 1e-6
    assert float(d["plate/dt_stability"]) == pytest.approx(float(d["plate/analytic"]), rel=1e-6)


def test_power_iteration_host_mirror_matches_oracle():
    """timestepping.estimate_spectral_radius (the host mirror callers use
    with their own apply callback) is the reference's iteration."""
    from cpu_oracle import spectral_radius
    A = np.diag(np.linspace(1.0, 10.0, 50))
    got = st.timestepping.estimate_spectral_radius(lambda v: A @ v, 50)
    ref, _ = spectral_radius(lambda v: A @ v, 50)
    assert got == ref


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_step_criteria_match_reference(gold, name):
    """Device power iteration (st_spectral_radius) against the reference's
    rho: identical start vector, same stopping rule; the device dot products
    sum in another order, so the Rayleigh quotients agree to ~1e-15 and the
    stopping iteration may move by one (rho then moves by < tol = 1e-9)."""
    d, _ = gold
    forest, dm, faces, params = _mesh(gold, name)
    op = st.ThermalOperator(forest, dm, params, st.SolverSettings())
    crit = st.compute_step_criteria(op)
    rho = 2.0 / crit.dt_stability
    ref = float(d[name + "/rho"])
    assert abs(rho - ref) <= 2e-9 * ref
    assert abs(op.last_power_iterations - len(d[name + "/lams"])) <= 1
    assert crit.dt_accuracy == float(d[name + "/dt_accuracy"])
    op.close()


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_gpu_step_criteria_structured_match_oracle(p):
    """Structured Q1-Q4 boxes: device rho against the oracle restatement."""
    from cpu_oracle import structured_tables
    h = 1.0 / 6
    nx, ny, nz = 5, 4, 3
    params = st.ProcessParams(
        st.MaterialParams(k_p=6.7, k_m=32.0, k_s=6.7, T_s=300.0, T_l=1928.0, rho=4430.0,
                          c=526.0),
        st.BoundaryParams(emissivity=0.3, T_inf=300.0, T_v=1e9),
        st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0),
        st.MeshParams(h_coarse=h, n_refine=0, h_powder=h))
    box = st.StructuredBox(nx, ny, nz, h, degree=p)
    op = st.ThermalOperator(box, box, params, st.SolverSettings())
    rho = 2.0 / st.compute_step_criteria(op).dt_stability
    ora = OracleOperator(structured_tables(nx, ny, nz, h, p, origin=box.origin), params)
    ref, applies = step_criteria_rho(ora)
    assert abs(rho - ref) <= 2e-9 * ref
    assert abs(op.last_power_iterations - applies) <= 1
    op.close()


@pytest.mark.gpu
def test_gpu_power_iteration_batches_are_exact():
    """Batched device power iteration (history of (w.w, v.w) read per batch,
    graph replay after the first batch): two calls on one context give the
    same rho and iteration count bitwise."""
    from cpu_oracle import structured_tables  # noqa: F401  (oracle on path)
    h = 1.0 / 8
    params = st.ProcessParams(
        st.MaterialParams(k_p=6.7, k_m=32.0, k_s=6.7, T_s=300.0, T_l=1928.0, rho=4430.0,
                          c=526.0),
        st.BoundaryParams(emissivity=0.3, T_inf=300.0, T_v=1e9),
        st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0),
        st.MeshParams(h_coarse=h, n_refine=0, h_powder=h))
    box = st.StructuredBox(8, 6, 5, h, degree=2)
    op = st.ThermalOperator(box, box, params, st.SolverSettings())
    r1 = 2.0 / st.compute_step_criteria(op).dt_stability
    n1 = op.last_power_iterations
    r2 = 2.0 / st.compute_step_criteria(op).dt_stability
    assert r1 == r2 and op.last_power_iterations == n1
    assert n1 > 4  # crosses at least one batch boundary
    op.close()
