"""Parity at BASELINE.json's sizes.

* config 1 at full size (128 x 128 x 32 Q2, 4,293,185 DoFs; k(T), latent
  heat, radiation + convection, the moving 70 W hatch beam): three device
  steps through the resident multi-step path against three steps of the
  CPU oracle, from a state with a melt pool so every material branch is
  hit -- max |dT| / max |T| <= 1e-9;
* config 2 at p = 1 on a 128^3 replica against the REFERENCE's own output
  (tests/golden/make_config2_replica.py: 20,000 seeded samples and three
  checksums of the rhs and of one explicit step);
* config 2 at p = 2, 3, 4 on 48^3-cell unit cubes against the oracle
  extension: rhs and one explicit step, consolidated material (the bench
  path) and a random history (the per-qp history path).
"""

import numpy as np
import pytest

from cpu_oracle import OracleOperator, structured_tables
from fixtures import load, rel

import paper_2302_05164_b200 as st
import workloads as w

pytestmark = pytest.mark.gpu


def _melt_pool_state(box, T0, x0, y0):
    xs = [box.node_coords_1d(a) for a in range(3)]
    X, Y, Z = np.meshgrid(*xs, indexing="ij")
    r2 = (X - x0) ** 2 + (Y - y0) ** 2 + (Z / 0.5) ** 2
    T = T0 + 2800.0 * np.exp(-r2 / (120e-6) ** 2).reshape(-1)
    T[box.is_dirichlet] = 300.0
    return T


@pytest.mark.timeout(900)
def test_config1_full_size_three_steps_vs_oracle():
    wl = w.workload_config1()
    box = w.build_problem(wl)
    params = wl["params"]
    op = st.ThermalOperator(box, box, params, st.SolverSettings())
    dts, beams = w.schedule(wl, 3)
    b0 = beams[0][0]
    T0 = _melt_pool_state(box, wl["T0"](op.nv), float(b0["x"]), float(b0["y"]))
    op.set_state(T0, 1.0)
    fail, _, _ = op.run_explicit(dts, beams)
    assert fail == 0
    T_gpu, _ = op.get_state()
    op.close()
    q = box.degree + 1
    orc = OracleOperator(structured_tables(*wl["dims"], wl["h"], box.degree), params)
    rc = np.ones((box.n_cells, q, q, q))
    T = T0.copy()
    for i in range(3):
        tb = [(float(b["x"]), float(b["y"]), float(b["z_top"]), float(b["power"]))
              for b in beams[i] if b["active"]]
        T = orc.explicit_step(T, float(dts[i]), rc, tb)
    assert T.max() > 1928.0 and np.any((T > 1878.0) & (T < 1928.0))  # melt + latent band
    assert rel(T_gpu, T) <= 1e-9
    # the increment itself, not only the state
    assert rel(T_gpu - T0, T - T0) <= 1e-9


@pytest.mark.timeout(600)
def test_config2_q1_replica_vs_reference():
    g = load("config2_replica_q1")
    n = int(g["n"])
    h = 1.0 / n
    mat = st.MaterialParams(k_p=6.7, k_m=32.0, k_s=6.7, rho=4430.0, c=526.0, T_s=300.0,
                            T_l=1928.0)
    bnd = st.BoundaryParams(emissivity=0.3, T_inf=300.0, T_v=1e9)
    las = st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0)
    params = st.ProcessParams(mat, bnd, las, st.MeshParams(h_coarse=h, n_refine=0, h_powder=h))
    box = st.StructuredBox(n, n, n, h, degree=1)
    op = st.ThermalOperator(box, box, params, st.SolverSettings())
    assert op.nv == int(g["nv"])
    T = np.random.default_rng(2).uniform(300.0, 2500.0, op.nv)
    u = np.random.default_rng(5).standard_normal(op.nv)
    idx = g["idx"]
    f = op.evaluate_rhs(T, np.ones(op.n_cells * 8), None)
    dT = op.explicit_fused_step(T, 1e-3, np.ones(op.n_cells * 8), None) - T
    op.close()
    for v, samples, checks, amax in ((f, g["f_samples"], g["f_checks"], g["f_absmax"]),
                                     (dT, g["dT_samples"], g["dT_checks"], g["dT_absmax"])):
        assert float(np.max(np.abs(v[idx] - samples))) <= 1e-12 * float(amax)
        assert abs(float(np.abs(v).max()) / float(amax) - 1.0) <= 1e-12
        got = np.array([v.sum(), np.abs(v).sum(), v @ u])
        scale = np.abs(v).sum()
        assert np.all(np.abs(got - checks) <= 1e-11 * scale), (got, checks)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("p", [2, 3, 4])
def test_config2_48cube_vs_oracle(p):
    n = 48
    h = 1.0 / n
    params = w._config1_params()
    box = st.StructuredBox(n, n, n, h, degree=p)
    op = st.ThermalOperator(box, box, params, st.SolverSettings())
    rng = np.random.default_rng(2)
    T = rng.uniform(300.0, 2500.0, op.nv)
    q = p + 1
    orc = OracleOperator(structured_tables(n, n, n, h, p), params)
    ones = np.ones((op.n_cells, q, q, q))
    dt = 1e-3
    # consolidated material through the resident path (the bench's kernel)
    op.set_state(T, 1.0)
    fail, _, _ = op.run_explicit(np.array([dt]), np.zeros((1, 0), dtype=st.physics.BEAM_DTYPE))
    assert fail == 0
    T1, _ = op.get_state()
    ref = orc.explicit_step(T, dt, ones, [])
    assert rel(T1 - T, ref - T) <= 1e-9
    assert rel(op.evaluate_rhs(T, ones, None), orc.evaluate_rhs(T, ones, [])) <= 1e-12
    # a random history (per-qp r_c kernel)
    rc = rng.uniform(0.0, 1.0, (op.n_cells, q, q, q))
    assert rel(op.evaluate_rhs(T, rc, None), orc.evaluate_rhs(T, rc, [])) <= 1e-12
    op.close()


@pytest.mark.timeout(900)
def test_config4_replica_vs_oracle():
    """configs[4] at 1/64 of the volume (h = 100 um: 750 x 50 x 120 lattice,
    15.2M DoFs, the same 20 mm base + 2.4 mm overhang and four spots): two
    resident steps vs the oracle on the same numbering, from a state with
    four melt pools."""
    from cpu_oracle import fitted_tables
    wl = w.workload_config4(scale=4)
    part = w.build_part(wl)
    params = wl["params"]
    op = st.ThermalOperator(part, part, params, st.SolverSettings())
    dts, beams = w.schedule(wl, 2)
    lat = part.node_lattice()
    xyz = np.stack([part.node_coords_1d(a)[lat[:, a]] for a in range(3)], axis=1)
    T0 = wl["T0"](op.nv)
    for b in beams[0]:
        r2 = (xyz[:, 0] - b["x"]) ** 2 + (xyz[:, 1] - b["y"]) ** 2 + (xyz[:, 2] / 0.5) ** 2
        T0 = T0 + 2800.0 * np.exp(-r2 / (300e-6) ** 2)
    T0[part.is_dirichlet] = 300.0
    op.set_state(T0, 1.0)
    fail, _, _ = op.run_explicit(dts, beams)
    assert fail == 0
    T_gpu, _ = op.get_state()
    op.close()
    orc = OracleOperator(fitted_tables(part), params)
    ones = np.ones((part.n_cells, 3, 3, 3))
    T = T0.copy()
    for i in range(2):
        tb = [(float(b["x"]), float(b["y"]), float(b["z_top"]), float(b["power"]))
              for b in beams[i] if b["active"]]
        T = orc.explicit_step(T, float(dts[i]), ones, tb)
    assert T.max() > 1928.0
    assert rel(T_gpu, T) <= 1e-9
    assert rel(T_gpu - T0, T - T0) <= 1e-9
