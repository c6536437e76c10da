"""Structured (uniform box, degree p) backend vs the CPU oracle.

Degree 1 is the reference algorithm (pinned by the golden vectors);
degrees 2..4, the apparent heat capacity, convection and multiple beams
are the oracle extension (validated against dense assembly in
tests/test_oracle_extension.py).  Box sizes are chosen so that tiles are
partial and x chunks, y and z seams all occur."""

import numpy as np
import pytest

from cpu_oracle import OracleOperator, structured_tables
from fixtures import load, rel

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.physics import BeamState

pytestmark = pytest.mark.gpu

DIMS = {1: (13, 19, 37), 2: (9, 11, 19), 3: (6, 10, 9), 4: (5, 6, 9)}
H = 40e-6


def _params(latent=False, hconv=0.0, evap=True):
    mat = st.MaterialParams(k_p=0.3, k_m=30.0, k_s=22.0, T_s=1450.0, T_l=1900.0,
                            latent_heat=2.86e5 if latent else 0.0, T_lat_s=1878.0,
                            T_lat_l=1928.0)
    bnd = st.BoundaryParams(emissivity=0.4, T_inf=300.0, T_v=2900.0 if evap else 1e9,
                            h_conv=hconv)
    las = st.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=90.0)
    return st.ProcessParams(mat, bnd, las, st.MeshParams(h_coarse=H, n_refine=0, h_powder=H))


def _setup(p, latent=False, hconv=0.0, seed=0):
    nx, ny, nz = DIMS[p]
    params = _params(latent, hconv)
    box = st.StructuredBox(nx, ny, nz, H, degree=p)
    op = st.ThermalOperator(box, box, params, st.SolverSettings())
    orc = OracleOperator(structured_tables(nx, ny, nz, H, p), params)
    rng = np.random.default_rng(seed + p)
    T = rng.uniform(300.0, 3300.0, op.nv)
    T[box.is_dirichlet] = 300.0
    q = p + 1
    rc = rng.uniform(0.0, 1.0, (op.n_cells, q, q, q))
    beams = [BeamState(np.array([nx * H * 0.45, ny * H * 0.55]), 0.0, 90.0, True),
             BeamState(np.array([nx * H * 0.8, ny * H * 0.2]), 0.0, 40.0, True)]
    tb = [(b.position[0], b.position[1], b.z_top, b.power) for b in beams]
    return box, op, orc, T, rc, beams, tb


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_structured_rhs_and_step_match_oracle(p):
    box, op, orc, T, rc, beams, tb = _setup(p)
    tol = 1e-12
    assert rel(op.evaluate_rhs(T, rc, beams), orc.evaluate_rhs(T, rc, tb)) < tol
    assert rel(op.evaluate_rhs(T, rc, None, faces=False, source=False),
               orc.evaluate_rhs(T, rc, [], faces=False, source=False)) < tol
    assert rel(op.evaluate_rhs(T, rc, None, diffusion=False, source=False),
               orc.evaluate_rhs(T, rc, [], diffusion=False, source=False)) < tol
    assert rel(op.evaluate_rhs(T, rc, beams, diffusion=False, faces=False),
               orc.evaluate_rhs(T, rc, tb, diffusion=False, faces=False)) < tol
    assert rel(op.evaluate_rhs(T, None, None, faces=False, source=False, frozen_k=20.0),
               orc.evaluate_rhs(T, None, [], faces=False, source=False, frozen_k=20.0)) < tol
    assert rel(op.lumped_capacity(), orc.lumped_capacity()) < tol
    dt = 2e-7
    assert rel(op.explicit_fused_step(T, dt, rc, beams), orc.explicit_step(T, dt, rc, tb)) < 1e-12
    h = st.HistoryField(rc.copy(), 0)
    op.update_history(h, T)
    assert rel(h.r_c, orc.update_history(rc, T)) < 1e-14


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_structured_implicit_pieces_match_oracle(p):
    box, op, orc, T, rc, beams, tb = _setup(p, seed=5)
    rng = np.random.default_rng(9)
    v = rng.standard_normal(op.nv)
    dt = 1e-4
    assert rel(op.apply_mass(v), orc.apply_mass(v)) < 1e-12
    assert rel(op.apply_jacobian(v, T, rc, dt), orc.apply_jacobian(v, T, rc, dt)) < 1e-12
    assert rel(op.jacobian_diagonal(T, rc, dt), orc.jacobian_diagonal(T, rc, dt)) < 1e-12
    # the implicit pieces are fixed-order gathers: bitwise reproducible
    assert np.array_equal(op.apply_jacobian(v, T, rc, dt), op.apply_jacobian(v, T, rc, dt))
    assert np.array_equal(op.jacobian_diagonal(T, rc, dt), op.jacobian_diagonal(T, rc, dt))


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_structured_latent_heat_and_convection(p):
    box, op, orc, T, rc, beams, tb = _setup(p, latent=True, hconv=10.0, seed=3)
    # put a band of nodes inside the latent interval
    T[::7] = 1900.0
    dt = 2e-7
    got = op.explicit_fused_step(T, dt, rc, beams)
    want = orc.explicit_step(T, dt, rc, tb)
    assert rel(got, want) < 1e-12
    assert rel(op.lumped_capacity(T), orc.lumped_capacity(T)) < 1e-12


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_structured_resident_loop_matches_oracle(p):
    """Multi-step device loop with a per-qp history field and the fused
    (deferred) history update."""
    from cpu_oracle import run_explicit
    box, op, orc, T, rc, beams, tb = _setup(p, seed=11)
    T = 300.0 + np.random.default_rng(2).uniform(0.0, 900.0, op.nv)
    dts = np.full(30, 1e-7)
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, box.ny * H / 2, box.nx * H, box.ny * H / 2,
                                          1.0, 150.0)], 0.0)
    dts, bm = st.flatten_schedule(lp, 1e-7, 30)
    op.set_state(T, rc)
    fail, ext, tmax = op.run_explicit(dts, bm)
    assert fail == 0
    Tg, rcg = op.get_state()
    from cpu_oracle import beam_tuple
    To, rco = run_explicit(orc, T, rc, dts, [[beam_tuple(b) for b in row] for row in bm])
    assert rel(Tg, To) < 1e-12
    assert rel(rcg, rco.reshape(-1)) < 1e-13
    assert tmax == pytest.approx(max(float(To.max()), 0.0), rel=1e-3) or tmax >= To.max() - 1


@pytest.mark.parametrize("kernel", ["march", "slab"])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_structured_both_hot_kernels_match_oracle(p, kernel, monkeypatch):
    """k_xmarch (one thread per cell) and k_xslab (p+1 threads per cell)
    are both kept; ST_KERNEL picks one at context creation."""
    monkeypatch.setenv("ST_KERNEL", kernel)
    box, op, orc, T, rc, beams, tb = _setup(p, latent=True, hconv=10.0, seed=21)
    T[::5] = 1900.0
    dt = 2e-7
    assert rel(op.explicit_fused_step(T, dt, rc, beams), orc.explicit_step(T, dt, rc, tb)) < 1e-12
    assert rel(op.evaluate_rhs(T, rc, beams), orc.evaluate_rhs(T, rc, tb)) < 1e-12


def test_structured_q1_config0_matches_reference():
    g = load("config0")
    h = 31.25e-6
    box = st.StructuredBox(64, 64, 32, h, degree=1)
    mat = st.MaterialParams(k_p=6.7, k_m=6.7, k_s=6.7, rho=4430.0, c=526.0)
    bnd = st.BoundaryParams(emissivity=0.0, T_inf=300.0, T_v=1e9)
    las = st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0, scan_velocity=1.0)
    params = st.ProcessParams(mat, bnd, las, st.MeshParams(h_coarse=h, n_refine=0, h_powder=h))
    op = st.ThermalOperator(box, box, params, st.SolverSettings())
    T0 = 300.0 + np.random.default_rng(0).uniform(0.0, 1.0, box.n_vertices)
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 1e-3, 2e-4, 1e-3, 1.0, 70.0)], 0.0)
    q = np.ones((box.n_cells, 2, 2, 2))
    state = st.SimulationState(box, box, op, T0.copy(), st.HistoryField(q, 0))
    stats = st.run_scan_phase(state, lp, 1e-6)
    assert stats.n_steps == 200
    assert rel(state.T, g["T200"]) <= 1e-9


def test_structured_determinism_run_to_run():
    box, op, orc, T, rc, beams, tb = _setup(2, seed=21)
    a = op.evaluate_rhs(T, rc, beams)
    b = op.evaluate_rhs(T, rc, beams)
    # seam partials are plain stores to per-CTA slots summed by k_seam_list
    # in a fixed order: bitwise reproducible
    assert np.array_equal(a, b)


@pytest.mark.parametrize("kernel", ["march", "slab"])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_structured_uniform_history_loop_matches_oracle(p, kernel, monkeypatch):
    """The config-1 path: consolidated material (r_c = 1 everywhere, never
    stored), latent heat, convection, two beams, resident multi-step loop."""
    from cpu_oracle import beam_tuple, run_explicit
    monkeypatch.setenv("ST_KERNEL", kernel)
    box, op, orc, T, rc, beams, tb = _setup(p, latent=True, hconv=10.0, seed=31)
    T = 300.0 + np.random.default_rng(4).uniform(0.0, 1700.0, op.nv)
    T[box.is_dirichlet] = 300.0
    # two concurrent beams (one LayerPath each)
    lp1 = st.LayerPath(0, 0.0, [st.Segment(0.0, box.ny * H / 2, box.nx * H, box.ny * H / 2,
                                           1.0, 150.0)], 0.0)
    lp2 = st.LayerPath(0, 0.0, [st.Segment(box.nx * H, box.ny * H * 0.3, 0.0, box.ny * H * 0.3,
                                           1.0, 80.0)], 0.0)
    dts, bm = st.flatten_schedule([lp1, lp2], 1e-7, 20)
    assert bm.shape[1] == 2
    op.set_state(T, 1.0)
    fail, ext, tmax = op.run_explicit(dts, bm)
    assert fail == 0
    Tg, rcg = op.get_state()
    ones = np.ones((op.n_cells, p + 1, p + 1, p + 1))
    To, _ = run_explicit(orc, T, ones, dts, [[beam_tuple(b) for b in row] for row in bm])
    assert rel(Tg, To) < 1e-12
    assert np.all(rcg == 1.0)


@pytest.mark.parametrize("kernel", ["march", "slab"])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_structured_instability_is_reported(p, kernel, monkeypatch):
    """run_scan_phase's divergence check on the resident loop: the failing
    step and a non-finite or > 1e7 K extreme (timestepping.py:186-192)."""
    monkeypatch.setenv("ST_KERNEL", kernel)
    box, op, orc, T, rc, beams, tb = _setup(p, seed=41)
    T = 300.0 + np.random.default_rng(5).uniform(0.0, 10.0, op.nv)
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, box.ny * H / 2, box.nx * H, box.ny * H / 2,
                                          1.0, 150.0)], 0.0)
    _, bm = st.flatten_schedule(lp, 1e-7, 40)
    dts = np.full(40, 1e-3)  # far above the stability bound
    op.set_state(T, 1.0)
    fail, ext, tmax = op.run_explicit(dts, bm)
    assert fail >= 1
    assert not (np.isfinite(ext) and ext <= 1e7)


def test_structured_too_many_tabled_beams_fail_loudly():
    box, op, orc, T, rc, beams, tb = _setup(2, seed=1)
    many = [BeamState(np.array([H * (1 + i), H * 3]), 0.0, 10.0, True) for i in range(9)]
    with pytest.raises(Exception):
        op.evaluate_rhs(T, rc, many)


def test_structured_seams_are_deterministic():
    """Seam partials go to per-CTA slots and are summed in a fixed order:
    repeated evaluations are bitwise identical."""
    box, op, orc, T, rc, beams, tb = _setup(2, seed=21)
    a = op.evaluate_rhs(T, rc, beams)
    b = op.evaluate_rhs(T, rc, beams)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("lx", ["1", "2", "3"])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_structured_extreme_x_chunking_matches_oracle(p, lx, monkeypatch):
    """Short x chunks make most node planes x seams (every p-th plane for
    Lx = 1): the seam list, its slot sums and the chunk-boundary facets."""
    monkeypatch.setenv("ST_LX", lx)
    box, op, orc, T, rc, beams, tb = _setup(p, latent=True, hconv=10.0, seed=51)
    T[::6] = 1900.0
    dt = 2e-7
    assert rel(op.explicit_fused_step(T, dt, rc, beams), orc.explicit_step(T, dt, rc, tb)) < 1e-12
    assert rel(op.evaluate_rhs(T, rc, beams), orc.evaluate_rhs(T, rc, tb)) < 1e-12
