"""Fitted part (BASELINE configs[4]'s base + overhang on the structured
backend, mesh.FittedPart) vs the CPU oracle on the same node numbering:
rhs (every term) and explicit steps through the resident path, with x
chunks, y / z tile seams, the re-entrant edge where the overhang leaves
the base, the overhang's adiabatic underside, latent heat, convection and
two beams; degrees 1-4; plus the bitwise determinism of the step."""

import numpy as np
import pytest

from cpu_oracle import OracleOperator, fitted_tables
from fixtures import rel

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.mesh import FittedPart
from paper_2302_05164_b200.physics import BEAM_DTYPE, BeamState, pack_beams

pytestmark = pytest.mark.gpu

H = 40e-6
# (nx, ny, nz, base rows, base extent): the extent changes at a tile-row
# boundary of the degree's kernel (CZ = 32, 16, 8, 8 cell rows)
GEOM = {1: (13, 11, 40, 32, 5), 2: (13, 11, 24, 16, 5), 3: (9, 6, 12, 8, 4), 4: (7, 5, 12, 8, 3)}


def _params(latent=True, hconv=10.0):
    mat = st.MaterialParams(k_p=0.3, k_m=30.0, k_s=22.0, T_s=1450.0, T_l=1900.0,
                            latent_heat=2.86e5 if latent else 0.0, T_lat_s=1878.0,
                            T_lat_l=1928.0)
    bnd = st.BoundaryParams(emissivity=0.4, T_inf=300.0, T_v=2900.0, h_conv=hconv)
    las = st.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=90.0)
    return st.ProcessParams(mat, bnd, las, st.MeshParams(h_coarse=H, n_refine=0, h_powder=H))


def _part(p):
    nx, ny, nz, nb, ext = GEOM[p]
    return FittedPart(nx, ny, nz, H, [ext] * nb + [nx] * (nz - nb), degree=p)


def _beams(part):
    return [BeamState(np.array([part.nx * H * 0.25, part.ny * H * 0.5]), 0.0, 90.0, True),
            BeamState(np.array([part.nx * H * 0.7, part.ny * H * 0.3]), 0.0, 60.0, True)]


@pytest.mark.parametrize("lx", [None, "2"])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_fitted_rhs_and_steps_match_oracle(p, lx, monkeypatch):
    if lx:
        monkeypatch.setenv("ST_LX", lx)
    part = _part(p)
    params = _params()
    op = st.ThermalOperator(part, part, params, st.SolverSettings())
    assert op.nv == part.n_vertices and op.n_cells == part.n_cells
    orc = OracleOperator(fitted_tables(part), params)
    rng = np.random.default_rng(p)
    T = rng.uniform(300.0, 3300.0, op.nv)
    T[part.is_dirichlet] = 300.0
    q = p + 1
    ones = np.ones((part.n_cells, q, q, q))
    beams = _beams(part)
    tb = [(b.position[0], b.position[1], b.z_top, b.power) for b in beams]
    for kw in ({}, {"faces": False, "source": False}, {"diffusion": False, "source": False},
               {"diffusion": False, "faces": False}):
        assert rel(op.evaluate_rhs(T, ones, beams, **kw), orc.evaluate_rhs(T, ones, tb, **kw)) \
            < 1e-12, kw
    # resident multi-step path (the bench's): three steps, beams moving
    dt = 2e-8
    op.set_state(T, 1.0)
    recs = np.zeros((3, 2), dtype=BEAM_DTYPE)
    Tref = T.copy()
    for s in range(3):
        bs = [BeamState(b.position + np.array([s * 3e-6, 0.0]), 0.0, b.power, True)
              for b in beams]
        recs[s] = pack_beams(bs)
        Tref = orc.explicit_step(Tref, dt, ones,
                                 [(b.position[0], b.position[1], 0.0, b.power) for b in bs])
    fail, _, _ = op.run_explicit(np.full(3, dt), recs)
    assert fail == 0
    Tgpu, _ = op.get_state()
    assert rel(Tgpu - T, Tref - T) < 1e-12
    assert rel(op.lumped_capacity(), orc.lumped_capacity()) < 1e-12 if not params.material.latent_heat \
        else True
    op.close()


def test_fitted_constant_capacity_and_determinism():
    part = _part(2)
    params = _params(latent=False, hconv=0.0)
    op = st.ThermalOperator(part, part, params, st.SolverSettings())
    orc = OracleOperator(fitted_tables(part), params)
    assert rel(op.lumped_capacity(), orc.lumped_capacity()) < 1e-13
    # total heat capacity = rho c V of the part
    assert abs(op.lumped_capacity().sum() / (params.material.rho * params.material.c *
                                             part.active_volume_m3()) - 1.0) < 1e-12
    T = np.random.default_rng(0).uniform(300.0, 3000.0, op.nv)
    ones = np.ones(part.n_cells * 27)
    a = op.explicit_fused_step(T, 1e-8, ones, _beams(part))
    b = op.explicit_fused_step(T, 1e-8, ones, _beams(part))
    assert np.array_equal(a, b)
    with pytest.raises(Exception):
        op.apply_mass(T)
    op.close()
