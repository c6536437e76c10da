"""The oracle extension (degree p = 2..4, apparent heat capacity,
convection, several beams) against the independent dense assembly in
oracle/dense.py.  These parts are not covered by any reference test
(SURVEY §8c); p = 1 ties the dense assembly back to the pinned oracle.
CPU only."""

import numpy as np
import pytest

from cpu_oracle import OracleOperator, structured_tables
from dense import dense_system
from fixtures import rel

from paper_2302_05164_b200 import params as P


def _params(latent, hconv):
    mat = P.MaterialParams(k_p=0.3, k_m=30.0, k_s=22.0, T_s=1450.0, T_l=1900.0,
                           latent_heat=2.86e5 if latent else 0.0)
    bnd = P.BoundaryParams(emissivity=0.4, T_inf=300.0, T_v=2900.0, h_conv=hconv)
    las = P.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=90.0)
    return P.ProcessParams(mat, bnd, las)


@pytest.mark.parametrize("p,dims", [(1, (3, 3, 2)), (2, (2, 3, 2)), (3, (2, 2, 2)),
                                    (4, (2, 1, 2))])
@pytest.mark.parametrize("latent,hconv", [(False, 0.0), (True, 10.0)])
def test_oracle_extension_matches_dense_assembly(p, dims, latent, hconv):
    h = 40e-6
    M = structured_tables(*dims, h, p)
    params = _params(latent, hconv)
    op = OracleOperator(M, params)
    rng = np.random.default_rng(p)
    T = rng.uniform(300.0, 3300.0, M["nv"])
    T[::5] = 1900.0                     # inside the latent band
    q = p + 1
    rc = rng.uniform(0.0, 1.0, (len(M["h"]), q, q, q))
    beams = [(dims[0] * h * 0.4, dims[1] * h * 0.6, 0.0, 90.0),
             (dims[0] * h * 0.9, dims[1] * h * 0.1, 0.0, 40.0)]
    rhs_d, lumped_d = dense_system(M, params, T, rc, beams)
    assert rel(op.evaluate_rhs(T, rc, beams), rhs_d) < 1e-12
    assert rel(op.lumped_capacity(T if latent else None), lumped_d) < 1e-12


def test_multi_beam_is_linear():
    M = structured_tables(4, 4, 2, 40e-6, 2)
    op = OracleOperator(M, _params(False, 0.0))
    T = np.full(M["nv"], 400.0)
    rc = np.ones((len(M["h"]), 3, 3, 3))
    b1, b2 = (5e-5, 6e-5, 0.0, 70.0), (1.2e-4, 1.0e-4, 0.0, 35.0)
    both = op.evaluate_rhs(T, rc, [b1, b2], diffusion=False, faces=False)
    one = op.evaluate_rhs(T, rc, [b1], diffusion=False, faces=False)
    two = op.evaluate_rhs(T, rc, [b2], diffusion=False, faces=False)
    assert rel(both, one + two) < 1e-14
