"""Asynchronous on-device snapshot (the output and
checkpoint phase of the reference's run_build, driver.py:275-337): the
snapshot taken between steps equals the state a separate run reads at that
step, bitwise, while the steps queued after it proceed; a restart from the
snapshot continues bitwise like the uninterrupted run (the reference's
restart test, test_driver.py:144-162)."""

import numpy as np
import pytest
import torch

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.mesh import FittedPart
from paper_2302_05164_b200.physics import flatten_schedule

pytestmark = pytest.mark.gpu
H = 40e-6


def _params():
    mat = st.MaterialParams(k_p=0.3, k_m=30.0, k_s=22.0, T_s=1450.0, T_l=1900.0,
                            latent_heat=2.86e5)
    bnd = st.BoundaryParams(emissivity=0.4, T_inf=300.0, T_v=2900.0, h_conv=10.0)
    las = st.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=150.0)
    return st.ProcessParams(mat, bnd, las)


def _pinned(n):
    return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()


@pytest.mark.parametrize("kind", ["box_history", "fitted_uniform"])
def test_snapshot_is_the_state_at_that_step_and_restarts_bitwise(kind):
    if kind == "box_history":
        mesh = st.StructuredBox(9, 7, 11, H, degree=2)
    else:
        mesh = FittedPart(13, 11, 24, H, [5] * 16 + [13] * 8, degree=2)
    params = _params()
    rng = np.random.default_rng(3)
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 3 * H, 9 * H, 3 * H, 1.0, 150.0)], 0.0)
    dts, beams = flatten_schedule(lp, 2e-8, 12)
    a = st.ThermalOperator(mesh, mesh, params, st.SolverSettings())
    T0 = rng.uniform(300.0, 2600.0, a.nv)
    rc0 = rng.uniform(0.0, 1.0, a.n_cells * a.qpc) if kind == "box_history" else 1.0
    # reference: the state after 6 steps, read synchronously
    b = st.ThermalOperator(mesh, mesh, params, st.SolverSettings())
    b.set_state(T0, rc0)
    b.run_explicit(dts[:6], beams[:6])
    T6, rc6 = b.get_state()
    b.run_explicit(dts[6:], beams[6:])
    T12, rc12 = b.get_state()
    b.close()
    # snapshot after 6 steps while 6 more are queued
    a.set_state(T0, rc0)
    a.run_explicit(dts[:6], beams[:6])
    Ts, rcs = _pinned(a.nv), _pinned(a.n_cells * a.qpc)
    a.snapshot(Ts, rcs)
    a.run_explicit(dts[6:], beams[6:])
    assert a.snapshot_wait()
    assert np.array_equal(Ts, T6)
    assert np.array_equal(rcs, np.broadcast_to(rc6, rcs.shape))
    T12a, _ = a.get_state()
    assert np.array_equal(T12a, T12)
    a.close()
    # restart from the snapshot (a checkpoint) continues bitwise
    c = st.ThermalOperator(mesh, mesh, params, st.SolverSettings())
    c.set_state(Ts.copy(), rcs.copy() if kind == "box_history" else 1.0)
    c.run_explicit(dts[6:], beams[6:])
    T12c, _ = c.get_state()
    c.close()
    assert np.array_equal(T12c, T12)
