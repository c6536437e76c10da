"""Device beam schedule (physics.py:135-151): the records
st_beam_schedule evaluates on the device equal the host expansion
(flatten_schedule, itself pinned to the per-step layer_beam_state loop) bit
for bit, for random multi-segment paths and several concurrent paths; a
scan phase driven by the device schedule (st_scan_layer) equals the one
driven by host records (st_explicit_steps) bitwise."""

import numpy as np
import pytest

from test_schedule import _paths

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.physics import flatten_schedule

pytestmark = pytest.mark.gpu
H = 40e-6


@pytest.fixture(scope="module")
def op():
    box = st.StructuredBox(6, 5, 4, H, degree=1)
    o = st.ThermalOperator(box, box, st.ProcessParams(), st.SolverSettings())
    yield o
    o.close()


@pytest.mark.parametrize("seed", range(12))
def test_device_schedule_equals_host(op, seed):
    lps = [_paths(seed), _paths(seed + 100)]
    dt = [1e-6, 7.3e-7, 2.5e-5][seed % 3]
    n = int(min(lp.scan_duration() for lp in lps) / dt) + 1
    for step0 in (1, 5):
        _, want = flatten_schedule(lps, dt, n, step0=step0)
        got = op.beam_schedule(lps, dt, n, step0=step0)
        for f in ("x", "y", "z_top", "power", "active"):
            assert np.array_equal(got[f], want[f]), (f, step0)


def test_scan_layer_equals_host_records():
    box = st.StructuredBox(10, 8, 6, H, degree=2)
    params = st.ProcessParams(st.MaterialParams(k_p=0.2, k_m=30.0, k_s=25.0),
                              st.BoundaryParams(emissivity=0.5, T_v=2800.0),
                              st.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=90.0))
    lps = [st.LayerPath(0, 0.0, [st.Segment(0.0, 2e-4, 4e-4, 2e-4, 1.0, 90.0),
                                 st.Segment(4e-4, 1e-4, 0.0, 1e-4, 1.0, 90.0)], 0.0),
           st.LayerPath(0, 0.0, [st.Segment(1e-4, 0.0, 1e-4, 3e-4, 0.8, 60.0)], 0.0)]
    dt, n = 2e-6, 150
    T0 = np.random.default_rng(4).uniform(300.0, 2500.0, box.n_vertices)
    a = st.ThermalOperator(box, box, params, st.SolverSettings())
    a.set_state(T0, 1.0)
    dts, beams = flatten_schedule(lps, dt, n)
    assert a.run_explicit(dts, beams)[0] == 0
    Ta, _ = a.get_state()
    a.set_state(T0, 1.0)
    assert a.run_scan(lps, dt, n)[0] == 0
    Tb, _ = a.get_state()
    a.close()
    assert np.array_equal(Ta, Tb)
