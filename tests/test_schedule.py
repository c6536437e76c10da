"""The vectorised beam schedule equals the per-step layer_beam_state loop
(physics.py:135-151 semantics: tau = (step - 1) dt, closed segment
windows, first match, beam off after the last segment) bit for bit."""

import numpy as np
import pytest

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.physics import flatten_schedule_loop


def _paths(seed):
    rng = np.random.default_rng(seed)
    segs = []
    for _ in range(int(rng.integers(1, 7))):
        x0, y0, x1, y1 = rng.uniform(0, 2e-3, 4)
        if rng.uniform() < 0.2:
            x1, y1 = x0, y0  # zero-length segment
        segs.append(st.Segment(x0, y0, x1, y1, float(rng.uniform(0.3, 2.0)),
                               float(rng.choice([0.0, 70.0, 200.0]))))
    return st.LayerPath(int(rng.integers(0, 5)), float(rng.uniform(-1e-4, 4e-4)), segs,
                        float(rng.uniform(0, 1e-3)))


@pytest.mark.parametrize("seed", range(12))
def test_vectorised_schedule_equals_loop(seed):
    lp = _paths(seed)
    dt = [1e-6, 7.3e-7, 2.5e-5][seed % 3]
    n = int(lp.scan_duration() / dt) + 3
    for step0 in (1, 5):
        a = st.flatten_schedule(lp, dt, n - step0 + 1, step0=step0)
        b = flatten_schedule_loop(lp, dt, n - step0 + 1, step0=step0)
        assert np.array_equal(a[0], b[0])
        assert a[1].tobytes() == b[1].tobytes()


def test_multi_spot_schedule_equals_loop():
    lps = [_paths(s) for s in (1, 2, 3, 4)]
    d = lps[0].scan_duration()
    for lp in lps[1:]:
        lp.cool_time = max(lp.cool_time, d)  # later spots may outlast the first
    n = int(d / 1e-6)
    a = st.flatten_schedule(lps, 1e-6, n)
    b = flatten_schedule_loop(lps, 1e-6, n)
    assert a[1].tobytes() == b[1].tobytes()
