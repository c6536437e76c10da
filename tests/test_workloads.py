"""The bench / test hatch generator reproduces the reference's hatch
segments bit for bit (golden: the reference generate_hatch output stored
in tests/golden/pointwise.npz).  CPU only."""

import numpy as np

from fixtures import load

from workloads import hatch_segments


def _arr(segs):
    return np.array([[s.x0, s.y0, s.x1, s.y1, s.v, s.power] for s in segs])


def test_hatch_matches_reference_golden():
    d = load("pointwise")
    got = _arr(hatch_segments([(0.0, 0.0, 4e-4, 3e-4)], 1e-4, 1.0, 70.0))
    assert np.array_equal(got, d["hatch"])


def test_hatch_properties():
    # 90 deg: tracks stacked along x, sense alternating across boxes too
    segs = hatch_segments([(0.0, 0.0, 2e-3, 2e-3), (3e-3, 0.0, 3.25e-3, 1e-3)], 1e-4, 1.0, 70.0, 90)
    a = _arr(segs)
    assert len(segs) == 20 + 2
    assert np.all(a[:, 0] == a[:, 2])
    assert np.all(np.diff(np.sign(a[:, 3] - a[:, 1])) != 0)  # serpentine throughout
    assert np.allclose(np.diff(a[:20, 0]), 1e-4)
