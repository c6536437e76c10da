"""Synthetic BASELINE workloads (bench.py and the tests; not part of the
product package).

BASELINE.json defines its scan patterns through the reference's hatch
generator (driver.py:85-111: n = max(1, floor(width / spacing)) tracks per
box, centred, serpentine across tracks and boxes; 0 deg along x, 90 along
y).  ``hatch_segments`` produces the same segments (the same float
operations per coordinate, tests/test_workloads.py pins it against the
reference's output) with the track grid computed per box in one go.
"""

import math

import numpy as np


def hatch_segments(boxes, spacing, v, power, direction_deg=0.0):
    """Serpentine hatch over (x0, y0, x1, y1) boxes -> list of Segment."""
    from paper_2302_05164_b200.physics import Segment
    if direction_deg not in (0, 90):
        raise ValueError("hatch direction must be 0 or 90 degrees")
    across = 1 if direction_deg == 0 else 0  # axis the tracks are stacked along
    out = []
    parity = 0
    for box in boxes:
        lo, hi = (box[1], box[3]) if across else (box[0], box[2])
        a0, a1 = (box[0], box[2]) if across else (box[1], box[3])
        width = hi - lo
        n = max(1, int(math.floor(width / spacing + 1e-9)))
        margin = (width - (n - 1) * spacing) / 2.0
        pos = [lo + (margin + i * spacing) for i in range(n)]
        for i, c in enumerate(pos):
            fwd = (parity + i) % 2 == 0
            s, e = (a0, a1) if fwd else (a1, a0)
            out.append(Segment(s, c, e, c, v, power) if across else Segment(c, s, c, e, v, power))
        parity = (parity + n) % 2
    return out
