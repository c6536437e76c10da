"""Consolidation history container (reference ``material.py:97-109``).

The pointwise material law itself (liquid fraction, phase fractions,
conductivity and its derivative, ``material.py:32-94``) runs on the
device inside the operator kernels (csrc/st_common.cuh).
"""

from dataclasses import dataclass

import numpy as np


@dataclass
class HistoryField:
    """Per-cell, per-quadrature-point consolidation state r_c."""

    r_c: np.ndarray
    epoch: int

    def copy(self):
        return HistoryField(self.r_c.copy(), self.epoch)
