"""Scattering-medium helpers (reference: medium.py).

Only ``logistic_remap`` is on the hot path; the render kernel fuses it into
its epilogue.  This host/torch version serves utilities and tests.
"""

from __future__ import annotations

import numpy as np
import torch

LOGISTIC_RATE = 0.1


def logistic_remap(depth_raw):
    """z = 2 / (1 + exp(-0.1 d)) - 1 (medium.py:26-29)."""
    if isinstance(depth_raw, torch.Tensor):
        d = depth_raw.double()
        return 2.0 / (1.0 + torch.exp(-LOGISTIC_RATE * d)) - 1.0
    d = np.asarray(depth_raw, dtype=np.float64)
    return 2.0 / (1.0 + np.exp(-LOGISTIC_RATE * d)) - 1.0
