"""Guidance refresh: the dark-pixel backscatter estimate.

CPU part: the oracle restatement (oracle/uwsplat_oracle.py ``estimate_backscatter``)
is pinned to the reference's own outputs (tests/golden/make_backscatter.py) --
bit-exact dark-pixel set and estimate.

GPU part: ``paper_2411_19588_b200.estimate_backscatter`` (the sm_100a kernels
behind ``uws_estimate_backscatter``) against the golden outputs / the oracle on
the same inputs.  Tolerances: the dark-pixel set (resize, clustering, stable
per-cluster selection) is bit-exact; the fitted (B_inf, B_b) agree to 1e-6 absolute
and the RMS residual to 1e-6 relative + 1e-12 -- the Levenberg-Marquardt sums
are reduced in a different order than numpy's BLAS calls, so the iterates
differ in the last bits and converge to the same minimum within the solver's
1e-10 step tolerance.
"""

import os

import numpy as np
import pytest

from golden_util import BACKSCATTER_CASES, GOLDEN, backscatter_inputs
from oracle import uwsplat_oracle as O

CASES = tuple(BACKSCATTER_CASES)
PARAM_TOL = 1e-6


@pytest.fixture(scope="module")
def golden():
    z = np.load(os.path.join(GOLDEN, "backscatter.npz"))
    return {k: z[k] for k in z.files}


def _oracle_inputs(name):
    img, depth, kw = backscatter_inputs(name)
    if BACKSCATTER_CASES[name][3] == "raw":
        depth = O.logistic(depth)
    return img, depth, kw


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(golden, name):
    img, depth, kw = _oracle_inputs(name)
    est = O.estimate_backscatter(img, depth, **kw)
    np.testing.assert_array_equal(est.dark_z, golden[f"{name}_dark_z"])
    np.testing.assert_array_equal(est.dark_rgb, golden[f"{name}_dark_rgb"])
    np.testing.assert_array_equal(est.water_color_est, golden[f"{name}_water"])
    np.testing.assert_array_equal(est.backscatter_est, golden[f"{name}_bsc"])
    np.testing.assert_array_equal(est.residual, golden[f"{name}_residual"])
    assert est.degenerate == bool(golden[f"{name}_degenerate"])


def test_oracle_known_answers():
    # a noiseless saturating curve is recovered (backscatter.py:178-208)
    z = np.linspace(0.05, 0.9, 24)
    y = 0.3 * (1 - np.exp(-1.7 * z))
    b_inf, b_b, rms, deg = O.bs_fit(z, y)
    assert not deg and abs(b_inf - 0.3) < 1e-6 and abs(b_b - 1.7) < 1e-5 and rms < 1e-8
    # fewer than three points: mean value, upper backscatter bound, flagged
    assert O.bs_fit(np.array([0.1, 0.2]), np.array([0.2, 0.4]))[1:] [0] == 5.0
    assert O.bs_fit(np.array([0.1, 0.2]), np.array([0.2, 0.4]))[3]
    # all-zero values: the lower box corner, not degenerate
    assert O.bs_fit(z, np.zeros_like(z)) == (0.0, 0.0, 0.0, False)
