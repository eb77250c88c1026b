"""Generate densification fixtures with the REFERENCE implementation.

Run in the build container (``/root/reference`` present):

    python tests/golden/make_densify.py

A seeded 300-Gaussian TrainState gets random Adam moments and densification
statistics chosen so that every branch of ``densify_and_prune``
(optim.py:132-198) fires -- unobserved, below/above the gradient threshold,
small (clone) and large (split) candidates, transparent (pruned) rows -- and
the reference runs it with ``np.random.default_rng(11)``.  Inputs, the
generator seed and every output array go to ``tests/golden/densify.npz``.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
FIELDS = ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits")


def main():
    sys.path.insert(0, REF)
    from uwsplat.fixtures import random_cloud
    from uwsplat.optim import OptimConfig, densify_and_prune
    from uwsplat.scene import MediumParams, TrainState

    rng = np.random.default_rng(3)
    n = 300
    cloud = random_cloud(n, rng)
    # spread the scales over two decades so both the clone and the split gate fire
    base = np.exp(rng.uniform(np.log(0.01), np.log(1.0), size=(n, 1)))
    cloud.log_scales[:] = np.log(base * rng.uniform(0.5, 1.5, size=(n, 3))).astype(np.float32)
    # un-normalized quaternions: quat_to_rotmat normalizes first
    cloud.rotations[:] = (cloud.rotations * rng.uniform(0.5, 2.0, size=(n, 1))).astype(np.float32)
    cloud.opacity_logits[::7] = np.float32(-3.0)        # sigmoid < 0.1 -> pruned
    medium = MediumParams((0.6, 0.45, 0.3), (0.2, 0.35, 0.5), (0.8, 1.0, 1.2))
    state = TrainState(cloud, medium, iteration=1500)
    for name in FIELDS:
        slot = state.adam[name]
        slot.m = rng.normal(size=slot.m.shape).astype(np.float32)
        slot.v = rng.uniform(0, 1, size=slot.v.shape).astype(np.float32)
        slot.step = 1500
    state.obs_count[:] = rng.integers(0, 5, size=n).astype(np.uint32)
    state.grad_accum[:] = (rng.uniform(0, 6e-4, size=n) * state.obs_count).astype(np.float32)
    cfg = OptimConfig()
    extent = 10.0  # percent_dense * extent = 0.1: about half the candidates clone

    rec = {"in_" + f: getattr(cloud, f).copy() for f in FIELDS}
    rec.update({"in_m_" + f: state.adam[f].m.copy() for f in FIELDS})
    rec.update({"in_v_" + f: state.adam[f].v.copy() for f in FIELDS})
    rec["in_grad_accum"] = state.grad_accum.copy()
    rec["in_obs_count"] = state.obs_count.copy()
    rec["extent"] = np.array(extent)
    rec["seed"] = np.array(11)

    counts = densify_and_prune(state, cfg, extent, np.random.default_rng(11))
    rec["counts"] = np.array(counts)
    rec.update({"out_" + f: getattr(cloud, f).copy() for f in FIELDS})
    rec.update({"out_m_" + f: state.adam[f].m.copy() for f in FIELDS})
    rec.update({"out_v_" + f: state.adam[f].v.copy() for f in FIELDS})
    np.savez_compressed(os.path.join(HERE, "densify.npz"), **rec)
    print("densify: (clones, splits, pruned) =", counts, "n ->", len(cloud))


if __name__ == "__main__":
    main()
