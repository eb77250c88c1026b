"""Generate SPLASH01 checkpoint fixtures with the REFERENCE implementation.

Run in the build container (``/root/reference`` present):

    python tests/golden/make_checkpoint.py

Builds a small seeded TrainState through the reference's own API -- a random
cloud, a guided medium, two real ``apply_gradients`` steps (so Adam moments,
step counters and densification statistics are non-trivial) -- and writes the
bytes of the reference's ``save_checkpoint`` (scene.py:288-317) to
``tests/golden/ckpt_guided.bin``; an unguided variant goes to
``ckpt_plain.bin``.  The tests load them with this package, save them back and
require identical bytes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def build(uw, guided: bool, seed: int):
    from uwsplat.fixtures import random_cloud
    from uwsplat.optim import OptimConfig, apply_gradients
    from uwsplat.backward import GradientBuffer
    from uwsplat.scene import MediumParams, TrainState

    rng = np.random.default_rng(seed)
    cloud = random_cloud(37, rng)
    medium = MediumParams((0.6, 0.45, 0.3), (0.2, 0.35, 0.5), (0.8, 1.0, 1.2),
                          (0.25, 0.3, 0.45) if guided else None,
                          (0.9, 1.0, 1.1) if guided else None)
    state = TrainState(cloud, medium, iteration=17)
    for _ in range(2):
        buf = GradientBuffer(len(cloud))
        buf.d_positions[:] = rng.normal(size=buf.d_positions.shape)
        buf.d_log_scales[:] = rng.normal(size=buf.d_log_scales.shape)
        buf.d_rotations[:] = rng.normal(size=buf.d_rotations.shape)
        buf.d_sh_coeffs[:] = rng.normal(size=buf.d_sh_coeffs.shape)
        buf.d_opacity_logits[:] = rng.normal(size=buf.d_opacity_logits.shape)
        buf.d_attenuation[:] = rng.normal(size=3)
        buf.d_water_color[:] = rng.normal(size=3)
        buf.d_backscatter[:] = rng.normal(size=3)
        apply_gradients(state, buf, OptimConfig())
        state.iteration += 1
    state.grad_accum[:] = rng.uniform(0, 2, size=len(cloud)).astype(np.float32)
    state.obs_count[:] = rng.integers(0, 9, size=len(cloud)).astype(np.uint32)
    return state


def main():
    sys.path.insert(0, REF)
    import uwsplat as uw
    from uwsplat.scene import save_checkpoint
    for name, guided, seed in (("ckpt_guided", True, 5), ("ckpt_plain", False, 6)):
        data = save_checkpoint(build(uw, guided, seed))
        with open(os.path.join(HERE, name + ".bin"), "wb") as f:
            f.write(data)
        print(name, len(data), "bytes")


if __name__ == "__main__":
    main()
