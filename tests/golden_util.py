"""Load the reference-generated golden fixtures (tests/golden/*.npz)."""

import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCENES = ("gradcheck", "survey2k", "clean500", "opaque3k")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    d = {k: z[k] for k in z.files}
    cloud = SimpleNamespace(**{k[3:]: d["in_" + k[3:]] for k in d if k.startswith("in_")})
    w, h = (int(v) for v in d["cam_wh"])
    fx, fy, cx, cy, near, far = (float(v) for v in d["cam_intr"])
    cam = SimpleNamespace(width=w, height=h, fx=fx, fy=fy, cx=cx, cy=cy, near=near, far=far,
                          R=d["cam_R"], t=d["cam_t"])
    medium = None
    if "medium_attenuation" in d:
        medium = SimpleNamespace(attenuation=d["medium_attenuation"],
                                 water_color=d["medium_water_color"],
                                 backscatter=d["medium_backscatter"],
                                 water_color_guide=d.get("medium_water_color_guide"),
                                 backscatter_guide=d.get("medium_backscatter_guide"))
    return SimpleNamespace(d=d, cloud=cloud, cam=cam, medium=medium, gt=d["gt"],
                           mode=str(d["mode"]), lambdas=tuple(float(x) for x in d["lambdas"]))


# ---------------------------------------------------------------------------
# guidance-refresh (estimate_backscatter) cases: inputs are regenerated from
# the seed here, tests/golden/backscatter.npz holds the reference's outputs
# ---------------------------------------------------------------------------
BACKSCATTER_CASES = {
    # name: (H, W, seed, kind, kwargs)
    "uw_small": (96, 128, 1, "scene", {}),
    "uw_resize": (450, 800, 2, "scene", {}),
    "uw_1080": (1080, 1920, 3, "scene", {}),
    "uw_params": (240, 320, 4, "scene", dict(p_dark=0.05, intervals_num=7, edges_num=5,
                                             resized_height=200)),
    "uw_raw_depth": (300, 400, 5, "raw", {}),
    "flat_depth": (64, 80, 6, "flat", {}),
    "two_depths": (64, 80, 7, "two", {}),
    "black": (64, 80, 8, "black", {}),
    "ragged_tiny": (13, 7, 9, "scene", {}),
}


def backscatter_inputs(name):
    """(image float32 (H,W,3), depth, kwargs).  ``depth`` is the remapped
    float64 depth, except for kind "raw": a raw float32 render depth, which the
    caller remaps with logistic_remap (the training loop's call,
    pipeline.py:205)."""
    h, w, seed, kind, kw = BACKSCATTER_CASES[name]
    rng = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.linspace(0, 1, h), np.linspace(0, 1, w), indexing="ij")
    raw = 2.0 + 25.0 * (0.6 * yy + 0.4 * xx) ** 1.5 + rng.normal(0, 0.3, (h, w))
    raw = np.maximum(raw, 0.0).astype(np.float32)
    z = 2.0 / (1.0 + np.exp(-0.1 * raw.astype(np.float64))) - 1.0
    if kind == "flat":
        z = np.full((h, w), 0.4)
    elif kind == "two":
        z = np.where(xx < 0.5, 0.3, 0.6)
    clean = rng.uniform(0, 1, (h, w, 3)) * (rng.uniform(0, 1, (h, w, 1)) > 0.08)
    att = np.array([0.6, 0.45, 0.3])
    binf = np.array([0.2, 0.35, 0.5])
    bb = np.array([0.8, 1.0, 1.2])
    zz = z[..., None]
    img = clean * np.exp(-att * zz) + binf * (1 - np.exp(-bb * zz))
    img = np.clip(img + rng.normal(0, 0.004, img.shape), 0.0, 1.0).astype(np.float32)
    if kind == "black":
        img[:] = 0.0
    depth = raw if kind == "raw" else z
    return img, depth, dict(kw)
