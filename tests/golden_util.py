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
