"""Generate guidance-refresh fixtures with the REFERENCE implementation.

Run in the build container (``/root/reference`` present):

    python tests/golden/make_backscatter.py

For every case of ``tests/golden_util.BACKSCATTER_CASES`` the inputs are
regenerated from their seed (numpy only, so the GPU box can rebuild them) and
the reference's ``estimate_backscatter`` (backscatter.py:211-270) runs on them;
for kind "raw" the depth goes through the reference's ``logistic_remap`` first,
as ``pipeline.py:205`` does.  The estimate and the intermediate dark-pixel set
(``select_dark_pixels`` on the resized inputs) go to
``tests/golden/backscatter.npz``.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def main():
    sys.path.insert(0, REF)
    from uwsplat import backscatter as bs
    from uwsplat.medium import logistic_remap

    from golden_util import BACKSCATTER_CASES, backscatter_inputs

    out = {}
    for name, (h, w, _seed, kind, _kw) in BACKSCATTER_CASES.items():
        img, depth, kw = backscatter_inputs(name)
        if kind == "raw":
            depth = logistic_remap(depth)
        est = bs.estimate_backscatter(img, depth, **kw)
        out[f"{name}_water"] = est.water_color_est
        out[f"{name}_bsc"] = est.backscatter_est
        out[f"{name}_residual"] = est.residual
        out[f"{name}_degenerate"] = np.array(est.degenerate)
        # the dark set of the resized inputs (the stage the GPU must match bit for bit)
        rh = kw.get("resized_height", bs.RESIZED_HEIGHT_DEFAULT)
        im, dp = np.asarray(img, np.float64), np.asarray(depth, np.float64)
        th = min(rh, h)
        if th != h:
            tw = max(1, round(w * th / h))
            im, dp = bs.resize_bilinear(im, th, tw), bs.resize_nearest(dp, th, tw)
        dark = bs.select_dark_pixels(np.maximum(im, 0), np.maximum(dp, 0),
                                     p_dark=kw.get("p_dark", bs.P_DARK_DEFAULT),
                                     edges_num=kw.get("edges_num", bs.EDGES_NUM_DEFAULT))
        out[f"{name}_dark_z"] = dark.dark_z
        out[f"{name}_dark_rgb"] = dark.colors
        out[f"{name}_resized_sum"] = np.array([im.sum(), dp.sum()])
        print(f"{name}: water {est.water_color_est} bsc {est.backscatter_est} "
              f"res {est.residual} deg {est.degenerate} dark {dark.dark_z.size}")
    np.savez_compressed(os.path.join(HERE, "backscatter.npz"), **out)


if __name__ == "__main__":
    main()
