"""GPU diagnostic (variant built with -DUWS_BWD_STATS): K8's (warp, entry) iterations by
the number of lanes that evaluate a pair, pairs per iteration, band-culled iterations.
usage (on the box): tools/variant.sh bstat raster_bwd -DUWS_BWD_STATS; mv build/variants/bstat.so build/; python tools/dbg_bwd.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_19588_b200 import _lib  # noqa: E402

lib = _lib.load(os.path.join(ROOT, "build/bstat.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2411_19588_b200 as uw  # noqa: E402


def stats():
    a = (ctypes.c_ulonglong * 35)()
    lib.uws_debug_bwd_stats(a)
    return np.array(a[:], dtype=np.float64)


cloud = uw.GaussianCloud(**bench.synthetic_cloud(bench.N_GAUSS))
med = uw.MediumParams(**bench.MEDIUM)
cam = uw.Camera.look_at(bench.view_eye(0), (0, 0, 12), width=bench.W, height=bench.H,
                        fx=1.2 * bench.W, fy=1.2 * bench.W)
gt = torch.from_numpy(bench.gt_image()).cuda()
out = uw.render(cloud, cam, med, "underwater")
_, dl = uw.total_loss(out.color, gt, med)
stats()
uw.backward_render(out, dl, cloud, med, 0.1)
torch.cuda.synchronize()
h = stats()
it = h[:33].sum()
print("iterations (warp, entry) past the band test: %.4g   band-culled: %.4g" % (it, h[34]))
print("pairs: %.4g   pairs per iteration: %.2f   per reduced iteration: %.2f"
      % (h[33], h[33] / it, h[33] / h[1:33].sum()))
print("no lane hit (no reduction): %.1f %%" % (100 * h[0] / it))
cum = np.cumsum(h[1:33]) / h[1:33].sum()
for k in (1, 2, 4, 8, 16, 24, 32):
    print("  <= %2d lanes: %.1f %% of reduced iterations" % (k, 100 * cum[k - 1]))
