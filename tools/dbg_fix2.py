"""GPU diagnostic (debug build, -DUWS_FIX_STATS): float32-vs-float64 final-T error
on the re-walked pixels, and its ratio to sum alpha/(1-alpha)."""
import sys, os, ctypes, struct
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_19588_b200 import _lib
_lib.load(os.path.join(ROOT, "build/dbg/libuwsplat_b200.so"))
import torch, numpy as np
import bench
import paper_2411_19588_b200 as uw
lib = _lib.load()
def stats():
    a = (ctypes.c_uint * 4)()
    lib.uws_debug_fix_stats(a)
    f = lambda u: struct.unpack("f", struct.pack("I", u))[0]
    return f(a[0]), f(a[1]), a[2], a[3]
stats()
for n, (w, h) in ((100_000, (800, 600)), (1_000_000, (1920, 1080)), (1_000_000, (3840, 2160)), (3_000_000, (1920, 1080))):
    host = bench.synthetic_cloud(n)
    cloud = uw.GaussianCloud(**host)
    med = uw.MediumParams(**bench.MEDIUM)
    for k in range(3):
        eye = bench.view_eye(k * 7)
        cam = uw.Camera.look_at(eye, (0, 0, 12), width=w, height=h, fx=1.2 * w, fy=1.2 * w)
        out = uw.render(cloud, cam, med, "underwater")
        torch.cuda.synchronize()
        print(n, w, h, k, "fixed", int(out.fix_count[2]), "maxrel %.3e  max rel/eb %.3e  cnt-mismatch %d  n %d" % stats())
