"""GPU diagnostic (debug build, -DUWS_FIX_STATS): the debug build re-walks every pixel
within +-2e-3 of T = 1e-4 and reports the float32-vs-float64 final-T error against the
adaptive band, and the count mismatches the adaptive band would have missed (must be 0)."""
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
    a = (ctypes.c_uint * 5)()
    lib.uws_debug_fix_stats(a)
    f = lambda u: struct.unpack("f", struct.pack("I", u))[0]
    return f(a[0]), f(a[1]), a[2], a[3], a[4]
stats()
cases = [(100_000, (800, 600), None), (100_000, (800, 600), (2.0, 6.0)),
         (1_000_000, (1920, 1080), None), (1_000_000, (1920, 1080), (1.0, 5.0)),
         (1_000_000, (3840, 2160), None), (3_000_000, (1920, 1080), None)]
for n, (w, h), op in cases:
    host = bench.synthetic_cloud(n)
    if op is not None:   # opaque scenes: alphas at the 0.99 clamp, large sum alpha/(1-alpha)
        host["opacity_logits"] = np.random.default_rng(5).uniform(*op, n).astype(np.float32)
    cloud = uw.GaussianCloud(**host)
    med = uw.MediumParams(**bench.MEDIUM)
    for k in range(3):
        eye = bench.view_eye(k * 7)
        cam = uw.Camera.look_at(eye, (0, 0, 12), width=w, height=h, fx=1.2 * w, fy=1.2 * w)
        out = uw.render(cloud, cam, med, "underwater")
        torch.cuda.synchronize()
        b = (ctypes.c_ulonglong * 2)()
        lib.uws_debug_ph2_stats(b)
        print("   phase-2 pixels", b[0], "chunks", b[1])
        print(n, w, h, op, k, "re-walked", int(out.fix_count[2]),
              "maxrel %.3e  max rel/band %.3f  missed-by-adaptive %d  n %d  cnt-mismatch %d" % stats())
