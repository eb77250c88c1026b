"""GPU diagnostic: pixels re-walked by the float64 transmittance fix-up at C3."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import bench
import paper_2411_19588_b200 as uw
host = bench.synthetic_cloud(bench.N_GAUSS)
cloud = uw.GaussianCloud(**host)
med = uw.MediumParams(**bench.MEDIUM)
for (w, h) in ((1920, 1080), (3840, 2160)):
    cam = uw.Camera.look_at(bench.view_eye(0), (0, 0, 12), width=w, height=h, fx=1.2 * w, fy=1.2 * w)
    out = uw.render(cloud, cam, med, "underwater")
    torch.cuda.synchronize()
    n = int(out.fix_count[2])
    T = out.final_transmittance
    band = ((T >= 1e-4 * (1 - 2e-3)) & (T <= 1e-4 * (1 + 2e-3))).sum().item()
    term = (T < 1e-4).float().mean().item()
    print(f"{w}x{h}: fixed {n} px ({n / (w * h):.4%}); final T in band {band}; terminated {term:.3f}")
