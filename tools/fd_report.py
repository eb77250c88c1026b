"""GPU diagnostic: the device finite-difference check on the reference's
canonical gradient scene (fixtures.gradient_check_scene via baseline/_ref)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import uwsplat
import uwsplat.cli  # noqa
from paper_2411_19588_b200 import dropin
dropin.install(uwsplat)
cloud, cam, medium, gt = uwsplat.fixtures.gradient_check_scene()
for e in (1e-3, 1e-4, 1e-5):
    rep = uwsplat.backward.finite_diff_check(cloud, cam, medium, gt, eps={k: e for k in
        ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits", "attenuation",
         "water_color", "backscatter")})
    rel = np.array([r.rel_err for r in rep.rows]); fd = np.array([abs(r.fd) for r in rep.rows])
    print(f"eps {e:g}: median {np.median(rel):.2e}  p90 {np.quantile(rel, .9):.2e}  "
          f"p99 {np.quantile(rel, .99):.2e} max {rel.max():.2e}; |fd|>1e-4: {(fd > 1e-4).sum()} "
          f"of which rel>1e-2: {((rel > 1e-2) & (fd > 1e-4)).sum()}")
    print(rep.table())
    worst = sorted(rep.rows, key=lambda r: -r.rel_err)[:5]
    for r in worst:
        print("   ", r)
