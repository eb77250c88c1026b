"""Spread of the canonical 2000-iteration StepEngine run (test_engine_fit_acceptance)
over initial clouds perturbed at 1e-7 (the reference's envelope recipe,
tests/golden/make_e2e_envelope.py).  usage: python tools/e2e_spread.py [runs]"""
import os, sys
import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import uwsplat  # noqa: E402
import paper_2411_19588_b200 as uw  # noqa: E402
from paper_2411_19588_b200 import dropin  # noqa: E402
from paper_2411_19588_b200.train import fit  # noqa: E402
from golden_util import GOLDEN  # noqa: E402

dropin.install(uwsplat)
R = uwsplat
g = np.load(os.path.join(GOLDEN, "e2e_canonical.npz"))
cams = []
for R_, t_, intr in zip(g["cam_R"], g["cam_t"], g["cam_intr"]):
    w, h, fx, fy, cx, cy, near, far = intr
    cams.append(R.scene.Camera(width=int(w), height=int(h), fx=fx, fy=fy, cx=cx, cy=cy,
                               R=R_, t=t_, near=near, far=far))
images = [np.asarray(a, np.float64) for a in g["images"]]
train_idx, _ = R.pipeline.split_dataset(len(images))
extent = R.pipeline.scene_extent(cams)
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 8
out = []
for i in range(runs):
    rng = np.random.default_rng(0)
    init = R.pipeline.init_cloud([cams[j] for j in train_idx], 1000, rng)
    if i:
        pert = np.random.default_rng(100 + i)
        with torch.no_grad():
            p = init.positions
            p += torch.as_tensor(pert.normal(size=tuple(p.shape)) * 1e-7, dtype=p.dtype,
                                 device=p.device)
    state = uw.TrainState(init, uw.MediumParams(np.full(3, 0.05), np.full(3, 0.3),
                                                np.full(3, 0.05)))
    imgs = [np.asarray(a, np.float32) for a in images]
    fit(state, cams, imgs, train_idx, uw.OptimConfig(iterations=2000), extent, rng)
    psnr = np.mean([uw.psnr(np.clip(np.asarray(uw.render(state.cloud, cams[j], state.medium,
                                                         "underwater").color.cpu()), 0, 1),
                            images[j]) for j in train_idx])
    med = np.asarray(state.medium.flat[:9].double().cpu())
    out.append(psnr)
    print(f"run {i}: psnr {psnr:.2f} n {len(state.cloud)} water {np.round(med[3:6], 3)}",
          flush=True)
print("psnr mean %.2f min %.2f max %.2f" % (np.mean(out), np.min(out), np.max(out)))
print("reference envelope:", np.round(np.append(g["env_psnr"], g["train_psnr"].mean()), 2))
