"""Golden fixture for the end-to-end training acceptance: the
reference's own 2000-iteration run on the canonical synthetic fixture.

Run HERE (needs /root/reference, pure Python + numpy/scipy):
    python tests/golden/make_e2e.py [iterations]
Writes tests/golden/e2e_canonical.npz with the canonical dataset the reference
generates (24 views, 64x64: observed images, remapped depths, cameras), its
truth values, and the reference's training trajectory: per-iteration loss
terms, Gaussian count and medium parameters, the final train-view PSNR and the
final medium.  The GPU tests drive the drop-in through the same loop and
compare against these numbers.
"""

import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import uwsplat  # noqa: E402
from uwsplat import dataset as D, pipeline as P  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main(iterations=2000):
    tmp = tempfile.mkdtemp()
    spec = D.canonical_spec()
    D.generate_synthetic(spec, tmp)
    ds = D.load_dataset(tmp)
    truth = D.load_truth(tmp)
    cfg = uwsplat.OptimConfig(iterations=iterations)
    t0 = time.time()
    res = P.train(ds, cfg, seed=0)
    wall = time.time() - t0
    rows = res.log_rows
    cols = [c for c in P.LOG_COLUMNS]
    log = np.array([[float(r[c]) for c in cols] for r in rows], dtype=np.float64)
    train_idx, test_idx = P.split_dataset(len(ds.images))
    ev_train = P.evaluate(res.state, ds, indices=train_idx)
    ev_test = P.evaluate(res.state, ds)
    m = res.state.medium
    out = dict(
        images=np.stack([np.asarray(im, np.float32) for im in ds.images]),
        depths=np.stack([np.asarray(d, np.float32) for d in ds.depths]),
        cam_R=np.stack([c.R for c in ds.cameras]), cam_t=np.stack([c.t for c in ds.cameras]),
        cam_intr=np.array([[c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.near, c.far]
                           for c in ds.cameras], np.float64),
        truth_keys=np.array(sorted(truth)), truth_vals=np.array([truth[k] for k in sorted(truth)]),
        log_cols=np.array(cols), log=log, iterations=np.int64(iterations),
        train_psnr=np.array([v["psnr"] for v in ev_train["per_view"]]),
        test_psnr=np.array([v["psnr"] for v in ev_test["per_view"]]),
        final_medium=np.concatenate([np.asarray(m.attenuation, np.float64),
                                     np.asarray(m.water_color, np.float64),
                                     np.asarray(m.backscatter, np.float64)]),
        final_n=np.int64(len(res.state.cloud)), wall_s=np.float64(wall))
    np.savez_compressed(os.path.join(HERE, "e2e_canonical.npz"), **out)
    print(f"{iterations} iterations in {wall:.1f} s; train PSNR {out['train_psnr'].mean():.2f} dB; "
          f"medium {out['final_medium']}; {out['final_n']} Gaussians")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2000)
