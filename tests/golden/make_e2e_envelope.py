"""Sensitivity envelope of the reference's 2000-iteration run (adds to
tests/golden/e2e_canonical.npz, written by make_e2e.py).

The canonical training run is chaotic: perturbing the initial positions at
float32-rounding level (relative 1e-7) moves the final train-view PSNR by
several dB and the learned medium by tenths.  This script re-runs the
reference's own pipeline.train with such perturbations (one process per seed)
and stores each run's final PSNR, medium and Gaussian count, the envelope a
float32 device run is judged against.

    python tests/golden/make_e2e_envelope.py 1 2 3 4 5 6   # perturbation seeds
"""

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

CHILD = r'''
import sys, json, tempfile
import numpy as np
sys.path.insert(0, "/root/reference/pkg/src")
import uwsplat
from uwsplat import dataset as D, pipeline as P
seed = int(sys.argv[1])
tmp = tempfile.mkdtemp()
D.generate_synthetic(D.canonical_spec(), tmp)
ds = D.load_dataset(tmp)
orig = P.init_cloud
def init(cams, n, rng):
    c = orig(cams, n, rng)
    g = np.random.default_rng(1000 + seed)
    c.positions *= (1 + 1e-7 * g.standard_normal(c.positions.shape)).astype(np.float32)
    return c
P.init_cloud = init
res = P.train(ds, uwsplat.OptimConfig(iterations=2000), seed=0)
tr, _ = P.split_dataset(len(ds.images))
ev = P.evaluate(res.state, ds, indices=tr)
m = res.state.medium
print(json.dumps({"seed": seed, "psnr": ev["mean_psnr"], "n": len(res.state.cloud),
                  "medium": [float(v) for v in np.concatenate([m.attenuation, m.water_color,
                                                                m.backscatter])]}))
'''


def main(seeds):
    env = dict(os.environ, OMP_NUM_THREADS="2", OPENBLAS_NUM_THREADS="2")
    procs = [subprocess.Popen([sys.executable, "-c", CHILD, str(s)], stdout=subprocess.PIPE,
                              text=True, env=env) for s in seeds]
    runs = [json.loads(p.communicate()[0].strip().splitlines()[-1]) for p in procs]
    path = os.path.join(HERE, "e2e_canonical.npz")
    d = dict(np.load(path))
    d["env_seeds"] = np.array([r["seed"] for r in runs])
    d["env_psnr"] = np.array([r["psnr"] for r in runs])
    d["env_medium"] = np.array([r["medium"] for r in runs])
    d["env_n"] = np.array([r["n"] for r in runs])
    np.savez_compressed(path, **d)
    for r in runs:
        print(r)


if __name__ == "__main__":
    main([int(s) for s in sys.argv[1:]] or [1, 2, 3, 4])
