"""Depth order with near-equal depths: the 32-bit high-word radix sort plus the
run fix-up must reproduce the reference's (tile, float64 depth, source) order
bit for bit -- short runs (insertion sort), long runs (per-CTA counting sort)
and exactly equal depths (stability)."""

import numpy as np
import pytest

import paper_2411_19588_b200 as uw
from oracle import uwsplat_oracle as O
from gpu_util import np_
from test_gpu_scale import _proj_ns

pytestmark = pytest.mark.gpu


def _cloud(n, z0, dz, seed, spread=1.5):
    rng = np.random.default_rng(seed)
    pos = np.stack([rng.uniform(-spread, spread, n), rng.uniform(-spread, spread, n),
                    z0 + rng.uniform(0.0, dz, n)], axis=1).astype(np.float32)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return uw.GaussianCloud(
        positions=pos, log_scales=np.log(rng.uniform(0.02, 0.08, (n, 3))).astype(np.float32),
        rotations=q.astype(np.float32),
        sh_coeffs=rng.normal(0, 0.5, (n, 1, 3)).astype(np.float32),
        opacity_logits=rng.uniform(-1, 2, n).astype(np.float32))


def _check(cloud, cam):
    p = uw.project_cloud(cloud, cam)
    bins = uw.bin_and_sort(p, cam.width, cam.height)
    offs, ent = O.tile_lists(_proj_ns(p), cam.width, cam.height)
    np.testing.assert_array_equal(np_(bins.offsets).astype(np.int64), offs)
    np.testing.assert_array_equal(np_(bins.entries).astype(np.int64), ent)
    d = np_(p.depth)
    hi = d.view(np.uint64) >> np.uint64(32)
    _, counts = np.unique(hi, return_counts=True)
    return counts.max(), int((counts > 1).sum())


def test_short_runs_match_reference():
    cam = uw.Camera.look_at((0.3, -0.2, -1.0), (0, 0, 10), width=160, height=120, fx=150.0, fy=150.0)
    longest, tied = _check(_cloud(3000, 10.0, 1e-3, seed=7, spread=0.01), cam)
    assert tied > 10                       # high-word ties really occur


def test_long_runs_match_reference():
    # identity rotation: depth = float32 z exactly; z within a few float32 ulps of 10,
    # so thousands of rows share the high word and differ in the low word
    cam = uw.Camera(width=128, height=96, fx=120.0, fy=120.0, cx=64.0, cy=48.0,
                    R=np.eye(3), t=np.zeros(3))
    longest, tied = _check(_cloud(3000, 10.0, 1e-5, seed=11), cam)
    assert longest > 16


def test_exactly_equal_depths_keep_source_order():
    # identity rotation: depth = z exactly; every Gaussian at the same z
    cam = uw.Camera(width=128, height=96, fx=120.0, fy=120.0, cx=64.0, cy=48.0,
                    R=np.eye(3), t=np.zeros(3))
    cloud = _cloud(2000, 6.0, 0.0, seed=3)
    longest, _ = _check(cloud, cam)
    assert longest > 1000


@pytest.mark.parametrize("near,far", [(0.01, 100.0), (1e-3, 1e5), (0.5, 0.75), (2.0, 3.0e8), (1.0, 1.001), (4.0, 4.0005)])
def test_depths_across_the_whole_near_far_range(near, far):
    # the depth keys are the high words relative to the near plane's, sorted over as many
    # 8-bit digits as hi(far) - hi(near) needs (1 to 4): depths log-uniform over (near, far)
    rng = np.random.default_rng(5)
    n = 4000
    z = np.exp(rng.uniform(np.log(near), np.log(far), n))
    xy = rng.uniform(-0.3, 0.3, (n, 2)) * z[:, None]
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    cloud = uw.GaussianCloud(
        positions=np.concatenate([xy, z[:, None]], axis=1).astype(np.float32),
        log_scales=np.repeat(np.log(0.02 * z)[:, None], 3, axis=1).astype(np.float32),
        rotations=q.astype(np.float32), sh_coeffs=rng.normal(0, 0.5, (n, 1, 3)).astype(np.float32),
        opacity_logits=rng.uniform(-1, 2, n).astype(np.float32))
    cam = uw.Camera(width=96, height=80, fx=90.0, fy=90.0, cx=48.0, cy=40.0,
                    R=np.eye(3), t=np.zeros(3), near=near, far=far)
    _check(cloud, cam)


def test_one_huge_bucket_of_equal_depths():
    # > 2048 rows in one depth bucket: the stable 12-pass counting sort of k_bucket_cta
    cam = uw.Camera(width=128, height=96, fx=120.0, fy=120.0, cx=64.0, cy=48.0,
                    R=np.eye(3), t=np.zeros(3))
    longest, _ = _check(_cloud(6000, 6.0, 0.0, seed=4), cam)
    assert longest > 2048


def test_buckets_of_every_size_class():
    # depths quantised to a few float32 values: buckets of 2..8 (thread), 9..32 (warp),
    # 33..2048 (CTA bitonic) rows side by side
    rng = np.random.default_rng(8)
    sizes = [2, 5, 8, 9, 20, 32, 33, 100, 700, 1500]
    z = np.concatenate([np.full(s, 5.0 + 0.25 * k) for k, s in enumerate(sizes)])
    n = z.size
    xy = rng.uniform(-0.3, 0.3, (n, 2)) * z[:, None]
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    perm = rng.permutation(n)
    cloud = uw.GaussianCloud(
        positions=np.concatenate([xy, z[:, None]], axis=1)[perm].astype(np.float32),
        log_scales=np.full((n, 3), np.log(0.02), dtype=np.float32),
        rotations=q.astype(np.float32), sh_coeffs=rng.normal(0, 0.5, (n, 1, 3)).astype(np.float32),
        opacity_logits=rng.uniform(-1, 2, n).astype(np.float32))
    cam = uw.Camera(width=96, height=80, fx=90.0, fy=90.0, cx=48.0, cy=40.0,
                    R=np.eye(3), t=np.zeros(3))
    _check(cloud, cam)
