"""K7 (loss) vs the float64 oracle over image shapes (GPU).

The C = 3 path is the fused single-pass kernel (column strips x row segments,
maps kept on chip); C = 1, 2, 4 take the two-pass kernels.  Shapes cover the
11x11 minimum, widths/heights around the 32-column strip and the 12-row step,
ragged edges, segment boundaries and 1080p.  Tolerances as test_gpu_scale:
values rtol 2e-5, dL/dC max error <= 1e-3 max|ref| and median relative < 1e-4.
"""

import numpy as np
import pytest
import torch

import paper_2411_19588_b200 as uw
from gpu_util import np_
from oracle import uwsplat_oracle as O

pytestmark = pytest.mark.gpu

SHAPES = [(11, 11), (11, 40), (40, 11), (12, 33), (23, 31), (24, 64), (37, 53), (64, 64),
          (65, 97), (100, 300), (257, 33), (301, 150), (600, 800), (1080, 1920)]


def _check(h, w, c, lam_s=0.3, seed=0):
    rng = np.random.default_rng(seed + 7 * h + w + c)
    img = rng.uniform(0, 1, (h, w, c)).astype(np.float32)
    gt = rng.uniform(0, 1, (h, w, c))
    bd_ref, g_ref = O.total_loss(img.astype(np.float64), gt, None, lam_s, 0.0)
    a = torch.from_numpy(img).cuda()
    bd, g = uw.total_loss(a, gt, None, lam_s, 0.0)
    np.testing.assert_allclose([bd.l1, bd.d_ssim, bd.total],
                               [bd_ref["l1"], bd_ref["d_ssim"], bd_ref["total"]], rtol=2e-5)
    g = np_(g).reshape(g_ref.shape)
    err = np.abs(g - g_ref)
    assert err.max() <= 1e-3 * np.abs(g_ref).max(), (h, w, c, err.max())
    assert np.median(err / np.maximum(np.abs(g_ref), 1e-30)) < 1e-4


@pytest.mark.parametrize("h,w", SHAPES)
def test_loss_rgb_shapes(h, w):
    _check(h, w, 3)


@pytest.mark.parametrize("c", [1, 2, 4])
@pytest.mark.parametrize("h,w", [(11, 11), (37, 53), (257, 33)])
def test_loss_other_channel_counts(h, w, c):
    _check(h, w, c)


def test_loss_ssim_only_and_l1_only():
    _check(97, 131, 3, lam_s=1.0)
    _check(97, 131, 3, lam_s=0.0)


def test_loss_deterministic():
    rng = np.random.default_rng(3)
    a = torch.from_numpy(rng.uniform(0, 1, (1080, 1920, 3)).astype(np.float32)).cuda()
    b = torch.from_numpy(rng.uniform(0, 1, (1080, 1920, 3)).astype(np.float32)).cuda()
    r1, g1 = uw.losses.total_loss_device(a, b, None, 0.3, 0.1)
    r2, g2 = uw.losses.total_loss_device(a, b, None, 0.3, 0.1)
    assert torch.equal(r1, r2) and torch.equal(g1, g2)
