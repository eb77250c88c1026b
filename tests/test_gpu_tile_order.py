"""Compositing schedule (uws_tile_order): the engine's forward and backward run the
tiles heaviest first; a permutation of independent tiles, so images, counts and
(deterministic) gradients are bitwise those of raster order (GPU)."""

import ctypes

import numpy as np
import pytest
import torch

import paper_2411_19588_b200 as uw
from paper_2411_19588_b200 import _lib, backward
from gpu_util import GRAD_FIELDS, host_cloud, np_, survey_camera, survey_medium

pytestmark = pytest.mark.gpu

ROWS_COMPLETE = 1 << 30


def _scene(n, W, H, seed=3):
    hc = host_cloud(n, seed=seed)
    med = survey_medium()
    cloud = uw.GaussianCloud(**vars(hc))
    m = uw.MediumParams(med.attenuation, med.water_color, med.backscatter,
                        med.water_color_guide, med.backscatter_guide)
    return cloud, m, survey_camera(W, H)


@pytest.mark.parametrize("n_tiles", [1, 7, 8160, 16384, 16385, 32400])
def test_order_is_a_cost_sorted_permutation(n_tiles):
    """Every tile exactly once, costs (low 30 bits / 8, capped at 127) non-increasing;
    sizes around the kernel's 16384-tile chunk and 4K (32400 tiles)."""
    g = torch.Generator().manual_seed(n_tiles)
    cost = torch.randint(0, 1400, (n_tiles,), generator=g, dtype=torch.int32)
    flag = torch.randint(0, 2, (n_tiles,), generator=g, dtype=torch.int32) * ROWS_COMPLETE
    nrows = (cost | flag).cuda()
    order = torch.full((n_tiles,), -1, dtype=torch.int32, device="cuda")
    _lib.call("uws_tile_order", _lib.ptr(nrows), n_tiles, _lib.ptr(order), _lib.stream_handle())
    o = order.cpu().numpy()
    assert np.array_equal(np.sort(o), np.arange(n_tiles))
    c = np.minimum(cost.numpy()[o], 1023) >> 3
    assert (np.diff(c) <= 0).all()


def test_ordered_forward_equals_raster_order():
    """The engine's second render runs the schedule its first render produced: every
    output bitwise the API render's (raster order)."""
    cloud, m, cam = _scene(200_000, 1280, 720)
    eng = uw.StepEngine(uw.TrainState(cloud, m), cam.width, cam.height, uw.OptimConfig())
    assert eng.TILE_ORDER
    eng.render(cam)
    order = eng.out.tile_order.cpu().numpy()
    assert not np.array_equal(order, np.arange(order.size))   # a real permutation
    out = eng.render(cam)
    api = uw.render(cloud, cam, m, "underwater")
    for f in ("color", "depth", "weight", "count", "final_transmittance", "last"):
        assert torch.equal(getattr(out, f), getattr(api, f)), f


def test_ordered_backward_equals_raster_order():
    """Deterministic backward through the engine's scheduled output vs the same output
    with the schedule removed: every gradient bitwise equal."""
    cloud, m, cam = _scene(200_000, 1280, 720, seed=5)
    eng = uw.StepEngine(uw.TrainState(cloud, m), cam.width, cam.height, uw.OptimConfig())
    eng.render(cam)
    out = eng.render(cam)          # scheduled forward; out.tile_order set
    rng = np.random.default_rng(1)
    dL = torch.as_tensor(rng.normal(size=(cam.height, cam.width, 3)) * 1e-3,
                         dtype=torch.float32).cuda()
    backward.set_deterministic(True)
    try:
        a = uw.backward_render(out, dL, cloud, m, 0.1)
        order, out.tile_order = out.tile_order, None
        b = uw.backward_render(out, dL, cloud, m, 0.1)
        out.tile_order = order
    finally:
        backward.set_deterministic(False)
    for f in GRAD_FIELDS + ("mean2d_grad_norm",):
        assert np.array_equal(np_(getattr(a, f)), np_(getattr(b, f))), f
    assert np.array_equal(np_(a.medium), np_(b.medium))
