"""Run-to-run determinism (reference backward.py:334-341
merges per-tile partials in a fixed tile order).

* the forward (render) is per-pixel and bit-identical from run to run;
* backward_render(deterministic=True) writes every (tile, Gaussian) partial to
  its own slot, sorts the slots by Gaussian and sums them in tile order: the
  gradients are bit-identical from run to run, equal the default (atomic)
  backward to float32 rounding, and meet the golden parity contract.
"""

import numpy as np
import pytest
import torch

import paper_2411_19588_b200 as uw
from golden_util import SCENES, load
from gpu_util import (GRAD_FIELDS, device_scene, grad_tolerance_ok, host_cloud, np_,
                      survey_camera, survey_medium)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    hc = host_cloud(100_000)
    cloud = uw.GaussianCloud(**vars(hc))
    m = survey_medium()
    med = uw.MediumParams(m.attenuation, m.water_color, m.backscatter, m.water_color_guide,
                          m.backscatter_guide)
    cam = survey_camera(800, 600)
    gt = torch.rand(600, 800, 3, generator=torch.Generator().manual_seed(0)).cuda()
    return cloud, cam, med, gt


def _grads(buf):
    return np_(buf.flat).copy()


def test_render_bit_identical_run_to_run(c2):
    cloud, cam, med, _ = c2
    a = uw.render(cloud, cam, med, "underwater")
    b = uw.render(cloud, cam, med, "underwater")
    for f in ("color", "depth", "weight", "final_transmittance", "count", "last", "color_clean"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f


def test_deterministic_backward_bit_identical(c2):
    cloud, cam, med, gt = c2
    out = uw.render(cloud, cam, med, "underwater")
    _, dL = uw.total_loss(out.color, gt, med)
    runs = [_grads(uw.backward_render(out, dL, cloud, med, 0.1, deterministic=True))
            for _ in range(3)]
    assert np.array_equal(runs[0], runs[1]) and np.array_equal(runs[0], runs[2])
    # against the default atomic backward: same values to float32 accumulation order
    ref = _grads(uw.backward_render(out, dL, cloud, med, 0.1))
    n = len(cloud)
    bad, worst = grad_tolerance_ok(runs[0][:14 * n], ref[:14 * n], rel=1e-4, abs_frac=1e-7)
    assert bad == 0, worst
    np.testing.assert_allclose(runs[0][16 * n:16 * n + 9], ref[16 * n:16 * n + 9], rtol=1e-6)


@pytest.mark.parametrize("name", SCENES)
def test_deterministic_backward_golden(name):
    g = load(name)
    cloud, cam, medium = device_scene(g)
    d = g.d
    med = medium if g.mode == "underwater" else None
    out = uw.render(cloud, cam, med, g.mode)
    dL = torch.as_tensor(d["dL_dC"], dtype=torch.float32).cuda()
    buf = uw.backward_render(out, dL, cloud, med, g.lambdas[1], deterministic=True)
    for f in GRAD_FIELDS:
        bad, worst = grad_tolerance_ok(np_(getattr(buf, f)), d["grad_" + f])
        assert bad == 0, f"{f}: {bad} out of tolerance (worst rel {worst:.2e})"
    for f in ("d_attenuation", "d_water_color", "d_backscatter"):
        np.testing.assert_allclose(np_(getattr(buf, f)), d["grad_" + f], rtol=1e-4,
                                   atol=1e-6 * max(1e-12, np.abs(d["grad_" + f]).max()))


def test_deterministic_backward_tile_lists(c2):
    """The CSR tile-list form (composite / render_naive outputs) too."""
    cloud, cam, med, gt = c2
    proj = uw.project_cloud(cloud, cam)
    out = uw.composite(proj, uw.bin_and_sort(proj, cam.width, cam.height), cam, med,
                       "underwater")
    _, dL = uw.total_loss(out.color, gt, med)
    a = _grads(uw.backward_render(out, dL, cloud, med, 0.1, deterministic=True))
    b = _grads(uw.backward_render(out, dL, cloud, med, 0.1, deterministic=True))
    assert np.array_equal(a, b)
