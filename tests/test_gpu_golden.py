"""CUDA path vs golden vectors produced by the reference itself (GPU).

Tolerances (SURVEY §8c parity contract, stated here):
  * integer stages (visible set, tile rectangles, entries, ranges, counts): exact;
  * float64 preprocess quantities: mean2d/depth bit-exact, others rtol 1e-12
    (CUDA vs libm exp/log differ in the last ulp);
  * images: max abs 1e-4; depth rel 1e-5;
  * gradients: |g - g_ref| <= 1e-3 |g_ref| + 1e-6 max|g_ref| per element;
  * Adam: bit-exact given the same float32 gradients.
"""

import numpy as np
import pytest
import torch

import paper_2411_19588_b200 as uw
from golden_util import SCENES, load
from gpu_util import GRAD_FIELDS, device_scene, grad_tolerance_ok, np_
from oracle import uwsplat_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(params=SCENES, scope="module")
def scene(request):
    g = load(request.param)
    g.cloud_d, g.cam_d, g.medium_d = device_scene(g)
    return g


def test_projection(scene):
    d = scene.d
    p = uw.project_cloud(scene.cloud_d, scene.cam_d)
    np.testing.assert_array_equal(np_(p.source_index), d["proj_source_index"])
    np.testing.assert_array_equal(np_(p.mean2d), d["proj_mean2d"])
    np.testing.assert_array_equal(np_(p.depth), d["proj_depth"])
    np.testing.assert_allclose(np_(p.radius), d["proj_radius"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(np_(p.cov2d), d["proj_cov2d"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(np_(p.conic), d["proj_conic"], rtol=1e-11, atol=1e-15)
    np.testing.assert_allclose(np_(p.opacity), d["proj_opacity"], rtol=1e-14, atol=0)
    np.testing.assert_allclose(np_(p.color), d["proj_color"], rtol=0, atol=1e-7)
    # tile rectangles: the oracle's _spans_for applied to the GPU's own mean2d/radius
    gx, gy = scene.cam_d.grid
    ref_rect = O.tile_rect(np_(p.mean2d), np_(p.radius), (gx, gy))
    np.testing.assert_array_equal(np_(p.rect).astype(np.int64), ref_rect)


def test_bins_bit_exact(scene):
    d = scene.d
    p = uw.project_cloud(scene.cloud_d, scene.cam_d)
    bins = uw.bin_and_sort(p, scene.cam_d.width, scene.cam_d.height)
    np.testing.assert_array_equal(np_(bins.offsets).astype(np.int64), d["bins_offsets"])
    np.testing.assert_array_equal(np_(bins.entries), d["bins_entries"])


def test_render(scene):
    d = scene.d
    out = uw.render(scene.cloud_d, scene.cam_d, scene.medium_d, scene.mode, medium_maps=True)
    np.testing.assert_array_equal(np_(out.count), d["out_count"])
    assert np.abs(np_(out.color) - d["out_color"]).max() < 1e-4
    if scene.mode == "underwater":
        assert np.abs(np_(out.color_clean) - d["out_color_clean"]).max() < 1e-4
        # medium images are exact functions of depth and the 9 medium scalars
        z = O.logistic(d["out_depth"])[..., None]
        att = np.exp(-d["medium_attenuation"].astype(np.float64) * z)
        bsc = d["medium_water_color"] * (1 - np.exp(-d["medium_backscatter"].astype(np.float64) * z))
        assert np.abs(np_(out.attenuation_map) - att).max() < 1e-5
        assert np.abs(np_(out.backscatter_map) - bsc).max() < 1e-5
    np.testing.assert_allclose(np_(out.depth), d["out_depth"], rtol=1e-5, atol=0)
    assert np.abs(np_(out.weight) - d["out_weight"]).max() < 1e-4
    tf, tf_ref = np_(out.final_transmittance), d["out_final_transmittance"]
    assert (np.abs(tf - tf_ref) <= 1e-4 * tf_ref + 1e-6).all()


def test_loss(scene):
    d = scene.d
    img = torch.as_tensor(d["out_color"], dtype=torch.float32).cuda()
    bd, grad = uw.total_loss(img, scene.gt, scene.medium_d, *scene.lambdas)
    got = np.array([bd.l1, bd.d_ssim, bd.l_bs, bd.total])
    np.testing.assert_allclose(got, d["loss"], rtol=2e-5, atol=1e-7)
    ref = d["dL_dC"]
    assert np.abs(np_(grad) - ref).max() <= 1e-4 * np.abs(ref).max()


def test_backward(scene):
    d = scene.d
    med = scene.medium_d if scene.mode == "underwater" else None
    out = uw.render(scene.cloud_d, scene.cam_d, med, scene.mode)
    dL = torch.as_tensor(d["dL_dC"], dtype=torch.float32).cuda()
    buf = uw.backward_render(out, dL, scene.cloud_d, med, scene.lambdas[1])
    for f in GRAD_FIELDS:
        bad, worst = grad_tolerance_ok(np_(getattr(buf, f)), d["grad_" + f])
        assert bad == 0, f"{f}: {bad} elements out of tolerance (worst rel {worst:.2e})"
    np.testing.assert_allclose(np_(buf.mean2d_grad_norm), d["grad_mean2d_grad_norm"],
                               rtol=1e-3, atol=1e-6 * d["grad_mean2d_grad_norm"].max())
    np.testing.assert_array_equal(np_(buf.observed), d["grad_observed"])
    for f in ("d_attenuation", "d_water_color", "d_backscatter"):
        np.testing.assert_allclose(np_(getattr(buf, f)), d["grad_" + f], rtol=1e-4,
                                   atol=1e-6 * max(1e-12, np.abs(d["grad_" + f]).max()))


def test_adam_bit_exact(scene):
    """apply_gradients on device == reference adam_step on the same float32 gradients."""
    d = scene.d
    cloud, medium = scene.cloud_d.copy(), (scene.medium_d or uw.MediumParams.zero()).copy()
    rng = np.random.default_rng(1)
    n = len(cloud)
    buf = uw.GradientBuffer(n)
    gflat = rng.normal(scale=1e-3, size=buf.flat.numel()).astype(np.float32)
    buf.flat.copy_(torch.as_tensor(gflat))
    state = uw.TrainState(cloud, medium, iteration=7)
    # two steps so the moments are non-trivial
    cfg = uw.OptimConfig()
    host = {f: d["in_" + f].copy() for f in ("positions", "log_scales", "rotations", "sh_coeffs",
                                             "opacity_logits")}
    mh = {f: np.zeros_like(v) for f, v in host.items()}
    vh = {f: np.zeros_like(v) for f, v in host.items()}
    med_names = ("attenuation", "water_color", "backscatter")
    med_host = {f: np_(getattr(medium, f)).copy() for f in med_names}
    mmh = {f: np.zeros(3, np.float32) for f in med_names}
    mvh = {f: np.zeros(3, np.float32) for f in med_names}
    lrs = {"positions": uw.position_lr(7, cfg), "log_scales": cfg.scaling_lr,
           "rotations": cfg.rotation_lr, "sh_coeffs": cfg.feature_lr,
           "opacity_logits": cfg.opacity_lr}
    for step in (1, 2):
        uw.apply_gradients(state, buf, cfg)
        for f in host:
            g = np_(getattr(buf, "d_" + f))
            host[f], mh[f], vh[f] = O.adam(host[f], g, mh[f], vh[f], step, lrs[f])
        host["rotations"] = O.renormalize(host["rotations"])
        new_med = []
        for j, f in enumerate(med_names):
            g = np_(buf.medium)[3 * j:3 * j + 3]
            q, mmh[f], mvh[f] = O.adam(med_host[f], g, mmh[f], mvh[f], step, 0.0025)
            new_med.append(q)
        for f, q in zip(med_names, O.clamp_medium(*new_med)):
            med_host[f] = q
    for f in host:
        np.testing.assert_array_equal(np_(getattr(cloud, f)), host[f], err_msg=f)
        np.testing.assert_array_equal(np_(state.adam[f].m), mh[f], err_msg=f)
        np.testing.assert_array_equal(np_(state.adam[f].v), vh[f], err_msg=f)
    for f in med_names:
        np.testing.assert_array_equal(np_(getattr(medium, f)), med_host[f], err_msg=f)


@pytest.mark.parametrize("n", [1999, 2000])
def test_adam_bit_exact_odd_and_even_n(n):
    """Both Adam kernels (vector for even n, scalar for odd n) == the reference adam_step."""
    g = load("survey2k")
    arrays = {f: getattr(g.cloud, f)[:n] for f in ("positions", "log_scales", "rotations",
                                                   "sh_coeffs", "opacity_logits")}
    cloud = uw.GaussianCloud(**arrays)
    state = uw.TrainState(cloud, uw.MediumParams.zero(), iteration=3)
    buf = uw.GradientBuffer(n)
    buf.flat.copy_(torch.as_tensor(np.random.default_rng(5).normal(
        scale=1e-3, size=buf.flat.numel()).astype(np.float32)))
    cfg = uw.OptimConfig()
    host = {f: np.asarray(v, np.float32).copy() for f, v in arrays.items()}
    mh = {f: np.zeros_like(v) for f, v in host.items()}
    vh = {f: np.zeros_like(v) for f, v in host.items()}
    lrs = {"positions": uw.position_lr(3, cfg), "log_scales": cfg.scaling_lr,
           "rotations": cfg.rotation_lr, "sh_coeffs": cfg.feature_lr,
           "opacity_logits": cfg.opacity_lr}
    for step in (1, 2):
        uw.apply_gradients(state, buf, cfg)
        for f in host:
            gr = np_(getattr(buf, "d_" + f))
            host[f], mh[f], vh[f] = O.adam(host[f], gr, mh[f], vh[f], step, lrs[f])
        host["rotations"] = O.renormalize(host["rotations"])
    for f in host:
        np.testing.assert_array_equal(np_(getattr(cloud, f)), host[f], err_msg=f)
        np.testing.assert_array_equal(np_(state.adam[f].m), mh[f], err_msg=f)
        np.testing.assert_array_equal(np_(state.adam[f].v), vh[f], err_msg=f)
