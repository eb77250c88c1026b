"""Parity of the TIMED path at the sizes it is timed on (GPU).

* C1 (10k Gaussians, 256x256): full-frame forward (clean + underwater), loss
  and backward against the float64 oracle -- every pixel, every gradient.
* C3 (1M, 1920x1080, the headline config): backward on seeded tiles (dL/dC
  zero elsewhere, so the other tiles contribute exactly nothing), with the
  oracle's OWN projection and tile lists; forward on seeded tiles.
* C5 (1M and 5M @ 3840x2160): forward on seeded tiles against the oracle's own
  binning of those tiles (5M through the two-set frame stream).
* C4's per-view size (3M @ 1080p): every parameter gradient on seeded tiles.
* StepEngine (the benchmarked path): one step with the gradients kept --
  its render, dL/dC and summed gradient buffer against the oracle, then its
  Adam update bit-exact against the reference's adam_step applied to the
  engine's own float32 gradients.  No fraction-of-elements criteria.

Tolerances: integer outputs (count) exact; images max abs 1e-4;
depth rel 1e-5; gradients |g - g_ref| <= 1e-3 |g_ref| + 1e-6 max|g_ref| per
element; medium gradients rtol 1e-4; Adam bit-exact.
"""

import numpy as np
import pytest
import torch

import paper_2411_19588_b200 as uw
from golden_util import load
from gpu_util import (GRAD_FIELDS, adam_replay, device_scene, grad_tolerance_ok, host_cloud,
                      host_grads, host_state, np_, survey_camera, survey_medium)
from oracle import uwsplat_oracle as O

pytestmark = pytest.mark.gpu


def _device(hc, med):
    cloud = uw.GaussianCloud(**vars(hc))
    m = None if med is None else uw.MediumParams(med.attenuation, med.water_color, med.backscatter,
                                                 med.water_color_guide, med.backscatter_guide)
    return cloud, m


def _tile_mask(cam, tiles):
    gx, _ = O.grid_dims(cam.width, cam.height)
    mask = np.zeros((cam.height, cam.width), bool)
    for t in tiles:
        ty, tx = divmod(int(t), gx)
        mask[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    return mask


def _sample_tiles(cam, n, seed):
    gx, gy = O.grid_dims(cam.width, cam.height)
    return np.sort(np.random.default_rng(seed).choice(gx * gy, n, replace=False))


def _check_images(out, ref, mask=None, medium=True):
    sel = (slice(None),) if mask is None else (mask,)
    np.testing.assert_array_equal(np_(out.count)[sel], ref.count[sel])
    assert np.abs(np_(out.color)[sel] - ref.color[sel]).max() < 1e-4
    if medium:
        assert np.abs(np_(out.color_clean)[sel] - ref.color_clean[sel]).max() < 1e-4
    np.testing.assert_allclose(np_(out.depth)[sel], ref.depth[sel], rtol=1e-5, atol=0)
    assert np.abs(np_(out.weight)[sel] - ref.weight[sel]).max() < 1e-4
    tf, tf_ref = np_(out.final_transmittance)[sel], ref.final_transmittance[sel]
    assert (np.abs(tf - tf_ref) <= 1e-4 * tf_ref + 1e-6).all()


def _check_grads(buf, g, screen_only=False):
    for f in GRAD_FIELDS:
        bad, worst = grad_tolerance_ok(np_(getattr(buf, f)), g[f])
        assert bad == 0, f"{f}: {bad} out of tolerance (worst rel {worst:.2e})"
    np.testing.assert_array_equal(np_(buf.observed), g["observed"])
    bad, worst = grad_tolerance_ok(np_(buf.mean2d_grad_norm), g["mean2d_grad_norm"])
    assert bad == 0, f"mean2d_grad_norm: {bad} out of tolerance (worst rel {worst:.2e})"
    for f in ("d_attenuation", "d_water_color", "d_backscatter"):
        np.testing.assert_allclose(np_(getattr(buf, f)), g[f], rtol=1e-4,
                                   atol=1e-6 * max(np.abs(g[f]).max(), 1e-30))


# ----------------------------------------------------------------------------
# C1: 10k Gaussians, 256x256, full frame
# ----------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c1():
    hc = host_cloud(10_000, seed=0)
    cam = survey_camera(256, 256)
    med = survey_medium()
    cloud, m = _device(hc, med)
    ref_proj = O.project(hc, cam)
    return hc, cam, med, cloud, m, ref_proj


@pytest.mark.parametrize("mode", ["clean", "underwater"])
def test_c1_full_frame_forward(c1, mode):
    hc, cam, med, cloud, m, ref_proj = c1
    out = uw.render(cloud, cam, m if mode == "underwater" else None, mode)
    ref = O.render(hc, cam, med if mode == "underwater" else None, mode, proj=ref_proj)
    _check_images(out, ref, medium=mode == "underwater")


def test_c1_full_frame_loss_and_backward(c1):
    hc, cam, med, cloud, m, ref_proj = c1
    out = uw.render(cloud, cam, m, "underwater")
    ref = O.render(hc, cam, med, "underwater", proj=ref_proj)
    gt = np.random.default_rng(1).uniform(0, 1, (cam.height, cam.width, 3))
    bd, dL = uw.total_loss(out.color, gt, m, 0.3, 0.1)
    bd_ref, dL_ref = O.total_loss(np_(out.color).astype(np.float64), gt, med, 0.3, 0.1)
    np.testing.assert_allclose([bd.l1, bd.d_ssim, bd.l_bs, bd.total],
                               [bd_ref["l1"], bd_ref["d_ssim"], bd_ref["l_bs"], bd_ref["total"]],
                               rtol=2e-5)
    assert np.abs(np_(dL) - dL_ref).max() <= 1e-4 * np.abs(dL_ref).max()
    # the backward from the same dL/dC on both sides
    buf = uw.backward_render(out, dL, cloud, m, 0.1)
    g = O.backward(ref, np_(dL).astype(np.float64), len(hc.positions), med, 0.1)
    _check_grads(buf, g)


# ----------------------------------------------------------------------------
# C3: 1M Gaussians, 1920x1080 (the headline config)
# ----------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c3():
    hc = host_cloud(1_000_000, seed=0)
    cam = survey_camera(1920, 1080)
    med = survey_medium()
    cloud, m = _device(hc, med)
    out = uw.render(cloud, cam, m, "underwater")
    ref_proj = O.project(hc, cam)
    return hc, cam, med, cloud, m, out, ref_proj


def test_c3_forward_sampled_tiles_count_exact(c3):
    hc, cam, med, cloud, m, out, ref_proj = c3
    tiles = _sample_tiles(cam, 32, seed=21)
    ref = O.render(hc, cam, med, "underwater", tiles=tiles, proj=ref_proj)   # oracle's own bins
    _check_images(out, ref, _tile_mask(cam, tiles))


def test_c3_backward_sampled_tiles(c3):
    """The dominant timed kernel at the config it is timed on: dL/dC restricted to
    24 seeded tiles, compared for EVERY parameter gradient of all 1M Gaussians."""
    hc, cam, med, cloud, m, out, ref_proj = c3
    tiles = _sample_tiles(cam, 24, seed=5)
    mask = _tile_mask(cam, tiles)
    rng = np.random.default_rng(9)
    dL = np.where(mask[..., None], rng.normal(size=(cam.height, cam.width, 3)), 0.0) / mask.sum()
    buf = uw.backward_render(out, torch.as_tensor(dL, dtype=torch.float32).cuda(), cloud, m, 0.1)
    ref = O.render(hc, cam, med, "underwater", tiles=tiles, proj=ref_proj)
    g = O.backward(ref, dL.astype(np.float32).astype(np.float64), len(hc.positions), med, 0.1,
                   tiles=tiles)
    _check_grads(buf, g)


def test_c3_engine_matches_api_full_frame(c3):
    """The benchmarked engine step at C3 (full frame) == the API path's render,
    loss and summed gradients (same kernels, different launch plumbing; only the
    order of the float atomics differs)."""
    hc, cam, med, cloud, m, out, ref_proj = c3
    gt = torch.rand(cam.height, cam.width, 3, device="cuda", generator=torch.Generator(
        device="cuda").manual_seed(0))
    state = uw.TrainState(cloud.copy(), m.copy(), iteration=1)
    eng = uw.StepEngine(state, cam.width, cam.height, uw.OptimConfig())
    eng.keep_gradients = True
    st = eng.step([(cam, gt)])
    assert not st.skipped
    o = eng.last_render()
    for f in ("color", "depth", "count", "last"):
        assert torch.equal(getattr(o, f), getattr(out, f)), f
    bd, dL = uw.total_loss(out.color, gt, m, 0.3, 0.1)
    np.testing.assert_allclose(st.total, bd.total, rtol=1e-6)
    assert torch.equal(eng.dL, dL)
    buf = uw.backward_render(out, dL, cloud, m, 0.1)
    for f in GRAD_FIELDS + ("mean2d_grad_norm",):
        a, b = np_(getattr(eng.grads, f)), np_(getattr(buf, f))
        bad, worst = grad_tolerance_ok(a, b, rel=1e-4, abs_frac=1e-6)
        assert bad == 0, f"{f}: {bad} out of tolerance (worst rel {worst:.2e})"
    assert torch.equal(eng.grads.observed, buf.observed)
    np.testing.assert_allclose(np_(eng.grads.medium), np_(buf.medium), rtol=1e-5)


# ----------------------------------------------------------------------------
# C5: 1M Gaussians @ 3840x2160 (render FPS config)
# ----------------------------------------------------------------------------
def test_c5_1m_4k_forward_sampled_tiles():
    hc = host_cloud(1_000_000, seed=0)
    cam = survey_camera(3840, 2160)
    med = survey_medium()
    cloud, m = _device(hc, med)
    eng = uw.StepEngine(uw.TrainState(cloud, m), cam.width, cam.height, uw.OptimConfig())
    out = eng.render(cam)       # the render-FPS path of bench.py
    tiles = _sample_tiles(cam, 16, seed=13)
    ref = O.render(hc, cam, med, "underwater", tiles=tiles)   # oracle projection + binning
    _check_images(out, ref, _tile_mask(cam, tiles))
    api = uw.render(cloud, cam, m, "underwater")
    for f in ("color", "depth", "count", "final_transmittance"):
        assert torch.equal(getattr(api, f), getattr(out, f)), f


def test_c5_5m_4k_frame_stream_sampled_tiles():
    """5M Gaussians @ 3840x2160 (the largest C5 point) through the two-set frame
    stream (the last frame lands in the side set): seeded tiles against the oracle,
    and the whole frame equal to the API render."""
    hc = host_cloud(5_000_000, seed=4)
    cam = survey_camera(3840, 2160)
    med = survey_medium()
    cloud, m = _device(hc, med)
    eng = uw.StepEngine(uw.TrainState(cloud, m), cam.width, cam.height, uw.OptimConfig())
    for _ in range(2):
        eng.render_async(cam)
    out = eng.render_flush()
    assert eng._latest is not None           # the side buffer set
    tiles = _sample_tiles(cam, 12, seed=17)
    ref = O.render(hc, cam, med, "underwater", tiles=tiles)
    _check_images(out, ref, _tile_mask(cam, tiles))
    api = uw.render(cloud, cam, m, "underwater")
    for f in ("color", "depth", "count", "final_transmittance", "last"):
        assert torch.equal(getattr(api, f), getattr(out, f)), f


def test_c4_3m_backward_sampled_tiles():
    """3M Gaussians at 1080p (C4's per-view size): every parameter gradient with
    dL/dC restricted to seeded tiles, against the oracle."""
    hc = host_cloud(3_000_000, seed=6)
    cam = survey_camera(1920, 1080)
    med = survey_medium()
    cloud, m = _device(hc, med)
    out = uw.render(cloud, cam, m, "underwater")
    tiles = _sample_tiles(cam, 12, seed=8)
    mask = _tile_mask(cam, tiles)
    rng = np.random.default_rng(10)
    dL = np.where(mask[..., None], rng.normal(size=(cam.height, cam.width, 3)), 0.0) / mask.sum()
    buf = uw.backward_render(out, torch.as_tensor(dL, dtype=torch.float32).cuda(), cloud, m, 0.1)
    ref = O.render(hc, cam, med, "underwater", tiles=tiles)
    _check_images(out, ref, mask)
    g = O.backward(ref, dL.astype(np.float32).astype(np.float64), len(hc.positions), med, 0.1,
                   tiles=tiles)
    _check_grads(buf, g)


# ----------------------------------------------------------------------------
# StepEngine vs the oracle, before and after Adam
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["gradcheck", "survey2k", "opaque3k", "c1"])
def test_engine_gradients_and_adam_vs_oracle(name):
    if name == "c1":
        hc = host_cloud(10_000, seed=2)
        cam = uw.Camera.from_any(survey_camera(256, 256))
        med = survey_medium()
        cloud, medium = _device(hc, med)
        gt = np.random.default_rng(3).uniform(0, 1, (256, 256, 3))
        lam = (0.3, 0.1)
    else:
        g = load(name)
        if g.mode != "underwater":
            pytest.skip("the engine trains in underwater mode")
        hc, med, gt, lam = g.cloud, g.medium, g.gt, g.lambdas
        cloud, cam, medium = device_scene(g)
    cfg = uw.OptimConfig(lambda_ssim=lam[0], lambda_guide=lam[1])
    params0, med0 = host_state(cloud, medium)
    state = uw.TrainState(cloud, medium, iteration=1)
    eng = uw.StepEngine(state, cam.width, cam.height, cfg)
    eng.keep_gradients = True
    st = eng.step([(cam, torch.as_tensor(gt, dtype=torch.float32))])   # host image path
    assert not st.skipped
    # forward: the engine's render vs the oracle, every pixel
    ref = O.render(hc, cam, med, "underwater")
    o = eng.last_render()
    _check_images(o, ref)
    # loss + dL/dC on the engine's own image
    gt32 = np.asarray(gt, np.float32).astype(np.float64)
    bd_ref, dL_ref = O.total_loss(np_(o.color).astype(np.float64), gt32, med, *lam)
    np.testing.assert_allclose(st.total, bd_ref["total"], rtol=2e-5)
    assert np.abs(np_(eng.dL) - dL_ref).max() <= 1e-4 * np.abs(dL_ref).max()
    # summed gradient buffer before Adam vs the oracle backward of that dL/dC
    gref = O.backward(ref, np_(eng.dL).astype(np.float64), len(hc.positions), med, lam[1])
    _check_grads(eng.grads, gref)
    # densification statistics accumulated by the fused Adam
    np.testing.assert_array_equal(np_(state.obs_count), np_(eng.grads.observed).astype(np.int32))
    np.testing.assert_array_equal(np_(state.grad_accum),
                                  np.where(np_(eng.grads.observed),
                                           np_(eng.grads.mean2d_grad_norm), 0).astype(np.float32))
    # Adam: bit-exact vs the reference update on the engine's own float32 gradients
    p1, m1, _ = adam_replay(params0, host_grads(eng.grads), med0, 1, cfg)
    for f, v in p1.items():
        np.testing.assert_array_equal(np_(getattr(state.cloud, f)), v, err_msg=f)
    for f, v in m1.items():
        np.testing.assert_array_equal(np_(getattr(state.medium, f)), v, err_msg=f)


# ----------------------------------------------------------------------------
# the float64 fix-up of the T >= 1e-4 decisions, through every list source
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("source", ["stored_rows", "small_cap", "row_filter", "tile_lists"])
def test_exact_transmittance_decisions_every_list_source(c1, source, monkeypatch):
    """count / last / T exact whichever list the float64 re-walk reads: the rows the
    forward stored per tile, a cap so small that it continues by filtering the row
    list, no stored rows at all, or the materialised CSR tile lists."""
    hc, cam, med, cloud, m, ref_proj = c1
    ref = O.render(hc, cam, med, "underwater", proj=ref_proj)
    if source == "small_cap":
        monkeypatch.setattr(uw.rasterizer, "TILE_ROWS_CAP", 8)
    if source == "tile_lists":
        proj = uw.project_cloud(cloud, cam)
        out = uw.composite(proj, uw.bin_and_sort(proj, cam.width, cam.height), cam, m,
                           "underwater")
    elif source == "row_filter":
        import ctypes
        from paper_2411_19588_b200 import _lib
        from paper_2411_19588_b200.rasterizer import _alloc_output, bin_rows
        proj = uw.project_cloud(cloud, cam, with_geometry=False)
        rows = bin_rows(proj, cam.width, cam.height)
        out = _alloc_output(cam.height, cam.width, proj.device, "underwater", False,
                            tile_rows=False)
        pc, cc, oc = proj.c_struct(), cam.c_struct(), out.c_struct()
        _lib.call("uws_raster_fwd_rows", ctypes.byref(pc), _lib.ptr(rows.row_start),
                  _lib.ptr(rows.items), ctypes.byref(cc), _lib.ptr(m.flat), ctypes.byref(oc),
                  _lib.stream_handle())
    else:
        out = uw.render(cloud, cam, m, "underwater")
    _check_images(out, ref)
    assert int(out.fix_count[:2].abs().sum()) == 0    # left zero for the next call
