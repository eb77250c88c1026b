"""CUDA path vs the float64 oracle at the survey's sizes (GPU).

C2 (100k Gaussians, 800x600, underwater + guidance): projection and binning in
full, compositing forward/backward on seeded tile subsets (the oracle costs
~10-30 us per tile entry).  C3 (1M, 1920x1080): size-independent structural
properties of the bins and the render.  Tolerances as in test_gpu_golden.
"""

import numpy as np
import pytest
import torch

import paper_2411_19588_b200 as uw
from gpu_util import GRAD_FIELDS, grad_tolerance_ok, host_cloud, np_, survey_camera, survey_medium
from oracle import uwsplat_oracle as O

pytestmark = pytest.mark.gpu


def _device(hc, med):
    cloud = uw.GaussianCloud(**vars(hc))
    m = None if med is None else uw.MediumParams(med.attenuation, med.water_color, med.backscatter,
                                                 med.water_color_guide, med.backscatter_guide)
    return cloud, m


@pytest.fixture(scope="module")
def c2():
    hc = host_cloud(100_000, seed=0)
    cam = survey_camera(800, 600)
    med = survey_medium()
    cloud, m = _device(hc, med)
    proj_ref = O.project(hc, cam)
    return hc, cam, med, cloud, m, proj_ref


def _proj_ns(p):
    """GPU projection as an oracle-compatible namespace (float64 fields)."""
    from types import SimpleNamespace
    return SimpleNamespace(source_index=np_(p.source_index).astype(np.int64),
                           mean2d=np_(p.mean2d), radius=np_(p.radius), depth=np_(p.depth),
                           conic=np_(p.conic), opacity=np_(p.opacity),
                           color=np_(p.color).astype(np.float64))


def test_c2_projection_exact(c2):
    hc, cam, med, cloud, m, ref = c2
    p = uw.project_cloud(cloud, cam)
    np.testing.assert_array_equal(np_(p.source_index), ref.source_index)
    np.testing.assert_array_equal(np_(p.mean2d), ref.mean2d)
    np.testing.assert_array_equal(np_(p.depth), ref.depth)
    np.testing.assert_allclose(np_(p.radius), ref.radius, rtol=1e-12, atol=0)
    np.testing.assert_allclose(np_(p.conic), ref.conic, rtol=1e-10, atol=1e-14)


def test_c2_bins_bit_exact(c2):
    hc, cam, med, cloud, m, ref = c2
    p = uw.project_cloud(cloud, cam)
    bins = uw.bin_and_sort(p, cam.width, cam.height)
    # stage-isolated: the reference binning applied to the GPU's own projection
    offs, ent = O.tile_lists(_proj_ns(p), cam.width, cam.height)
    np.testing.assert_array_equal(np_(bins.offsets).astype(np.int64), offs)
    np.testing.assert_array_equal(np_(bins.entries).astype(np.int64), ent)
    # end to end: the reference binning of the oracle's projection
    offs2, ent2 = O.tile_lists(ref, cam.width, cam.height)
    np.testing.assert_array_equal(offs, offs2)
    np.testing.assert_array_equal(ent, ent2)


def _sample_tiles(cam, n, seed=3):
    gx, gy = O.grid_dims(cam.width, cam.height)
    return np.sort(np.random.default_rng(seed).choice(gx * gy, n, replace=False))


def test_c2_render_sampled_tiles(c2):
    hc, cam, med, cloud, m, ref = c2
    out = uw.render(cloud, cam, m, "underwater")
    tiles = _sample_tiles(cam, 40)
    bins = (np_(out.bins.offsets).astype(np.int64), np_(out.bins.entries).astype(np.int64))
    o = O.render(hc, cam, med, "underwater", tiles=tiles, proj=ref, bins=bins)
    gx, _ = O.grid_dims(cam.width, cam.height)
    mask = np.zeros((cam.height, cam.width), bool)
    for t in tiles:
        ty, tx = divmod(int(t), gx)
        mask[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    assert np.abs(np_(out.color)[mask] - o.color[mask]).max() < 1e-4
    assert np.abs(np_(out.color_clean)[mask] - o.color_clean[mask]).max() < 1e-4
    np.testing.assert_allclose(np_(out.depth)[mask], o.depth[mask], rtol=1e-5)
    # the T >= 1e-4 decisions are exact (float64 fix-up pass): counts bit-exact
    np.testing.assert_array_equal(np_(out.count)[mask], o.count[mask])


def test_c2_loss_full_frame(c2):
    hc, cam, med, cloud, m, ref = c2
    out = uw.render(cloud, cam, m, "underwater")
    gt = np.random.default_rng(0).uniform(0, 1, (cam.height, cam.width, 3))
    img = np_(out.color).astype(np.float64)
    bd_ref, g_ref = O.total_loss(img, gt, med, 0.3, 0.1)
    bd, g = uw.total_loss(out.color, gt, m, 0.3, 0.1)
    np.testing.assert_allclose([bd.l1, bd.d_ssim, bd.l_bs, bd.total],
                               [bd_ref["l1"], bd_ref["d_ssim"], bd_ref["l_bs"], bd_ref["total"]],
                               rtol=2e-5)
    err = np.abs(np_(g) - g_ref)
    assert err.max() <= 1e-3 * np.abs(g_ref).max()
    assert np.median(err / np.maximum(np.abs(g_ref), 1e-30)) < 1e-4


def test_c2_backward_sampled_tiles(c2):
    """dL/dC restricted to seeded tiles: the other tiles contribute exactly zero."""
    hc, cam, med, cloud, m, ref = c2
    out = uw.render(cloud, cam, m, "underwater")
    tiles = _sample_tiles(cam, 24, seed=5)
    gx, _ = O.grid_dims(cam.width, cam.height)
    rng = np.random.default_rng(9)
    dL = np.zeros((cam.height, cam.width, 3))
    for t in tiles:
        ty, tx = divmod(int(t), gx)
        dL[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = rng.normal(
            size=dL[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16].shape) / dL.size
    buf = uw.backward_render(out, torch.as_tensor(dL, dtype=torch.float32).cuda(), cloud, m, 0.1)
    bins = (np_(out.bins.offsets).astype(np.int64), np_(out.bins.entries).astype(np.int64))
    # dL/dC is zero outside the sampled tiles, so only their depth/colour matter
    o = O.render(hc, cam, med, "underwater", tiles=tiles, proj=ref, bins=bins)
    g = O.backward(o, dL, len(hc.positions), med, 0.1, tiles=tiles)
    for f in GRAD_FIELDS:
        bad, worst = grad_tolerance_ok(np_(getattr(buf, f)), g[f])
        assert bad == 0, f"{f}: {bad} out of tolerance (worst rel {worst:.2e})"
    np.testing.assert_array_equal(np_(buf.observed), g["observed"])
    for f in ("d_attenuation", "d_water_color", "d_backscatter"):
        np.testing.assert_allclose(np_(getattr(buf, f)), g[f], rtol=1e-4,
                                   atol=1e-6 * np.abs(g[f]).max())


@pytest.fixture(scope="module")
def c3():
    hc = host_cloud(1_000_000, seed=0)
    cam = survey_camera(1920, 1080)
    cloud, m = _device(hc, survey_medium())
    out = uw.render(cloud, cam, m, "underwater")
    return hc, cam, cloud, m, out


def test_c3_bins_structure(c3):
    hc, cam, cloud, m, out = c3
    proj, bins = out.proj, out.bins
    gx, gy = cam.grid
    offs = bins.offsets.long()
    ent = bins.entries.long()
    E = ent.numel()
    rect = proj.rect.long()
    cnt = ((rect[:, 2] - rect[:, 0] + 1).clamp(min=0) * (rect[:, 3] - rect[:, 1] + 1).clamp(min=0))
    assert int(cnt.sum()) == E == int(offs[-1])
    assert bool((offs[1:] >= offs[:-1]).all()) and int(offs[0]) == 0
    tile_of = torch.repeat_interleave(torch.arange(gx * gy, device=offs.device), offs[1:] - offs[:-1])
    tx, ty = tile_of % gx, tile_of // gx
    r = rect[ent]
    assert bool(((tx >= r[:, 0]) & (tx <= r[:, 2]) & (ty >= r[:, 1]) & (ty <= r[:, 3])).all())
    d = proj.depth[ent]
    s = proj.source_index.long()[ent]
    same = tile_of[1:] == tile_of[:-1]
    ordered = (d[1:] > d[:-1]) | ((d[1:] == d[:-1]) & (s[1:] > s[:-1]))
    assert bool((ordered | ~same).all())
    # each (tile, Gaussian) pair appears once: counts per Gaussian match rects
    per_g = torch.bincount(ent, minlength=len(proj))
    assert bool((per_g == cnt).all())


def test_c3_render_properties(c3):
    hc, cam, cloud, m, out = c3
    w, tf = out.weight, out.final_transmittance
    live = tf >= 1e-4
    assert float((w + tf - 1).abs()[live].max()) < 2e-5
    assert bool((out.depth >= cam.near).all()) and bool((out.depth <= cam.far).all())
    assert bool(torch.isfinite(out.color).all())
    assert float(out.count.float().mean()) > 10


def test_c3_render_sampled_tiles(c3):
    hc, cam, cloud, m, out = c3
    p = uw.project_cloud(cloud, cam)      # same projection, with radius/cov2d materialised
    tiles = _sample_tiles(cam, 12, seed=11)
    bins = (np_(out.bins.offsets).astype(np.int64), np_(out.bins.entries).astype(np.int64))
    o = O.render(hc, cam, survey_medium(), "underwater", tiles=tiles, proj=_proj_ns(p), bins=bins)
    gx, _ = cam.grid
    mask = np.zeros((cam.height, cam.width), bool)
    for t in tiles:
        ty, tx = divmod(int(t), gx)
        mask[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    assert np.abs(np_(out.color)[mask] - o.color[mask]).max() < 1e-4
    np.testing.assert_allclose(np_(out.depth)[mask], o.depth[mask], rtol=1e-5)


# ----------------------------------------------------------------------------
# edge cases
# ----------------------------------------------------------------------------
def _cloud_from(pos, logit=2.0, scale=0.3, color=(1.0, 0.0, 0.0)):
    pos = np.asarray(pos, np.float32).reshape(-1, 3)
    n = len(pos)
    sh = np.tile(((np.asarray(color) - 0.5) / uw.scene.SH_C0)[None, None, :], (n, 1, 1))
    return uw.GaussianCloud(pos, np.full((n, 3), np.log(scale), np.float32),
                            np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1)), sh,
                            np.full(n, logit, np.float32))


def _front(w=32, h=32, f=40.0):
    return uw.Camera(width=w, height=h, fx=f, fy=f, cx=w / 2, cy=h / 2, R=np.eye(3),
                     t=np.zeros(3), near=0.1, far=60.0)


def test_empty_and_culled_clouds():
    cam = _front()
    med = survey_medium(guided=False)
    m = uw.MediumParams(med.attenuation, med.water_color, med.backscatter)
    for cloud in (_cloud_from(np.zeros((0, 3))), _cloud_from([[0, 0, -5.0], [0, 0, 80.0]])):
        out = uw.render(cloud, cam, m, "underwater")
        assert len(out.proj) == 0 and out.bins.entries.numel() == 0
        assert float(out.weight.abs().max()) == 0 and float((out.final_transmittance - 1).abs().max()) == 0
        assert float((out.depth - cam.far).abs().max()) == 0
        z = O.logistic(cam.far)
        water = med.water_color * (1 - np.exp(-med.backscatter.astype(np.float64) * z))
        assert np.abs(np_(out.color) - water).max() < 1e-6
        dL = torch.full((32, 32, 3), 1e-3, device="cuda")
        buf = uw.backward_render(out, dL, cloud, m, 0.0)
        assert float(buf.params.abs().max() if buf.n else 0) == 0
        ref = O.medium_grads(np.full((32, 32), cam.far), np.zeros((32, 32, 3)), np_(dL), med, 0.0)
        np.testing.assert_allclose(np_(buf.medium), np.concatenate(ref), rtol=1e-5)


def test_single_opaque_gaussian_kat():
    """single opaque contributor of colour (1,0,0) at depth 2 -> (0.99,0,0), z=2."""
    cam = _front()
    # centred on pixel (16,16): centre (16.5,16.5) -> world x = 0.5*z/f
    z = 2.0
    cloud = _cloud_from([[0.5 * z / 40.0, 0.5 * z / 40.0, z]], logit=20.0, scale=0.05)
    out = uw.render(cloud, cam)
    c = np_(out.color)[16, 16]
    np.testing.assert_allclose(c, [0.99, 0, 0], atol=1e-6)
    assert abs(float(out.depth[16, 16]) - z) < 1e-6 and int(out.count[16, 16]) == 1


def test_zero_medium_equals_clean():
    hc = host_cloud(3000, seed=4)
    cam = survey_camera(96, 80)
    cloud = uw.GaussianCloud(**vars(hc))
    clean = uw.render(cloud, cam)
    uwz = uw.render(cloud, cam, uw.MediumParams.zero(), "underwater")
    assert torch.equal(clean.color, uwz.color)


def test_errors():
    cloud = _cloud_from([[0, 0, 5.0]])
    with pytest.raises(ValueError):
        uw.render(cloud, _front(), mode="bogus")
    with pytest.raises(ValueError):
        uw.render(cloud, _front(), mode="underwater")
    with pytest.raises(uw.DataError):
        uw.total_loss(torch.zeros(8, 8, 3, device="cuda"), np.zeros((8, 8, 3)), None)
    with pytest.raises(uw.DataError):
        uw.total_loss(torch.zeros(16, 16, 3, device="cuda"), np.zeros((16, 12, 3)), None)
    out = uw.render(cloud, _front(), retain=False)
    with pytest.raises(ValueError):
        uw.backward_render(out, torch.zeros(32, 32, 3, device="cuda"), cloud)


def test_multiview_accumulation_is_sum_of_views():
    hc = host_cloud(4000, seed=6)
    med = survey_medium()
    cloud, m = _device(hc, med)
    cams = [uw.Camera.look_at((3 + 0.4 * k, -2, -1), (0, 0, 12), width=80, height=64, fx=96, fy=96)
            for k in range(3)]
    rng = np.random.default_rng(0)
    total = uw.GradientBuffer(len(cloud))
    singles = []
    for cam in cams:
        out = uw.render(cloud, cam, m, "underwater")
        dL = torch.as_tensor(rng.normal(size=(64, 80, 3)) * 1e-4, dtype=torch.float32).cuda()
        uw.backward_render(out, dL, cloud, m, 0.1, buf=total)
        singles.append(np_(uw.backward_render(out, dL, cloud, m, 0.1).flat).astype(np.float64))
    ref = np.sum(singles, axis=0)
    got = np_(total.flat)
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()


def test_train_step_matches_oracle_step():
    from golden_util import load
    g = load("survey2k")
    cloud, m = _device(g.cloud, g.medium)
    cam = uw.Camera.from_any(g.cam)
    state = uw.TrainState(cloud, m, iteration=1)
    cfg = uw.OptimConfig()
    st = uw.train_step(state, cam, g.gt, cfg)
    assert not st.skipped
    np.testing.assert_allclose(st.total, g.d["loss"][3], rtol=1e-5)
    # Adam's first step is lr * g/|g| per element: compare with the reference's update
    for f in ("positions", "log_scales", "sh_coeffs", "opacity_logits"):
        got, ref = np_(getattr(cloud, f)), g.d["adam_" + f]
        close = np.abs(got - ref) <= 1e-6 * np.maximum(np.abs(ref), 1.0)
        assert close.mean() > 0.995, f"{f}: {close.mean():.4f}"
        # every element: a first Adam step moves a scalar by at most lr (m/sqrt(v) = g/|g|),
        # so two runs whose gradients differ in rounding stay within 2 lr of each other
        lr = cfg.position_lr_init if f == "positions" else getattr(cfg, uw.optim._LR_FIELDS[f])
        assert np.abs(got - ref).max() <= 2.0 * lr * 1.0001 + 1e-7, f
    assert int(state.obs_count.sum()) == int(g.d["grad_observed"].sum())
