"""The sync-free StepEngine (persistent buffers, device-side sizes, fused
skip/densify/zeroing) against the reference-API step path (GPU)."""

import numpy as np
import pytest
import torch

import paper_2411_19588_b200 as uw
from golden_util import load
from gpu_util import (GRAD_FIELDS, adam_replay, device_scene, grad_tolerance_ok, host_grads,
                      host_state, np_)

pytestmark = pytest.mark.gpu

FIELDS = ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits")


def _state(g):
    cloud, cam, medium = device_scene(g)
    return uw.TrainState(cloud, medium, iteration=1), cam


def _grads_close(a, b, rel=1e-4, abs_frac=1e-6):
    """Two gradient buffers of the same inputs through the same kernels: equal up
    to the order of the float atomics, on EVERY element."""
    for f in GRAD_FIELDS + ("mean2d_grad_norm",):
        bad, worst = grad_tolerance_ok(np_(getattr(a, f)), np_(getattr(b, f)), rel, abs_frac)
        assert bad == 0, f"{f}: {bad} out of tolerance (worst rel {worst:.2e})"
    assert torch.equal(a.observed, b.observed)
    np.testing.assert_allclose(np_(a.medium), np_(b.medium), rtol=1e-5, atol=1e-9)


def _lr(cfg, f):
    return cfg.position_lr_init if f == "positions" else getattr(cfg, uw.optim._LR_FIELDS[f])


def _trajectory_close(sa, sb, cfg, steps):
    """Two runs of ``steps`` Adam steps whose gradients differ only by float-atomic
    order: >= 99.9 % of the parameters agree to 1e-6, and EVERY parameter within
    the largest distance two Adam trajectories can drift apart (|update| <=
    lr * sqrt((1-b1)^2 / (1-b2)) ~ 3.17 lr per step, plus renormalisation)."""
    for f in FIELDS:
        a, b = np_(getattr(sa.cloud, f)), np_(getattr(sb.cloud, f))
        d = np.abs(a - b)
        assert (d <= 1e-6 * np.maximum(np.abs(b), 1.0)).mean() >= 0.999, f
        bound = 2 * steps * 3.17 * _lr(cfg, f) * (2.0 if f == "rotations" else 1.0) + 1e-6
        assert d.max() <= bound, f"{f}: max deviation {d.max():.3g} > {bound:.3g}"


def test_engine_step_matches_api_step():
    """Engine (the timed path) vs the API step: identical loss and gradients before
    Adam (every element), and each Adam update bit-exact against the reference
    adam_step on the engine's own float32 gradients (two steps: moments chained)."""
    g = load("survey2k")
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    cfg = uw.OptimConfig()
    sa, cam = _state(g)
    sb, _ = _state(g)
    eng = uw.StepEngine(sa, cam.width, cam.height, cfg)
    eng.keep_gradients = True
    bufb = uw.GradientBuffer(len(sb.cloud))
    moments = None
    for it in range(2):
        pa, ma = host_state(sa.cloud, sa.medium)
        eng.grads.zero_()
        st = eng.step([(cam, gt)])
        ref = uw.train_step(sb, cam, gt, cfg, buf=bufb)
        assert not st.skipped and not ref.skipped
        if it == 0:   # identical inputs on both sides
            np.testing.assert_allclose(st.total, ref.total, rtol=1e-6)
            _grads_close(eng.grads, bufb)
            assert torch.equal(sa.obs_count, sb.obs_count)
            np.testing.assert_allclose(np_(sa.grad_accum), np_(sb.grad_accum), rtol=1e-4,
                                       atol=1e-9)
        p1, m1, moments = adam_replay(pa, host_grads(eng.grads), ma, sa.iteration, cfg,
                                      moments, step=it + 1)
        for f, v in p1.items():
            np.testing.assert_array_equal(np_(getattr(sa.cloud, f)), v, err_msg=f)
        for f, v in m1.items():
            np.testing.assert_array_equal(np_(getattr(sa.medium, f)), v, err_msg=f)
        sa.iteration += 1
        sb.iteration += 1
    assert all(sa.adam[k].step == sb.adam[k].step == 2 for k in sa.adam)
    _trajectory_close(sa, sb, cfg, 2)


def test_engine_zeroes_consumed_gradients():
    g = load("survey2k")
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    s, cam = _state(g)
    eng = uw.StepEngine(s, cam.width, cam.height, uw.OptimConfig())
    for _ in range(2):
        assert not eng.step([(cam, gt)]).skipped
        s.iteration += 1
    assert float(eng.grads.flat.abs().max()) == 0.0


def test_engine_overflow_grows_and_reruns():
    g = load("survey2k")
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    cfg = uw.OptimConfig()
    sa, cam = _state(g)
    sb, _ = _state(g)
    small = uw.StepEngine(sa, cam.width, cam.height, cfg, entry_capacity=64)
    big = uw.StepEngine(sb, cam.width, cam.height, cfg)
    small.keep_gradients = big.keep_gradients = True
    pa, ma = host_state(sa.cloud, sa.medium)
    st = small.step([(cam, gt)])
    assert st.reruns >= 1 and not st.skipped
    assert small.s_cap >= 64
    big.step([(cam, gt)])
    assert all(sa.adam[k].step == 1 for k in sa.adam)
    _grads_close(small.grads, big.grads)
    p1, _, _ = adam_replay(pa, host_grads(small.grads), ma, 1, cfg)
    for f, v in p1.items():
        np.testing.assert_array_equal(np_(getattr(sa.cloud, f)), v, err_msg=f)


def test_engine_nonfinite_skips_on_device():
    g = load("gradcheck")
    cfg = uw.OptimConfig()
    s, cam = _state(g)
    eng = uw.StepEngine(s, cam.width, cam.height, cfg)
    before = s.cloud.flat.clone()
    gt = torch.full((cam.height, cam.width, 3), float("nan"), device="cuda")
    st = eng.step([(cam, gt)])
    assert st.skipped
    assert torch.equal(s.cloud.flat, before)
    assert all(slot.step == 0 for slot in s.adam.values())
    assert int(s.obs_count.sum()) == 0
    # the next (finite) step proceeds normally
    st = eng.step([(cam, torch.as_tensor(g.gt, dtype=torch.float32).cuda())])
    assert not st.skipped and all(slot.step == 1 for slot in s.adam.values())


@pytest.mark.parametrize("name", ["survey2k", "clean500", "opaque3k"])
def test_row_list_render_matches_tile_list_render(name):
    """Tiles filtering their row lists on the fly == the materialised tile lists, bitwise."""
    g = load(name)
    s, cam = _state(g)
    mode = g.mode
    med = s.medium if mode == "underwater" else None
    # the tile-list kernel on the materialised CSR lists (rasterizer.bin_and_sort)
    proj = uw.project_cloud(s.cloud, cam)
    ref = uw.composite(proj, uw.bin_and_sort(proj, cam.width, cam.height), cam, med, mode)
    api = uw.render(s.cloud, cam, med, mode)     # row lists, materialised on demand only
    for f in ("color", "depth", "weight", "final_transmittance", "count", "last"):
        assert torch.equal(getattr(api, f), getattr(ref, f)), f
    eng = uw.StepEngine(s, cam.width, cam.height, uw.OptimConfig(), entry_capacity=16)
    out = eng.render(cam, mode)      # tiny capacity: exercises the overflow re-run
    for f in ("color", "depth", "weight", "final_transmittance", "count", "last"):
        assert torch.equal(getattr(out, f), getattr(ref, f)), f


def _run(eng, state, views, pipelined):
    """Drive an engine over a list of (cam, gt) views, one view per step."""
    out = []
    for v in views:
        if pipelined:
            r = eng.step_async([v])
            if r is not None:
                out.append(r)
        else:
            out.append(eng.step([v]))
        state.iteration += 1
    if pipelined:
        out.append(eng.flush())
    return out


@pytest.mark.parametrize("cap", [0, 64])
def test_pipelined_steps_match_synchronous(cap):
    """step_async (host GT copied on the side stream, result read one step late)
    == step(), including a non-finite step in the middle (the queued step behind
    it is discarded and re-launched) and, with cap=64, overflow re-runs."""
    g = load("survey2k")
    gt_host = torch.as_tensor(g.gt, dtype=torch.float32).pin_memory()
    nan = torch.full_like(gt_host, float("nan"))
    cfg = uw.OptimConfig()
    sa, cam = _state(g)
    sb, _ = _state(g)
    ea = uw.StepEngine(sa, cam.width, cam.height, cfg, entry_capacity=cap)
    eb = uw.StepEngine(sb, cam.width, cam.height, cfg, entry_capacity=cap)
    views = [(cam, gt_host), (cam, gt_host), (cam, nan), (cam, gt_host), (cam, gt_host)]
    ra = _run(ea, sa, views, pipelined=True)
    rb = _run(eb, sb, views, pipelined=False)
    assert [r.skipped for r in ra] == [r.skipped for r in rb] == [False, False, True, False, False]
    for x, y in zip(ra, rb):
        if not x.skipped:
            np.testing.assert_allclose(x.total, y.total, rtol=1e-5)
    assert all(sa.adam[k].step == sb.adam[k].step == 4 for k in sa.adam)
    _trajectory_close(sa, sb, cfg, 4)
    assert torch.equal(sa.obs_count, sb.obs_count)
    assert float(ea.grads.flat.abs().max()) == 0.0


def test_engine_with_nothing_visible():
    """Every Gaussian behind the camera: K = 0 through sort, lists, both raster
    kernels and Adam; the image is the medium alone and only the medium learns."""
    g = load("survey2k")
    s, cam = _state(g)
    pos = s.cloud.positions.clone()
    pos[:, 2] = -50.0                       # behind the look_at camera
    s.cloud.positions.copy_(pos)
    before = {f: getattr(s.cloud, f).clone() for f in FIELDS}
    eng = uw.StepEngine(s, cam.width, cam.height, uw.OptimConfig())
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    st = eng.step([(cam, gt)])
    assert not st.skipped and np.isfinite(st.total)
    out = eng.last_render()
    assert int(out.count.sum()) == 0
    for f in FIELDS:   # zero gradients: only the renormalisation touches rotations
        if f != "rotations":
            assert torch.equal(getattr(s.cloud, f), before[f]), f
    assert float(s.medium_exp_avg.abs().sum()) > 0.0
    r = eng.render(cam)
    assert int(r.count.sum()) == 0


def test_engine_two_views_per_step_equals_summed_api_gradients():
    """max_views=2: the engine's step (first view stores, second accumulates) ==
    apply_gradients on the sum of the two API backward buffers."""
    g = load("survey2k")
    sa, cam0 = _state(g)
    sb, _ = _state(g)
    cam1 = uw.Camera.look_at((2.5, -2.2, -1.2), (0, 0, 12), width=cam0.width,
                             height=cam0.height, fx=cam0.fx, fy=cam0.fy)
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    cfg = uw.OptimConfig()
    eng = uw.StepEngine(sa, cam0.width, cam0.height, cfg, max_views=2)
    eng.keep_gradients = True
    pa, ma = host_state(sa.cloud, sa.medium)
    st = eng.step([(cam0, gt), (cam1, gt)])
    assert not st.skipped and st.views == 2
    buf = uw.GradientBuffer(len(sb.cloud))
    for cam in (cam0, cam1):
        out = uw.render(sb.cloud, cam, sb.medium, "underwater")
        _, dL = uw.total_loss(out.color, gt, sb.medium, cfg.lambda_ssim, cfg.lambda_guide)
        uw.backward_render(out, dL, sb.cloud, sb.medium, cfg.lambda_guide, buf=buf)
    _grads_close(eng.grads, buf)
    p1, _, _ = adam_replay(pa, host_grads(eng.grads), ma, 1, cfg)
    for f, v in p1.items():
        np.testing.assert_array_equal(np_(getattr(sa.cloud, f)), v, err_msg=f)


@pytest.mark.parametrize("nviews", [3, 4])
def test_overlapped_views_equal_serial_views(nviews):
    """Several views per step on two streams / buffer sets (overlap_views) == the same
    views one after another on one stream: per-view losses and the summed gradients,
    over two steps (the second after an Adam update), and the guidance refresh reads
    the last view's depth from whichever set holds it."""
    g = load("survey2k")
    _, cam0 = _state(g)
    cams = [cam0] + [uw.Camera.look_at((2.5 - 0.2 * k, -2.2 + 0.1 * k, -1.2), (0, 0, 12),
                                       width=cam0.width, height=cam0.height, fx=cam0.fx,
                                       fy=cam0.fy) for k in range(1, nviews)]
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    res = []
    for overlap in (False, True):
        s, _ = _state(g)
        eng = uw.StepEngine(s, cams[0].width, cams[0].height, uw.OptimConfig(), max_views=nviews)
        eng.overlap_views = overlap
        eng.keep_gradients = True
        stats = []
        for _ in range(2):
            st = eng.step([(c, gt) for c in cams])
            assert not st.skipped
            stats.append(st.total)
        grads = np_(eng.grads.flat).copy()
        depth = np_(eng.out.depth if eng._last_view_set is None
                    else eng._last_view_set.out.depth).copy()
        res.append((stats, grads, depth))
    (sa, ga, da), (sb, gb, db) = res
    np.testing.assert_allclose(sa, sb, rtol=1e-6)
    np.testing.assert_array_equal(da, db)
    n = (ga.size - 16) // 16
    bad, worst = grad_tolerance_ok(gb[:14 * n], ga[:14 * n], rel=1e-4, abs_frac=1e-6)
    assert bad == 0, worst


@pytest.mark.parametrize("name", ["survey2k", "opaque3k"])
def test_tile_list_backward_matches_row_list_backward(name):
    """backward_render through the materialised tile lists (composite) == through the
    row lists (render): same pairs, same order, same partials."""
    g = load(name)
    s, cam = _state(g)
    med = s.medium if g.mode == "underwater" else None
    mode = g.mode
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    out_rows = uw.render(s.cloud, cam, med, mode)
    proj = uw.project_cloud(s.cloud, cam)
    out_tiles = uw.composite(proj, uw.bin_and_sort(proj, cam.width, cam.height), cam, med, mode)
    assert out_tiles.rows is None and out_rows.rows is not None
    bufs = []
    for out in (out_rows, out_tiles):
        _, dL = uw.total_loss(out.color, gt, med, 0.3, 0.1)
        bufs.append(np_(uw.backward_render(out, dL, s.cloud, med, 0.1).flat).astype(np.float64))
    a, b = bufs
    assert np.abs(a - b).max() <= 1e-5 * max(np.abs(b).max(), 1e-30)


@pytest.mark.parametrize("name", ["survey2k", "opaque3k"])
def test_forward_stored_rows_are_the_tile_list_prefix(name):
    """tile_rows[t, :tile_nrows[t]] is the head of tile t's list in the reference order
    (the rows the forward staged, reused by the backward)."""
    g = load(name)
    s, cam = _state(g)
    med = s.medium if g.mode == "underwater" else None
    out = uw.render(s.cloud, cam, med, g.mode)
    offs = np_(out.bins.offsets).astype(np.int64)
    ent = np_(out.bins.entries).astype(np.int64)
    rows, nrows = np_(out.tile_rows), np_(out.tile_nrows)
    last = np_(out.last)
    assert nrows.shape[0] == offs.shape[0] - 1 and (nrows > 0).any()
    gx = (cam.width + 15) // 16
    complete = (nrows & (1 << 30)) != 0
    nrows = nrows & ~(1 << 30)
    for t in range(nrows.shape[0]):
        n = int(nrows[t])
        assert n <= offs[t + 1] - offs[t]
        # flagged complete <=> the stored rows are the tile's whole list
        if complete[t]:
            assert n == offs[t + 1] - offs[t]
        np.testing.assert_array_equal(rows[t, :n], ent[offs[t]:offs[t] + n])
        ty, tx = divmod(t, gx)
        consumed = last[16 * ty:16 * ty + 16, 16 * tx:16 * tx + 16].max()
        assert consumed <= n or n == uw.rasterizer.TILE_ROWS_CAP


@pytest.mark.parametrize("name", ["survey2k", "opaque3k"])
def test_backward_from_stored_rows_matches_refiltering(name, monkeypatch):
    """The backward reading the forward's stored rows == re-filtering the row lists,
    also when a small cap sends the longer tiles down the re-filtering path."""
    g = load(name)
    s, cam = _state(g)
    med = s.medium if g.mode == "underwater" else None
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    outs = [uw.render(s.cloud, cam, med, g.mode)]
    monkeypatch.setattr(uw.rasterizer, "TILE_ROWS_CAP", 8)
    outs.append(uw.render(s.cloud, cam, med, g.mode))
    assert outs[1].tile_rows.shape[1] == 8
    outs.append(uw.render(s.cloud, cam, med, g.mode))
    outs[2].tile_rows = outs[2].tile_nrows = None      # re-filter every tile
    bufs = []
    for out in outs:
        _, dL = uw.total_loss(out.color, gt, med, 0.3, 0.1)
        bufs.append(np_(uw.backward_render(out, dL, s.cloud, med, 0.1).flat).astype(np.float64))
    for a in bufs[:2]:
        assert np.abs(a - bufs[2]).max() <= 1e-5 * max(np.abs(bufs[2]).max(), 1e-30)


@pytest.mark.parametrize("parts", [1, 3, 7])
def test_range_update_equals_single_launch(parts):
    """The cloud update split into group ranges (as after a chunked all-reduce) gives the
    single launch's parameters, moments, densification statistics and zeroed buffer."""
    from paper_2411_19588_b200.optim import apply_gradients_device, range_chunks
    g = load("survey2k")
    results = []
    for chunked in (False, True):
        s, _ = _state(g)
        s.iteration = 7
        n = len(s.cloud)
        buf = uw.GradientBuffer(n, s.cloud.device)
        gen = torch.Generator(device="cuda").manual_seed(3)
        buf.flat[:14 * n] = torch.randn(14 * n, device="cuda", generator=gen) * 1e-3
        buf.flat[14 * n:15 * n] = torch.rand(n, device="cuda", generator=gen)
        buf.flat[15 * n:16 * n] = (torch.rand(n, device="cuda", generator=gen) > 0.3).float()
        buf.flat[16 * n:16 * n + 9] = torch.randn(9, device="cuda", generator=gen) * 1e-2
        for _ in range(2):   # second step: non-zero moments
            chunks = None
            if chunked:
                chunks = [(a, b, None) for a, b in range_chunks(s, buf, parts)]
            apply_gradients_device(s, buf, uw.OptimConfig(), 1.0, chunks=chunks)
            buf.flat[:14 * n] = torch.randn(14 * n, device="cuda", generator=gen) * 1e-3
            buf.flat[15 * n:16 * n] = 1.0
        results.append([np_(t).copy() for t in (s.cloud.flat, s.exp_avg, s.exp_avg_sq,
                                                s.grad_accum, s.obs_count, s.medium.flat,
                                                buf.flat[14 * n:])])
    for a, b in zip(*results):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("capacity", [None, 64])
def test_render_async_stream_matches_render(capacity):
    """A queued frame stream (render_async + render_flush) leaves the most recent
    frame in the output buffers, identical to a synchronous render -- also when the
    row lists overflow and are grown mid-stream."""
    g = load("survey2k")
    s, cam = _state(g)
    ref = uw.StepEngine(s, cam.width, cam.height, uw.OptimConfig())
    want = {k: np_(v).copy() for k, v in vars(ref.render(cam)).items()
            if isinstance(v, torch.Tensor) and k in ("color", "depth", "final_transmittance")}
    kw = {} if capacity is None else {"entry_capacity": capacity}
    eng = uw.StepEngine(s, cam.width, cam.height, uw.OptimConfig(), **kw)
    other = uw.Camera.look_at((0.5, -0.2, -1.0), (0, 0, 5), width=cam.width, height=cam.height,
                              fx=cam.fx, fy=cam.fy)
    for c in (other, cam, other, cam):
        eng.render_async(c)
    out = eng.render_flush()
    for k, v in want.items():
        np.testing.assert_array_equal(np_(getattr(out, k)), v)
    # an odd-length stream ends in the engine's own buffer set, an even one in the side
    # set; a training step after the stream sees the right buffers either way
    for c in (other, other, cam):
        eng.render_async(c)
    out = eng.render_flush()
    for k, v in want.items():
        np.testing.assert_array_equal(np_(getattr(out, k)), v)
    # a synchronous render after an even stream: flush then returns that render
    for c in (other, other):
        eng.render_async(c)
    eng.render_flush()
    eng.render(cam)
    out = eng.render_flush()
    for k, v in want.items():
        np.testing.assert_array_equal(np_(getattr(out, k)), v)
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    eng.render_async(other)
    st = eng.step([(cam, gt)])
    assert not st.skipped and np.isfinite(st.total)


def test_nonfinite_step_with_many_visible_gaussians_is_not_an_overflow():
    """A NaN ground truth at >= 65536 visible Gaussians: every visible Gaussian's
    gradient is non-finite, yet the step is a plain skip (no row-list re-runs):
    overflows are counted in their own slot."""
    from gpu_util import host_cloud, survey_camera, survey_medium
    hc = host_cloud(100_000, seed=1)
    cam = survey_camera(320, 240)
    med = survey_medium()
    cloud = uw.GaussianCloud(**vars(hc))
    m = uw.MediumParams(med.attenuation, med.water_color, med.backscatter,
                        med.water_color_guide, med.backscatter_guide)
    s = uw.TrainState(cloud, m, iteration=1)
    eng = uw.StepEngine(s, cam.width, cam.height, uw.OptimConfig())
    before = s.cloud.flat.clone()
    gt = torch.full((cam.height, cam.width, 3), float("nan"), device="cuda")
    st = eng.step([(cam, gt)])
    assert st.skipped and st.reruns == 0
    assert len(uw.project_cloud(cloud, cam)) >= 65536
    assert torch.equal(s.cloud.flat, before)
    assert all(slot.step == 0 for slot in s.adam.values())
    assert float(eng.grads.skip_counters.abs().sum()) == 0.0


def test_step_after_render_async_flushes_the_frame_stream():
    g = load("survey2k")
    s, cam = _state(g)
    eng = uw.StepEngine(s, cam.width, cam.height, uw.OptimConfig())
    eng.render_async(cam)
    with pytest.raises(RuntimeError):
        eng.refresh_guidance(g.gt)
    st = eng.step([(cam, torch.as_tensor(g.gt, dtype=torch.float32).cuda())])
    assert not st.skipped and eng._async_pending is None
