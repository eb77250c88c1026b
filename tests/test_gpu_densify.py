"""Densification on the device against the reference (tests/golden/densify.npz,
written by the reference's densify_and_prune with the same generator seed)."""

import os

import numpy as np
import pytest
import torch

import paper_2411_19588_b200 as uw
from golden_util import load
from gpu_util import device_scene, np_

pytestmark = pytest.mark.gpu

F5 = ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits")


def _golden_state():
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "densify.npz"))
    cloud = uw.GaussianCloud(**{f: d["in_" + f] for f in F5})
    medium = uw.MediumParams((0.6, 0.45, 0.3), (0.2, 0.35, 0.5), (0.8, 1.0, 1.2))
    st = uw.TrainState(cloud, medium, iteration=1500)
    for f in F5:
        st.adam[f].m.copy_(torch.as_tensor(d["in_m_" + f]).reshape(st.adam[f].m.shape))
        st.adam[f].v.copy_(torch.as_tensor(d["in_v_" + f]).reshape(st.adam[f].v.shape))
        st.adam[f].step = 1500
    st.grad_accum.copy_(torch.as_tensor(d["in_grad_accum"]))
    st.obs_count.copy_(torch.as_tensor(d["in_obs_count"].astype(np.int32)))
    return d, st


def test_densify_matches_reference():
    d, st = _golden_state()
    gen = st.cloud.generation
    counts = uw.densify_and_prune(st, uw.OptimConfig(), float(d["extent"]),
                                  np.random.default_rng(int(d["seed"])))
    assert counts == tuple(int(c) for c in d["counts"])
    assert st.cloud.generation == gen + 1
    n_new = d["out_positions"].shape[0]
    assert len(st.cloud) == n_new
    for f in F5:
        np.testing.assert_array_equal(np_(getattr(st.cloud, f)), d["out_" + f], err_msg=f)
        np.testing.assert_array_equal(np_(st.adam[f].m), d["out_m_" + f], err_msg=f)
        np.testing.assert_array_equal(np_(st.adam[f].v), d["out_v_" + f], err_msg=f)
        assert st.adam[f].step == 1500
    assert int(st.obs_count.abs().sum()) == 0 and float(st.grad_accum.abs().sum()) == 0.0
    assert st.grad_accum.numel() == n_new


def test_densify_refuses_to_empty_and_reset_opacities():
    d, st = _golden_state()
    st.cloud.opacity_logits.fill_(-10.0)            # everything transparent -> all pruned
    before = st.cloud.flat.clone()
    assert uw.densify_and_prune(st, uw.OptimConfig(), 10.0, np.random.default_rng(0)) == (0, 0, 0)
    assert torch.equal(st.cloud.flat, before)
    cfg = uw.OptimConfig()
    uw.reset_opacities(st, cfg)
    target = np.float32(np.log(cfg.opacity_reset_value / (1 - cfg.opacity_reset_value)))
    assert bool((st.cloud.opacity_logits == float(target)).all())
    assert float(st.adam["opacity_logits"].m.abs().sum()) == 0.0
    assert float(st.adam["opacity_logits"].v.abs().sum()) == 0.0


def test_engine_follows_densification():
    """Train, densify on the device, keep training with the same engine."""
    g = load("survey2k")
    cloud, cam, medium = device_scene(g)
    st = uw.TrainState(cloud, medium, iteration=1)
    eng = uw.StepEngine(st, cam.width, cam.height, uw.OptimConfig())
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    for _ in range(3):
        eng.step_async([(cam, gt)])
        st.iteration += 1
    eng.flush()
    cfg = uw.OptimConfig(densify_grad_threshold=1e-9)
    n0 = len(st.cloud)
    c, s, p = uw.densify_and_prune(st, cfg, 1.0, np.random.default_rng(1))
    assert c + s > 0 and len(st.cloud) == n0 + c + s - p
    r = eng.step([(cam, gt)])
    assert not r.skipped and np.isfinite(r.total)
    assert eng.n == len(st.cloud) and eng.grads.n == len(st.cloud)
    with pytest.raises(RuntimeError, match="flush"):
        eng.step_async([(cam, gt)])
        uw.densify_and_prune(st, cfg, 1.0, np.random.default_rng(2))
        eng.step_async([(cam, gt)])
    eng._pending = None
