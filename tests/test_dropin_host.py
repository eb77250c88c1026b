"""The drop-in boundary on the host (no GPU): the DeviceArray numpy protocol the
reference's callers use, and dropin.install rebinding exactly the hot-path names
in the reference's own modules (and uninstall restoring them)."""

import os
import sys

import numpy as np
import pytest
import torch

from paper_2411_19588_b200 import dropin
from paper_2411_19588_b200.interop import DeviceArray, as_ref, plain

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIRS = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


def _reference():
    for d in REF_DIRS:
        if os.path.isdir(os.path.join(d, "uwsplat")):
            if d not in sys.path:
                sys.path.insert(0, d)
            import uwsplat
            import uwsplat.cli  # noqa: F401  (loads every module of the package)
            return uwsplat
    pytest.skip("reference package not installed")


def test_device_array_numpy_protocol():
    a = as_ref(torch.arange(6, dtype=torch.float32).reshape(2, 3))
    mask = a > 2
    # pipeline.py:191: boolean-mask indexing + astype stay tensors
    sel = a[mask].astype(np.float32)
    assert isinstance(sel, DeviceArray) and sel.dtype == torch.float32
    assert sel.tolist() == [3.0, 4.0, 5.0]
    # in-place masked update with a numpy mask and numpy scalar
    g = as_ref(torch.zeros(6))
    g[np.array([True, False, True, False, False, False])] += np.float32(2.5)
    assert g.tolist() == [2.5, 0, 2.5, 0, 0, 0]
    # numpy functions see a host copy (pipeline.py:259, dataset.py:90-91)
    c = np.clip(a, 0.0, 1.0)
    assert isinstance(c, np.ndarray) and c.max() == 1.0
    assert np.asarray(a, dtype=np.float64).dtype == np.float64
    assert isinstance(np.exp(a), np.ndarray)
    assert (np.round(a * 255.0).astype(np.uint8) == np.arange(6).reshape(2, 3) * 255 % 256).all()
    # host operand + device array (fixtures.py:64-67)
    s = a + np.ones((2, 3))
    assert np.allclose(np.asarray(s), np.arange(6).reshape(2, 3) + 1)
    # copy is a copy
    x = a.copy()
    x[0, 0] = 7.0
    assert float(a[0, 0]) == 0.0 and float(x[0, 0]) == 7.0
    assert type(plain(a)) is torch.Tensor


def test_install_rebinds_every_hot_path_name_and_uninstall_restores():
    R = _reference()
    import uwsplat.pipeline as P
    import uwsplat.dataset as D
    import uwsplat.cli as C
    orig = {"render": P.render, "backward_render": P.backward_render,
            "gc": D.GaussianCloud, "err": C.DataError}
    dropin.install(R)
    try:
        assert P.render is dropin.render and D.render is dropin.render
        assert P.backward_render is dropin.backward_render
        assert P.total_loss is dropin.total_loss
        assert P.apply_gradients is dropin.REPLACEMENTS["apply_gradients"]
        assert P.densify_and_prune is dropin.REPLACEMENTS["densify_and_prune"]
        assert P.estimate_backscatter is dropin.REPLACEMENTS["estimate_backscatter"]
        assert D.GaussianCloud is dropin.GaussianCloud and R.GaussianCloud is dropin.GaussianCloud
        assert R.rasterizer.render_naive is dropin.render_naive      # cli.py:209 imports lazily
        assert C.DataError is dropin.REPLACEMENTS["DataError"]       # one exception hierarchy
        # out-of-scope names stay the reference's
        assert D.apply_medium is R.medium.apply_medium and D.write_pfm.__module__ == "uwsplat.dataset"
        dropin.install(R)                                            # idempotent
    finally:
        dropin.uninstall()
    assert P.render is orig["render"] and P.backward_render is orig["backward_render"]
    assert D.GaussianCloud is orig["gc"] and C.DataError is orig["err"]


def test_every_reference_export_has_a_device_name():
    """The package exports each public name of the reference's hot-path modules
    ('same Python signatures')."""
    R = _reference()
    import paper_2411_19588_b200 as uw
    hot = ("GradientBuffer", "backward_medium", "backward_pixel", "backward_render",
           "finite_diff_check", "CheckpointError", "DataError", "NumericError", "LossBreakdown",
           "d_ssim_loss", "guidance_loss", "l1_loss", "psnr", "ssim_value", "total_loss",
           "logistic_remap", "OptimConfig", "adam_step", "densify_and_prune", "position_lr",
           "Projected2D", "project_cloud", "project_gaussian", "tile_span", "RenderOutput",
           "TileBins", "alpha_at", "bin_and_sort", "composite_pixel", "render", "render_naive",
           "Camera", "Gaussian", "GaussianCloud", "MediumParams", "TrainState", "covariance",
           "load_checkpoint", "opacity", "save_checkpoint", "BackscatterEstimate",
           "estimate_backscatter")
    for name in hot:
        assert hasattr(R, name), name          # the list is the reference's __init__
        assert hasattr(uw, name), name


def test_float64_loss_of_the_fd_harness_equals_the_oracle():
    """losses.loss_value_f64 (the finite-difference harness's objective) is the
    reference objective (losses.py:140-160) in float64: equal to the oracle."""
    from types import SimpleNamespace
    from oracle import uwsplat_oracle as O
    from paper_2411_19588_b200.losses import loss_value_f64
    rng = np.random.default_rng(0)
    a, b = rng.uniform(0, 1, (40, 37, 3)), rng.uniform(0, 1, (40, 37, 3))
    f32 = lambda v: torch.tensor(v, dtype=torch.float32)  # noqa: E731
    med = SimpleNamespace(flat=torch.zeros(15), has_guidance=True,
                          attenuation=f32([0.5, 0.4, 0.3]), water_color=f32([0.25, 0.35, 0.45]),
                          backscatter=f32([0.9, 1.1, 1.3]), water_color_guide=f32([0.3, 0.3, 0.4]),
                          backscatter_guide=f32([1.0, 1.0, 1.0]))
    ref_med = SimpleNamespace(**{k: np.asarray(getattr(med, k)) for k in (
        "attenuation", "water_color", "backscatter", "water_color_guide", "backscatter_guide")})
    ref = O.total_loss(a, b, ref_med, 0.3, 0.1)
    total = ref[0]["total"]
    assert abs(loss_value_f64(a, b, med, 0.3, 0.1) - total) <= 1e-12
