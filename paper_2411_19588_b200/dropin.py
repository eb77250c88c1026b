"""Run the reference's own callers on this package (SURVEY 8b "callers of the path").

The hot path of the reference package ``uwsplat`` -- projection, binning,
compositing, loss, backward, Adam, densification, the guidance refresh and
the checkpoint codec -- lives in its modules ``scene``, ``projection``,
``rasterizer``, ``losses``, ``backward``, ``optim``, ``medium``,
``backscatter`` and ``errors``; its callers (``pipeline.train`` /
``evaluate`` / ``render_novel``, ``dataset.generate_synthetic``,
``fixtures.gradient_check_scene``, ``cli``) reach it through names they
import from those modules (reference pipeline.py:21-31, dataset.py:23-26,
fixtures.py:9, 50, cli.py:24-34, 209).  :func:`install` rebinds exactly those
names, in every loaded ``uwsplat`` module, to this package's device
implementations, so the callers run UNCHANGED on the GPU::

    import uwsplat
    from paper_2411_19588_b200 import dropin
    dropin.install(uwsplat)
    uwsplat.pipeline.train(dataset, uwsplat.OptimConfig(iterations=2000))

Objects handed back to the callers carry their arrays as
:class:`~paper_2411_19588_b200.interop.DeviceArray` views (device tensors with
the numpy protocol the callers use: ``.astype``, boolean-mask indexing,
numpy functions by explicit device-to-host copy).  Names the package does not
implement (dataset I/O, ``apply_medium`` / ``invert_medium``, the backscatter
curve-fit helpers, the CLI) stay the reference's: they are outside the hot
path.  :func:`uninstall` restores the reference's bindings.
"""

from __future__ import annotations

import sys
from typing import Optional

import numpy as np
import torch

from . import backscatter as _bs
from . import backward as _bw
from . import checkpoint as _ck
from . import errors as _er
from . import losses as _ls
from . import medium as _md
from . import optim as _op
from . import projection as _pj
from . import rasterizer as _rs
from . import scene as _sc
from .interop import DeviceArray, as_ref, plain

# ----------------------------------------------------------------------------
# reference-shaped containers: the package's device types whose array fields
# read as DeviceArray views
# ----------------------------------------------------------------------------


class GaussianCloud(_sc.GaussianCloud):
    """Device cloud whose field arrays are DeviceArray views (scene.py:90-147)."""

    def __getattr__(self, name):
        return as_ref(super().__getattr__(name))


class MediumParams(_sc.MediumParams):
    """Device medium whose triplets are DeviceArray views (scene.py:150-187)."""

    attenuation = property(lambda s: as_ref(_sc.MediumParams.attenuation.fget(s)),
                           _sc.MediumParams.attenuation.fset)
    water_color = property(lambda s: as_ref(_sc.MediumParams.water_color.fget(s)),
                           _sc.MediumParams.water_color.fset)
    backscatter = property(lambda s: as_ref(_sc.MediumParams.backscatter.fget(s)),
                           _sc.MediumParams.backscatter.fset)
    water_color_guide = property(lambda s: as_ref(_sc.MediumParams.water_color_guide.fget(s)),
                                 _sc.MediumParams.water_color_guide.fset)
    backscatter_guide = property(lambda s: as_ref(_sc.MediumParams.backscatter_guide.fget(s)),
                                 _sc.MediumParams.backscatter_guide.fset)

    @staticmethod
    def zero(device=None) -> "MediumParams":
        return MediumParams(np.zeros(3), np.zeros(3), np.zeros(3), device=device)


def _stat_property(key):
    return property(lambda s: as_ref(s.__dict__[key]),
                    lambda s, v: s.__dict__.__setitem__(key, plain(torch.as_tensor(v))))


class TrainState(_sc.TrainState):
    """Device training state; ``grad_accum`` / ``obs_count`` read as DeviceArrays
    (scene.py:262-281; pipeline.py:191-192 updates them in place)."""

    grad_accum = _stat_property("_grad_accum")
    obs_count = _stat_property("_obs_count")

    def __init__(self, cloud, medium, iteration: int = 0):
        super().__init__(_adopt_cloud(cloud), _adopt_medium(medium), iteration)


class GradientBuffer(_bw.GradientBuffer):
    """Device gradient buffer with DeviceArray fields (backward.py:46-69)."""

    def __init__(self, n: int, device=None):
        super().__init__(n, device)
        for name in ("d_positions", "d_log_scales", "d_rotations", "d_sh_coeffs",
                     "d_opacity_logits", "mean2d_grad_norm", "observed_count", "d_attenuation",
                     "d_water_color", "d_backscatter"):
            setattr(self, name, as_ref(getattr(self, name)))

    @property
    def observed(self) -> DeviceArray:
        return as_ref(plain(self.observed_count) > 0)


def _adopt_cloud(c):
    if c is None or isinstance(c, GaussianCloud):
        return c
    if isinstance(c, _sc.GaussianCloud):
        c.__class__ = GaussianCloud
        return c
    return GaussianCloud(c.positions, c.log_scales, c.rotations, c.sh_coeffs, c.opacity_logits)


def _adopt_medium(m):
    if m is None or isinstance(m, MediumParams):
        return m
    if isinstance(m, _sc.MediumParams):
        m.__class__ = MediumParams
        return m
    return MediumParams(m.attenuation, m.water_color, m.backscatter,
                        getattr(m, "water_color_guide", None), getattr(m, "backscatter_guide", None))


def _adopt_state(s):
    if isinstance(s, TrainState):
        return s
    ga, oc = s.__dict__.pop("grad_accum"), s.__dict__.pop("obs_count")
    s.__class__ = TrainState
    s.grad_accum, s.obs_count = ga, oc
    _adopt_cloud(s.cloud)
    _adopt_medium(s.medium)
    return s


def _ref_output(out: _rs.RenderOutput) -> _rs.RenderOutput:
    for f in ("color", "depth", "weight", "final_transmittance", "count", "color_clean",
              "attenuation_map", "backscatter_map"):
        setattr(out, f, as_ref(getattr(out, f)))
    return out


# ----------------------------------------------------------------------------
# the reference's function names
# ----------------------------------------------------------------------------
def render(cloud, cam, medium=None, mode: str = "clean", workers: int = 1, retain: bool = True):
    return _ref_output(_rs.render(_adopt_cloud(cloud), cam, _adopt_medium(medium), mode, workers,
                                  retain))


def render_naive(cloud, cam, medium=None, mode: str = "clean", row_chunk: int = 16):
    return _ref_output(_rs.render_naive(_adopt_cloud(cloud), cam, _adopt_medium(medium), mode,
                                        row_chunk))


def backward_render(out, dL_dC, cloud, medium=None, lambda_guide: float = 0.0,
                    workers: int = 1) -> GradientBuffer:
    buf = GradientBuffer(len(cloud), cloud.device)
    _bw.backward_render(out, plain(dL_dC) if isinstance(dL_dC, torch.Tensor) else dL_dC, cloud,
                        medium, lambda_guide, workers, buf=buf)
    return buf


def backward_medium(out, dL_dC, medium, lambda_guide: float):
    return tuple(as_ref(t) for t in _bw.backward_medium(out, dL_dC, medium, lambda_guide))


def total_loss(rendered, gt, medium, lambda_ssim: float = 0.3, lambda_guide: float = 0.1):
    bd, grad = _ls.total_loss(rendered, gt, medium, lambda_ssim, lambda_guide)
    return bd, as_ref(grad)


def l1_loss(a, b):
    v, g = _ls.l1_loss(a, b)
    return v, as_ref(g)


def d_ssim_loss(a, b):
    v, g = _ls.d_ssim_loss(a, b)
    return v, as_ref(g)


def logistic_remap(depth_raw):
    r = _md.logistic_remap(depth_raw)
    return as_ref(r) if isinstance(r, torch.Tensor) else r


def apply_water(color_clean, depth, medium):
    return as_ref(_rs.apply_water(color_clean, depth, medium))


def load_checkpoint(data: bytes, device=None) -> TrainState:
    return _adopt_state(_ck.load_checkpoint(data, device))


def finite_diff_check(cloud, cam, medium, gt, lambda_ssim: float = 0.3,
                      lambda_guide: float = 0.1, eps: Optional[dict] = None, tol: float = 1e-3,
                      analytic=None):
    return _bw.finite_diff_check(_adopt_cloud(cloud), cam, _adopt_medium(medium), gt,
                                 lambda_ssim, lambda_guide, eps, tol, analytic)


def frozen_depth_loss(cloud, cam, medium, gt, depth_frozen, lambda_ssim, lambda_guide):
    return _bw.frozen_depth_loss(_adopt_cloud(cloud), cam, _adopt_medium(medium), gt,
                                 depth_frozen, lambda_ssim, lambda_guide)


# name -> implementation, for every name the reference's modules bind
REPLACEMENTS = {
    # scene.py
    "GaussianCloud": GaussianCloud, "MediumParams": MediumParams, "TrainState": TrainState,
    "AdamSlot": _sc.AdamSlot, "Gaussian": _sc.Gaussian, "covariance": _sc.covariance,
    "opacity": _sc.opacity, "save_checkpoint": _ck.save_checkpoint,
    "load_checkpoint": load_checkpoint,
    # projection.py
    "project_cloud": _pj.project_cloud, "project_gaussian": _pj.project_gaussian,
    "tile_span": _pj.tile_span, "ProjectedCloud": _pj.ProjectedCloud,
    "Projected2D": _pj.Projected2D,
    # rasterizer.py
    "render": render, "render_naive": render_naive, "bin_and_sort": _rs.bin_and_sort,
    "alpha_at": _rs.alpha_at, "composite_pixel": _rs.composite_pixel,
    "apply_water": apply_water, "RenderOutput": _rs.RenderOutput, "TileBins": _rs.TileBins,
    # backward.py
    "backward_render": backward_render, "backward_medium": backward_medium,
    "backward_pixel": _bw.backward_pixel, "finite_diff_check": finite_diff_check,
    "frozen_depth_loss": frozen_depth_loss, "GradientBuffer": GradientBuffer,
    "GradCheckRow": _bw.GradCheckRow, "GradCheckReport": _bw.GradCheckReport,
    # losses.py
    "total_loss": total_loss, "l1_loss": l1_loss, "d_ssim_loss": d_ssim_loss,
    "guidance_loss": _ls.guidance_loss, "psnr": _ls.psnr, "ssim_value": _ls.ssim_value,
    "LossBreakdown": _ls.LossBreakdown,
    # medium.py
    "logistic_remap": logistic_remap,
    # optim.py
    "apply_gradients": _op.apply_gradients, "adam_step": _op.adam_step,
    "densify_and_prune": _op.densify_and_prune, "reset_opacities": _op.reset_opacities,
    "position_lr": _op.position_lr,
    # backscatter.py
    "estimate_backscatter": _bs.estimate_backscatter,
    "BackscatterEstimate": _bs.BackscatterEstimate,
    # errors.py: one set of exception classes on both sides of the boundary
    "DataError": _er.DataError, "CheckpointError": _er.CheckpointError,
    "NumericError": _er.NumericError,
}

_saved: dict = {}


def install(pkg=None):
    """Rebind the hot-path names in every loaded module of the reference package
    ``pkg`` (default: ``import uwsplat``).  Idempotent; returns ``pkg``."""
    if pkg is None:
        import uwsplat as pkg  # noqa: F811
    root = pkg.__name__
    for name, mod in list(sys.modules.items()):
        if mod is None or not (name == root or name.startswith(root + ".")):
            continue
        for attr, impl in REPLACEMENTS.items():
            if attr in vars(mod):
                _saved.setdefault((name, attr), vars(mod)[attr])
                setattr(mod, attr, impl)
    return pkg


def uninstall():
    """Restore every binding :func:`install` replaced."""
    for (name, attr), orig in _saved.items():
        mod = sys.modules.get(name)
        if mod is not None:
            setattr(mod, attr, orig)
    _saved.clear()
