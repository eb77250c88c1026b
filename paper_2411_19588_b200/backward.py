"""Analytic gradients on the device (reference: backward.py).

``backward_render`` runs the back-to-front compositing backward kernel
(screen-space gradients + medium sums) and the projection backward kernel
(chain to positions / log-scales / quaternions / SH / opacity logits) into a
:class:`GradientBuffer`.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _lib
from .medium import logistic_remap
from .rasterizer import RenderOutput
from .scene import GaussianCloud, MediumParams, flat_views

GRAD_FLOATS_PER_GAUSSIAN = 16   # 14 params + mean2d_grad_norm + observed
MEDIUM_SLOTS = 16               # 9 medium gradients, non-finite + overflow counters, pad


class GradientBuffer:
    """Gradients co-indexed with a cloud generation (backward.py:46-69).

    One flat float32 device buffer ``[d_params 14n | mean2d_grad_norm n |
    observed n | medium 9 | non-finite count | overflow count | pad]`` so
    multi-view accumulation and the NCCL all-reduce are a single contiguous
    array (the two device skip counters included).  ``observed`` counts the views
    that saw each Gaussian (the reference's boolean is ``observed > 0``).
    """

    def __init__(self, n: int, device=None):
        device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n = n
        self.flat = torch.zeros(GRAD_FLOATS_PER_GAUSSIAN * n + MEDIUM_SLOTS, dtype=torch.float32,
                                device=device)
        v = flat_views(self.flat, n)
        self.d_positions = v["positions"]
        self.d_log_scales = v["log_scales"]
        self.d_rotations = v["rotations"]
        self.d_sh_coeffs = v["sh_coeffs"]
        self.d_opacity_logits = v["opacity_logits"]
        self.mean2d_grad_norm = self.flat[14 * n:15 * n]
        self.observed_count = self.flat[15 * n:16 * n]
        self.medium = self.flat[16 * n:16 * n + 9]
        self.d_attenuation = self.flat[16 * n:16 * n + 3]
        self.d_water_color = self.flat[16 * n + 3:16 * n + 6]
        self.d_backscatter = self.flat[16 * n + 6:16 * n + 9]
        # device skip counters {non-finite values, row-list overflows}; kernels
        # that count non-finite values get a pointer to slot 9, the binning
        # guard and Adam read both slots
        self.skip_counters = self.flat[16 * n + 9:16 * n + 11]
        self.nonfinite = self.flat[16 * n + 9:16 * n + 10]
        self.overflow = self.flat[16 * n + 10:16 * n + 11]
        self.generation = -1

    @property
    def params(self) -> torch.Tensor:
        return self.flat[:14 * self.n]

    @property
    def observed(self) -> torch.Tensor:
        return self.observed_count > 0

    def zero_(self):
        self.flat.zero_()
        return self

    def all_finite_device(self) -> torch.Tensor:
        n = self.n
        return torch.isfinite(self.flat[:14 * n]).all() & torch.isfinite(self.medium).all()

    def all_finite(self) -> bool:
        return bool(self.all_finite_device().item())


def backward_medium(out: RenderOutput, dL_dC, medium: MediumParams, lambda_guide: float):
    """Medium-parameter gradients (backward.py:261-275).

    float64 torch utility; on the hot path the backward kernel fuses these sums.
    """
    dL = dL_dC.double()
    z = logistic_remap(out.depth)[..., None]
    att = torch.exp(-medium.attenuation.double() * z)
    ebs = torch.exp(-medium.backscatter.double() * z)
    d_att = (dL * out.color_clean.double() * (-z) * att).sum(dim=(0, 1))
    d_water = (dL * (1.0 - ebs)).sum(dim=(0, 1))
    d_bsc = (dL * medium.water_color.double() * z * ebs).sum(dim=(0, 1))
    if medium.has_guidance and lambda_guide != 0.0:
        d_water = d_water + lambda_guide * torch.sign(medium.water_color.double()
                                                      - medium.water_color_guide.double())
        d_bsc = d_bsc + lambda_guide * torch.sign(medium.backscatter.double()
                                                  - medium.backscatter_guide.double())
    return d_att, d_water, d_bsc


def backward_render(out: RenderOutput, dL_dC, cloud: GaussianCloud,
                    medium: Optional[MediumParams] = None, lambda_guide: float = 0.0,
                    workers: int = 1, buf: Optional[GradientBuffer] = None) -> GradientBuffer:
    """Accumulate all parameter gradients for one rendered view (backward.py:278-344).

    ``buf`` (optional) is accumulated into instead of a fresh buffer, which is
    how several views are summed before one optimizer step.
    """
    rows = getattr(out, "rows", None)
    if out.proj is None or (out.bins is None and rows is None):
        raise ValueError("render output was produced without retained buffers")
    proj, bins, cam = out.proj, out.bins, out.camera
    if buf is None:
        buf = GradientBuffer(len(cloud), cloud.device)
    buf.generation = cloud.generation
    underwater = out.mode == "underwater"
    if underwater and medium is None:
        raise ValueError("underwater backward requires medium parameters")
    dev = cloud.device
    dL = dL_dC if isinstance(dL_dC, torch.Tensor) else torch.as_tensor(dL_dC)
    dL = dL.to(device=dev, dtype=torch.float32).contiguous()
    k_cap = proj.n_source
    screen = torch.zeros(max(k_cap, 1), 9, dtype=torch.float32, device=dev)
    med_acc = torch.zeros(9, dtype=torch.float64, device=dev) if underwater else None
    st = _lib.stream_handle()
    pc, cc, oc = proj.c_struct(), cam.c_struct(), out.c_struct()
    med = _lib.ptr(medium.flat) if underwater else 0
    if rows is not None:   # the forward composited from row lists: filter them again
        _lib.call("uws_raster_bwd_rows", ctypes.byref(pc), _lib.ptr(rows.row_start),
                  _lib.ptr(rows.items), ctypes.byref(cc), med, ctypes.byref(oc), _lib.ptr(dL),
                  _lib.ptr(screen), _lib.ptr(med_acc), st)
    else:
        _lib.call("uws_raster_bwd", ctypes.byref(pc), _lib.ptr(bins.offsets),
                  _lib.ptr(bins.entries), ctypes.byref(cc), med, ctypes.byref(oc), _lib.ptr(dL),
                  _lib.ptr(screen), _lib.ptr(med_acc), st)
    cl = cloud.c_struct()
    guided = 1 if (medium is not None and medium.has_guidance) else 0
    _lib.call("uws_preprocess_bwd", ctypes.byref(cl), ctypes.byref(cc), ctypes.byref(pc), k_cap,
              _lib.ptr(screen), _lib.ptr(med_acc), med, guided, float(lambda_guide),
              _lib.ptr(buf.flat), 0, 1, st)
    return buf
