"""Training objective on the device (reference: losses.py).

``total_loss`` runs the fused L1 + D-SSIM kernel pair and returns the
reference's ``(LossBreakdown, dL_dC)``.  The breakdown holds Python floats
(one 48-byte device-to-host read); ``total_loss_device`` keeps them on the
device for the training step.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from .errors import DataError
from .scene import MediumParams, default_device

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2


@dataclass
class LossBreakdown:
    l1: float
    d_ssim: float
    l_bs: float
    total: float
    lambda_ssim: float
    lambda_guide: float
    guidance_present: bool


def _image(x, dev) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.device != dev or t.dtype != torch.float32:
            t = t.to(device=dev, dtype=torch.float32)
    else:
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float32)), device=dev)
    return t.contiguous()


def _prep(a, b):
    dev = a.device if isinstance(a, torch.Tensor) and a.is_cuda else default_device()
    a, b = _image(a, dev), _image(b, dev)
    if a.shape != b.shape:
        raise DataError(f"shape mismatch {tuple(a.shape)} vs {tuple(b.shape)}")
    if a.dim() not in (2, 3):
        raise DataError(f"expected (H, W[, C]) images, got {tuple(a.shape)}")
    return a, b


def total_loss_device(rendered, gt, medium: Optional[MediumParams], lambda_ssim: float = 0.3,
                      lambda_guide: float = 0.1, result=None, grad=None, workspace=None,
                      nonfinite=None):
    """Kernel call; returns (result double[6] on device, dL_dC).  Optional
    preallocated ``result``/``grad``/``workspace`` and a device ``nonfinite``
    counter (incremented when the total is not finite) serve the engine."""
    a, b = _prep(rendered, gt)
    h, w = a.shape[0], a.shape[1]
    c = a.shape[2] if a.dim() == 3 else 1
    if h < SSIM_WINDOW or w < SSIM_WINDOW:
        raise DataError(f"image {(h, w)} smaller than the {SSIM_WINDOW}x{SSIM_WINDOW} window")
    grad = torch.empty_like(a) if grad is None else grad
    res = torch.empty(6, dtype=torch.float64, device=a.device) if result is None else result
    if workspace is None:
        nb = _lib.size_out()
        _lib.call("uws_loss_workspace_size", h, w, c, ctypes.byref(nb))
        workspace = torch.empty(nb.value, dtype=torch.uint8, device=a.device)
    med = _lib.ptr(medium.flat) if medium is not None else 0
    guided = 1 if (medium is not None and medium.has_guidance) else 0
    _lib.call("uws_loss_fwd_bwd", _lib.ptr(a), _lib.ptr(b), h, w, c, med, guided,
              float(lambda_ssim), float(lambda_guide), _lib.ptr(grad), _lib.ptr(res),
              _lib.ptr(nonfinite), _lib.ptr(workspace), workspace.numel(), _lib.stream_handle())
    return res, grad


def total_loss(rendered, gt, medium: Optional[MediumParams], lambda_ssim: float = 0.3,
               lambda_guide: float = 0.1) -> Tuple[LossBreakdown, torch.Tensor]:
    """Weighted objective and dL/d(rendered) (losses.py:140-160)."""
    res, grad = total_loss_device(rendered, gt, medium, lambda_ssim, lambda_guide)
    v = res.tolist()
    present = bool(medium is not None and medium.has_guidance)
    return LossBreakdown(l1=v[0], d_ssim=v[1], l_bs=v[2], total=v[3], lambda_ssim=lambda_ssim,
                         lambda_guide=lambda_guide, guidance_present=present), grad


def l1_loss(a, b) -> Tuple[float, torch.Tensor]:
    """Mean |a-b| and sign(a-b)/size (losses.py:40-49)."""
    a, b = _prep(a, b)
    if a.shape[0] < SSIM_WINDOW or a.shape[1] < SSIM_WINDOW:
        d = (a.double() - b.double())
        return float(d.abs().mean()), torch.sign(d) / d.numel()
    res, grad = total_loss_device(a, b, None, 0.0, 0.0)
    return float(res[0].item()), grad


def d_ssim_loss(a, b) -> Tuple[float, torch.Tensor]:
    """1 - mean SSIM and its gradient (losses.py:83-123)."""
    res, grad = total_loss_device(a, b, None, 1.0, 0.0)
    return float(res[1].item()), grad


def ssim_value(a, b) -> float:
    v, _ = d_ssim_loss(a, b)
    return 1.0 - v


def guidance_loss(m: MediumParams):
    """l1 distance of (water_color, backscatter) from their anchors (losses.py:126-137)."""
    if not m.has_guidance:
        return 0.0, np.zeros(3), np.zeros(3)
    dw = (m.water_color.double() - m.water_color_guide.double()).cpu().numpy()
    db = (m.backscatter.double() - m.backscatter_guide.double()).cpu().numpy()
    return float(np.abs(dw).sum() + np.abs(db).sum()), np.sign(dw), np.sign(db)


def psnr(a, b, cap: float = 99.0) -> float:
    a = a.double() if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, np.float64))
    b = b.double() if isinstance(b, torch.Tensor) else torch.as_tensor(np.asarray(b, np.float64))
    mse = float(((a - b.to(a.device)) ** 2).mean())
    if mse <= 10 ** (-cap / 10.0):
        return cap
    return float(-10.0 * np.log10(mse))


def loss_value_f64(rendered, gt, medium: Optional[MediumParams], lambda_ssim: float = 0.3,
                   lambda_guide: float = 0.1) -> float:
    """The objective of total_loss (losses.py:140-160) evaluated in float64 with
    torch ops on the device -- no gradient, for the finite-difference harness,
    whose difference quotients need the loss far below the float32 kernel's
    rounding (its per-tile partial sums are float32)."""
    dev = medium.flat.device if medium is not None else default_device()
    a = torch.as_tensor(rendered if isinstance(rendered, torch.Tensor) else np.asarray(rendered))
    b = torch.as_tensor(gt if isinstance(gt, torch.Tensor) else np.asarray(gt))
    a = a.to(device=dev, dtype=torch.float64)
    b = b.to(device=dev, dtype=torch.float64)
    if a.shape != b.shape:
        raise DataError(f"shape mismatch {tuple(a.shape)} vs {tuple(b.shape)}")
    l1 = float((a - b).abs().mean())
    x = torch.arange(SSIM_WINDOW, dtype=torch.float64, device=dev) - (SSIM_WINDOW - 1) / 2
    k = torch.exp(-x * x / (2 * SSIM_SIGMA ** 2))
    k = k / k.sum()
    img = torch.stack([a, b]).permute(0, 3, 1, 2) if a.dim() == 3 else torch.stack([a, b])[:, None]
    c = img.shape[1]

    def filt(t):  # valid separable 11x11 Gaussian filter per channel
        t = torch.nn.functional.conv2d(t, k.view(1, 1, 1, -1).expand(c, 1, 1, -1), groups=c)
        return torch.nn.functional.conv2d(t, k.view(1, 1, -1, 1).expand(c, 1, -1, 1), groups=c)

    pa, pb = img[0:1], img[1:2]
    mu_a, mu_b = filt(pa), filt(pb)
    saa = filt(pa * pa) - mu_a * mu_a
    sbb = filt(pb * pb) - mu_b * mu_b
    sab = filt(pa * pb) - mu_a * mu_b
    ssim = ((2 * mu_a * mu_b + SSIM_C1) * (2 * sab + SSIM_C2)) / \
        ((mu_a * mu_a + mu_b * mu_b + SSIM_C1) * (saa + sbb + SSIM_C2))
    d_ssim = 1.0 - float(ssim.mean())
    lb = 0.0
    if medium is not None and medium.has_guidance:
        lb = float((medium.water_color.double() - medium.water_color_guide.double()).abs().sum()
                   + (medium.backscatter.double() - medium.backscatter_guide.double()).abs().sum())
    return (1.0 - lambda_ssim) * l1 + lambda_ssim * d_ssim + lambda_guide * lb
