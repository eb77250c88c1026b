"""Guidance refresh: the dark-pixel backscatter estimate on the device
(reference: backscatter.py, called by pipeline.py:204-208).

``estimate_backscatter`` keeps the reference signature and result type; the
whole estimate (resize, depth clustering, per-cluster dark-pixel selection,
per-interval minima, multi-start Levenberg-Marquardt fits) runs in the
``uws_estimate_backscatter`` kernels and one 96-byte result record comes back.
``refresh_guidance`` is the training loop's call: the estimate from the
current view's ground truth and the raw render depth (remapped inside the
kernel, as pipeline.py:205 remaps before calling) written straight into the
medium's guidance slots on the device when it is not degenerate.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import DataError
from .scene import MediumParams, default_device

WATER_COLOR_BOX = (0.0, 1.0)       # backscatter.py:21
BACKSCATTER_BOX = (0.0, 5.0)       # backscatter.py:22
P_DARK_DEFAULT = 0.01              # backscatter.py:24-27
EDGES_NUM_DEFAULT = 10
INTERVALS_NUM_DEFAULT = 25
RESIZED_HEIGHT_DEFAULT = 300
RESULT_SLOTS = 12


@dataclass
class BackscatterEstimate:
    """backscatter.py:42-47 (float64 numpy arrays, as the reference returns)."""

    water_color_est: np.ndarray
    backscatter_est: np.ndarray
    residual: np.ndarray
    degenerate: bool = False
    n_dark: int = 0


class _Workspace:
    """Per-device workspace cache (the refit runs every few hundred steps)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, dev) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != dev:
            self.buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        return self.buf


_WS = _Workspace()


def _cfg(p_dark, intervals_num, resized_height, edges_num) -> _lib.BackscatterCfgC:
    for name, v in (("intervals_num", intervals_num), ("edges_num", edges_num)):
        if not 0 <= int(v) <= 257:
            raise ValueError(f"{name} must be in [0, 257] on the device path")
    if int(resized_height) < 1:
        raise ValueError("resized_height must be >= 1")
    return _lib.BackscatterCfgC(float(p_dark), int(intervals_num), int(resized_height),
                                int(edges_num), 0)


def _as_image(image, dev) -> torch.Tensor:
    t = image if isinstance(image, torch.Tensor) else torch.as_tensor(np.asarray(image))
    if t.ndim != 3 or t.shape[2] != 3:
        raise DataError(f"expected (H, W, 3) image, got {tuple(t.shape)}")
    if t.shape[0] == 0 or t.shape[1] == 0:
        raise DataError("empty image")
    return t.to(device=dev, dtype=torch.float32).contiguous()


def _launch(img: torch.Tensor, depth: torch.Tensor, raw: bool, cfg, result: torch.Tensor,
            guide: Optional[torch.Tensor], dark: Optional[torch.Tensor]):
    h, w = int(img.shape[0]), int(img.shape[1])
    nb = _lib.size_out()
    _lib.call("uws_backscatter_workspace_size", h, w, ctypes.byref(cfg), ctypes.byref(nb))
    ws = _WS.get(nb.value, img.device)
    _lib.call("uws_estimate_backscatter", _lib.ptr(img), _lib.ptr(depth), 1 if raw else 0, h, w,
              ctypes.byref(cfg), _lib.ptr(result), _lib.ptr(guide), _lib.ptr(dark),
              _lib.ptr(ws), ws.numel(), _lib.stream_handle())


def _estimate(res: np.ndarray) -> BackscatterEstimate:
    if res[11] != 0.0:
        raise DataError("cluster edges must be strictly increasing")
    return BackscatterEstimate(water_color_est=res[0:3].copy(), backscatter_est=res[3:6].copy(),
                               residual=res[6:9].copy(), degenerate=bool(res[9] != 0.0),
                               n_dark=int(res[10]))


def estimate_backscatter(image, depth, p_dark: float = P_DARK_DEFAULT,
                         intervals_num: int = INTERVALS_NUM_DEFAULT,
                         resized_height: int = RESIZED_HEIGHT_DEFAULT,
                         edges_num: int = EDGES_NUM_DEFAULT, *, depth_is_raw: bool = False,
                         return_dark: bool = False):
    """estimate_backscatter (backscatter.py:211-270) on the device.

    ``image`` (H, W, 3) and ``depth`` (H, W): numpy arrays or tensors.  ``depth``
    is the remapped depth (float64, the reference's argument) unless
    ``depth_is_raw`` -- then it is a raw render depth and logistic_remap
    (medium.py:26-29) is applied inside the kernel.  With ``return_dark`` the
    dark-pixel set is returned too, as (z, rgb) float64 device tensors.
    """
    dev = image.device if isinstance(image, torch.Tensor) and image.is_cuda else default_device()
    img = _as_image(image, dev)
    d = depth if isinstance(depth, torch.Tensor) else torch.as_tensor(np.asarray(depth))
    if tuple(d.shape) != tuple(img.shape[:2]):
        raise DataError("image and depth are not co-registered")
    d = d.to(device=dev, dtype=torch.float32 if depth_is_raw else torch.float64).contiguous()
    cfg = _cfg(p_dark, intervals_num, resized_height, edges_num)
    result = torch.empty(RESULT_SLOTS, dtype=torch.float64, device=dev)
    dark = None
    if return_dark:
        h, w = img.shape[:2]
        th = min(int(resized_height), h)
        tw = w if th == h else max(1, round(w * th / h))
        dark = torch.empty(th * tw, 4, dtype=torch.float64, device=dev)
    _launch(img, d, depth_is_raw, cfg, result, None, dark)
    est = _estimate(result.cpu().numpy())
    if return_dark:
        rows = dark[:est.n_dark]
        return est, rows[:, 0], rows[:, 1:]
    return est


def refresh_guidance(medium: MediumParams, gt, depth_raw: torch.Tensor,
                     p_dark: float = P_DARK_DEFAULT, intervals_num: int = INTERVALS_NUM_DEFAULT,
                     resized_height: int = RESIZED_HEIGHT_DEFAULT,
                     edges_num: int = EDGES_NUM_DEFAULT) -> BackscatterEstimate:
    """pipeline.py:204-208: estimate from (gt, logistic_remap(render depth)) and,
    unless degenerate, make it the medium's guidance (float32).  The guidance
    slots are written by the kernel; the host reads the 96-byte record once to
    learn whether guidance is now active."""
    dev = medium.flat.device
    img = _as_image(gt, dev)
    d = depth_raw.to(device=dev, dtype=torch.float32).contiguous()
    if tuple(d.shape) != tuple(img.shape[:2]):
        raise DataError("image and depth are not co-registered")
    cfg = _cfg(p_dark, intervals_num, resized_height, edges_num)
    result = torch.empty(RESULT_SLOTS, dtype=torch.float64, device=dev)
    _launch(img, d, True, cfg, result, medium.flat[9:15], None)
    est = _estimate(result.cpu().numpy())
    if not est.degenerate:
        medium.mark_guidance()
    return est
