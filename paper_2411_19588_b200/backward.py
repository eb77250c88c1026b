"""Analytic gradients on the device (reference: backward.py).

``backward_render`` runs the back-to-front compositing backward kernel
(screen-space gradients + medium sums) and the projection backward kernel
(chain to positions / log-scales / quaternions / SH / opacity logits) into a
:class:`GradientBuffer`.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import _lib
from .errors import NumericError
from .medium import logistic_remap
from .rasterizer import ALPHA_CLAMP, T_EARLY_STOP, RenderOutput, alpha_at, apply_water, render
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


# Default of backward_render's ``deterministic``: run-to-run bit-identical
# gradients (the reference's fixed tile-order merge, backward.py:334-341) at the
# cost of a per-view host read, a slot buffer and a sort; off by default (the
# float atomics' order varies, values agree to float32 rounding).
DETERMINISTIC = False


def set_deterministic(on: bool = True) -> None:
    """Make backward_render deterministic by default (e.g. under dropin)."""
    global DETERMINISTIC
    DETERMINISTIC = bool(on)


def _raster_bwd_det(proj, bins, rows, cam, med, out, dL, screen, med_acc, st):
    """Deterministic K8: per-(tile, Gaussian) slots, row sort, tile-order sums."""
    dev = dL.device
    gx, gy = cam.grid
    tiles = gx * gy
    count = torch.empty(tiles, dtype=torch.int32, device=dev)
    base = torch.empty(tiles + 1, dtype=torch.int32, device=dev)
    cc, oc = cam.c_struct(), out.c_struct()
    _lib.call("uws_raster_bwd_det_prefix", ctypes.byref(cc), ctypes.byref(oc), _lib.ptr(count),
              _lib.ptr(base), st)
    r = int(base[tiles].item())
    k = proj.k
    nb = _lib.size_out()
    _lib.call("uws_raster_bwd_det_workspace_size", tiles, r, k, ctypes.byref(nb))
    ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=dev)
    pc = proj.c_struct()
    if rows is not None:
        lists = (0, 0, _lib.ptr(rows.row_start), _lib.ptr(rows.items))
    else:
        lists = (_lib.ptr(bins.offsets), _lib.ptr(bins.entries), 0, 0)
    _lib.call("uws_raster_bwd_det", ctypes.byref(pc), *lists, ctypes.byref(cc), med,
              ctypes.byref(oc), _lib.ptr(dL), _lib.ptr(screen), _lib.ptr(med_acc),
              _lib.ptr(base), r, k, _lib.ptr(ws), ws.numel(), st)


def backward_render(out: RenderOutput, dL_dC, cloud: GaussianCloud,
                    medium: Optional[MediumParams] = None, lambda_guide: float = 0.0,
                    workers: int = 1, buf: Optional[GradientBuffer] = None,
                    deterministic: Optional[bool] = None) -> GradientBuffer:
    """Accumulate all parameter gradients for one rendered view (backward.py:278-344).

    ``buf`` (optional) is accumulated into instead of a fresh buffer, which is
    how several views are summed before one optimizer step.  ``deterministic``
    (default: module DETERMINISTIC) makes the result bit-identical run to run.
    """
    if deterministic is None:
        deterministic = DETERMINISTIC
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
    if deterministic:
        _raster_bwd_det(proj, bins, rows, cam, med, out, dL, screen, med_acc, st)
    elif rows is not None:   # the forward composited from row lists: filter them again
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


def backward_pixel(contributors, pixel, dL_dC, att):
    """Per-contributor gradients of one pixel (backward.py:72-121): replay the
    blend of ``composite_pixel``, then walk back with the suffix sum
    sum_{j>i} c_j alpha_j T_j.  Returns a list of dicts d_color, d_logit,
    d_mean2d, d_conic (zeros where the floor, clamp or early stop applies).
    Scalar host helper (float64) mirroring the backward kernel's rules."""
    G = np.asarray(dL_dC, dtype=np.float64) * np.asarray(att, dtype=np.float64)
    pix = np.asarray(pixel, dtype=np.float64)
    replay, t = [], 1.0
    for p, logit, rgb in contributors:
        live = t >= T_EARLY_STOP
        a = alpha_at(p, logit, pix) if live else 0.0
        replay.append((p, float(logit), np.asarray(rgb, dtype=np.float64), a, t, live))
        if live and a > 0.0:
            t *= 1.0 - a
    grads = [None] * len(replay)
    suffix = np.zeros(3)
    for i in range(len(replay) - 1, -1, -1):
        p, logit, rgb, a, t_i, live = replay[i]
        g = {"d_color": np.zeros(3), "d_logit": 0.0, "d_mean2d": np.zeros(2),
             "d_conic": np.zeros(3)}
        if live and a > 0.0:
            g["d_color"] = a * t_i * G
            d_alpha = float(G @ (rgb * t_i - suffix / (1.0 - a)))
            s = 1.0 / (1.0 + np.exp(-logit))
            d = pix - np.asarray(p.mean2d, dtype=np.float64)
            inv = np.linalg.inv(np.asarray(p.cov2d, dtype=np.float64))
            a_raw = s * np.exp(-0.5 * float(d @ inv @ d))
            if ALPHA_FLOOR <= a_raw < ALPHA_CLAMP:
                d_power = d_alpha * a_raw
                g["d_logit"] = d_power * (1.0 - s)
                g["d_mean2d"] = d_power * (inv @ d)
                g["d_conic"] = d_power * np.array([-0.5 * d[0] * d[0], -d[0] * d[1],
                                                   -0.5 * d[1] * d[1]])
            suffix = suffix + rgb * a * t_i
        grads[i] = g
    return grads


# ----------------------------------------------------------------------------
# finite-difference check of the device gradients (backward.py:353-494)
# ----------------------------------------------------------------------------
# Central-difference steps.  The reference takes 1e-5 steps on a float64
# forward; the device forward composites in float32, whose rounding noise
# (~1e-7 relative per pixel) would swamp a 1e-5 difference quotient, so the
# default steps are 1e-3 (still far below the scale of the forward's gates).
EPS_DEFAULTS = {name: 1e-3 for name in ("positions", "log_scales", "rotations", "sh_coeffs",
                                        "opacity_logits", "attenuation", "water_color",
                                        "backscatter")}
ALPHA_FLOOR = 1.0 / 255.0


@dataclass
class GradCheckRow:
    param: str
    index: tuple
    analytic: float
    fd: float
    rel_err: float
    step: float = 0.0     # the central-difference step finally used


@dataclass
class GradCheckReport:
    rows: List[GradCheckRow] = field(default_factory=list)
    tol: float = 1e-3

    @property
    def max_rel_err(self) -> float:
        return max((r.rel_err for r in self.rows), default=0.0)

    @property
    def flagged(self) -> List[GradCheckRow]:
        return [r for r in self.rows if r.rel_err >= self.tol]

    def group_max(self) -> dict:
        out = {}
        for r in self.rows:
            out[r.param] = max(out.get(r.param, 0.0), r.rel_err)
        return out

    def table(self) -> str:
        counts, flags = {}, {}
        for r in self.rows:
            counts[r.param] = counts.get(r.param, 0) + 1
            flags[r.param] = flags.get(r.param, 0) + int(r.rel_err >= self.tol)
        lines = [f"{'param':<16}{'max rel err':>14}{'entries':>9}{'flagged':>9}"]
        for param, mx in self.group_max().items():
            lines.append(f"{param:<16}{mx:>14.3e}{counts[param]:>9}{flags[param]:>9}")
        lines.append(f"overall max rel err {self.max_rel_err:.3e} "
                     f"({'PASS' if not self.flagged else 'FAIL'} at tol {self.tol:g})")
        return "\n".join(lines)


def _frozen_depth_eval(cloud, cam, medium, gt, depth_frozen, lambda_ssim, lambda_guide):
    """(loss, per-pixel blend counts) of the frozen-depth objective."""
    from .losses import loss_value_f64
    out = render(cloud, cam, mode="clean", retain=False)
    img = apply_water(out.color, depth_frozen, medium) if medium is not None else out.color
    total = loss_value_f64(img, gt, medium, lambda_ssim, lambda_guide)
    if not np.isfinite(total):
        raise NumericError("non-finite loss in finite-difference evaluation")
    return total, out.count


def frozen_depth_loss(cloud: GaussianCloud, cam, medium: Optional[MediumParams], gt,
                      depth_frozen, lambda_ssim: float, lambda_guide: float) -> float:
    """The objective with the depth map pinned (backward.py:391-405): device clean
    render, the water model applied with ``depth_frozen`` (float64), and the loss
    evaluated in float64 on the device (losses.loss_value_f64)."""
    return _frozen_depth_eval(cloud, cam, medium, gt, depth_frozen, lambda_ssim,
                              lambda_guide)[0]


def finite_diff_check(cloud: GaussianCloud, cam, medium: Optional[MediumParams], gt,
                      lambda_ssim: float = 0.3, lambda_guide: float = 0.1,
                      eps: Optional[dict] = None, tol: float = 1e-3,
                      analytic: Optional[GradientBuffer] = None) -> GradCheckReport:
    """Every device gradient against central finite differences of the device
    forward + loss (backward.py:408-494): perturbations are the representable
    float32 steps of each parameter, the depth map is frozen at the base render.
    Meant for small scenes (one render + loss per perturbation)."""
    from .losses import total_loss
    eps_map = dict(EPS_DEFAULTS)
    eps_map.update(eps or {})
    mode = "clean" if medium is None else "underwater"
    out = render(cloud, cam, medium=medium, mode=mode)
    depth_frozen = out.depth.clone()
    if analytic is None:
        _, dL = total_loss(out.color, gt, medium, lambda_ssim, lambda_guide)
        analytic = backward_render(out, dL, cloud, medium, lambda_guide)
    cloud2 = cloud.copy()
    medium2 = medium.copy() if medium is not None else None
    report = GradCheckReport(tol=tol)

    def loss():
        return _frozen_depth_eval(cloud2, cam, medium2, gt, depth_frozen, lambda_ssim,
                                  lambda_guide)

    _, count0 = loss()

    def check(param, arr, grads):
        host_grads = grads.detach().double().cpu().numpy()
        base_all = arr.detach().cpu().numpy()
        for idx in np.ndindex(base_all.shape):
            base = np.float32(base_all[idx])
            # the forward's hard gates (1/255 floor, T >= 1e-4 stop) are steps in the
            # loss: a step that moves any pixel's blend count across one measures the
            # jump, so the step is shrunk (x1/10, at most twice) until no count moves
            e = eps_map[param]
            for _ in range(3):
                hi, lo = np.float32(base + e), np.float32(base - e)
                arr[idx] = float(hi)
                l_plus, c_plus = loss()
                arr[idx] = float(lo)
                l_minus, c_minus = loss()
                arr[idx] = float(base)
                if torch.equal(c_plus, count0) and torch.equal(c_minus, count0):
                    break
                e *= 0.1
            fd = (l_plus - l_minus) / (np.float64(hi) - np.float64(lo))
            a = float(host_grads[idx])
            report.rows.append(GradCheckRow(param, idx, a, float(fd),
                                            float(abs(a - fd) / max(abs(fd), 1e-6)),
                                            float(np.float64(hi) - np.float64(lo)) / 2))

    for param in ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits"):
        check(param, getattr(cloud2, param), getattr(analytic, "d_" + param))
    if medium2 is not None:
        for param in ("attenuation", "water_color", "backscatter"):
            check(param, getattr(medium2, param), getattr(analytic, "d_" + param))
    return report
