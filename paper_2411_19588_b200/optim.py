"""Optimizer (reference: optim.py).

``apply_gradients`` is one fused sm_100a kernel over the flat parameter
buffer (Adam for the five cloud tensors, quaternion renormalisation) plus a
9-thread kernel for the medium (Adam + box clamp).  Learning rates and bias
corrections are computed here in Python exactly as the reference computes
them, so the device update is bit-identical given the same gradients.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, fields

import torch

from . import _lib
from .scene import CLOUD_FIELDS, MEDIUM_FIELDS, AdamSlot, TrainState

BETA1, BETA2, EPS = 0.9, 0.999, 1e-15


@dataclass
class OptimConfig:
    """Training hyper-parameters (optim.py:16-52)."""

    iterations: int = 30000
    position_lr_init: float = 0.00016
    position_lr_final: float = 0.0000016
    position_lr_delay_mult: float = 0.01
    position_lr_max_steps: int = 30000
    feature_lr: float = 0.0025
    attenuation_lr: float = 0.0025
    backscatter_lr: float = 0.0025
    opacity_lr: float = 0.05
    scaling_lr: float = 0.005
    rotation_lr: float = 0.001
    lambda_ssim: float = 0.3
    lambda_guide: float = 0.1
    densify_interval: int = 100
    opacity_reset_interval: int = 3000
    densify_from: int = 1500
    densify_until: int = 15000
    densify_grad_threshold: float = 0.0002
    min_opacity: float = 0.1
    refit_period: int = 500
    percent_dense: float = 0.01
    split_scale_factor: float = 1.6
    opacity_reset_value: float = 0.01
    checkpoint_interval: int = 1000
    workers: int = 1

    def validate(self):
        for f in fields(self):
            v = getattr(self, f.name)
            if isinstance(v, (int, float)) and v < 0:
                raise ValueError(f"{f.name} must be non-negative")
        if not (self.densify_from <= self.densify_until <= max(self.iterations, self.densify_until)):
            raise ValueError("require densify_from <= densify_until")


def position_lr(iteration: int, cfg: OptimConfig, spatial_scale: float = 1.0) -> float:
    """Sine-ramped log-linear position lr (optim.py:55-66)."""
    t = min(max(iteration / cfg.position_lr_max_steps, 0.0), 1.0)
    ramp = cfg.position_lr_delay_mult + (1.0 - cfg.position_lr_delay_mult) * math.sin(0.5 * math.pi * t)
    log_lerp = math.exp(math.log(cfg.position_lr_init) * (1 - t)
                        + math.log(cfg.position_lr_final) * t)
    return ramp * log_lerp * spatial_scale


_LR_FIELDS = {
    "positions": None,
    "log_scales": "scaling_lr",
    "rotations": "rotation_lr",
    "sh_coeffs": "feature_lr",
    "opacity_logits": "opacity_lr",
    "attenuation": "attenuation_lr",
    "water_color": "backscatter_lr",
    "backscatter": "backscatter_lr",
}


def adam_step(params: torch.Tensor, grads, slot: AdamSlot, lr: float, beta1: float = BETA1,
              beta2: float = BETA2, eps: float = EPS) -> None:
    """One bias-corrected Adam update of a single tensor (optim.py:69-83).

    Standalone float64 torch utility; ``apply_gradients`` uses the fused kernel.
    """
    slot.step += 1
    g = torch.as_tensor(grads, device=params.device).double().reshape(params.shape)
    m = beta1 * slot.m.double() + (1 - beta1) * g
    v = beta2 * slot.v.double() + ((1 - beta2) * g) * g
    m_hat = m / (1 - beta1 ** slot.step)
    v_hat = v / (1 - beta2 ** slot.step)
    params.copy_((params.double() - (lr * m_hat) / (torch.sqrt(v_hat) + eps)).float())
    slot.m.copy_(m.float())
    slot.v.copy_(v.float())


def adam_hparams(state: TrainState, cfg: OptimConfig, spatial_scale: float = 1.0,
                 advance: bool = True) -> _lib.AdamParamsC:
    """Per-tensor lr and bias corrections for the next step (host, float64)."""
    hp = _lib.AdamParamsC()
    for j, name in enumerate(CLOUD_FIELDS + MEDIUM_FIELDS):
        slot = state.adam[name]
        step = slot.step + 1
        if advance:
            slot.step = step
        lr = position_lr(state.iteration, cfg, spatial_scale) if name == "positions" \
            else getattr(cfg, _LR_FIELDS[name])
        hp.lr[j] = lr
        hp.bias1[j] = 1 - BETA1 ** step
        hp.bias2[j] = 1 - BETA2 ** step
        hp.inv_bias1[j] = 1.0 / hp.bias1[j]
        hp.inv_bias2[j] = 1.0 / hp.bias2[j]
    hp.beta1, hp.beta2 = BETA1, BETA2
    hp.one_minus_beta1, hp.one_minus_beta2 = 1 - BETA1, 1 - BETA2
    hp.eps = EPS
    return hp


def apply_gradients(state: TrainState, buf, cfg: OptimConfig, spatial_scale: float = 1.0) -> None:
    """Adam-update every learnable tensor, then re-project constraints (optim.py:98-120)."""
    cloud, medium = state.cloud, state.medium
    if buf.n != len(cloud):
        raise ValueError("gradient buffer does not match the cloud")
    hp = adam_hparams(state, cfg, spatial_scale)
    n = len(cloud)
    _lib.call("uws_adam_step", _lib.ptr(cloud.flat), _lib.ptr(state.exp_avg),
              _lib.ptr(state.exp_avg_sq), _lib.ptr(buf.flat), n, _lib.ptr(medium.flat),
              _lib.ptr(state.medium_exp_avg), _lib.ptr(state.medium_exp_avg_sq),
              _lib.ptr(buf.medium), ctypes.byref(hp), 0, 0, 0, 0, _lib.stream_handle())


def apply_gradients_device(state: TrainState, buf, cfg: OptimConfig, spatial_scale: float = 1.0,
                           zero_grads: bool = True, chunks=None) -> _lib.AdamParamsC:
    """Engine form: skip on device when buf.nonfinite > 0, accumulate the
    densification statistics and leave ``buf`` zeroed.  Advances the step
    counters; the caller rolls them back (``rollback_steps``) if the device
    reported a skip.

    ``chunks`` (optional, see ``range_chunks``): [(group_begin, group_end, wait)]
    covering the cloud's float4 groups; the medium update runs first, then each
    range after its ``wait()`` (e.g. the all-reduce of that part of the buffer),
    with results identical to the single launch."""
    cloud, medium = state.cloud, state.medium
    hp = adam_hparams(state, cfg, spatial_scale)
    st = _lib.stream_handle()
    zg = 1 if zero_grads else 0
    n = len(cloud) if chunks is None else 0
    _lib.call("uws_adam_step", _lib.ptr(cloud.flat), _lib.ptr(state.exp_avg),
              _lib.ptr(state.exp_avg_sq), _lib.ptr(buf.flat), n, _lib.ptr(medium.flat),
              _lib.ptr(state.medium_exp_avg), _lib.ptr(state.medium_exp_avg_sq),
              _lib.ptr(buf.medium), ctypes.byref(hp), _lib.ptr(buf.nonfinite),
              _lib.ptr(state.grad_accum), _lib.ptr(state.obs_count), zg, st)
    for g0, g1, wait in chunks or ():
        if wait is not None:
            wait()
        _lib.call("uws_adam_step_range", _lib.ptr(cloud.flat), _lib.ptr(state.exp_avg),
                  _lib.ptr(state.exp_avg_sq), _lib.ptr(buf.flat), len(cloud), ctypes.byref(hp),
                  _lib.ptr(buf.nonfinite), _lib.ptr(state.grad_accum), _lib.ptr(state.obs_count),
                  zg, int(g0), int(g1), st)
    return hp


def range_chunks(state: TrainState, buf, parts: int):
    """Float4-group ranges [(g0, g1)] splitting the cloud update into ``parts``
    launches, or None when the range form does not apply (odd n or buffers not
    16-byte aligned: the single launch then takes its scalar path)."""
    n = len(state.cloud)
    ptrs = (state.cloud.flat, state.exp_avg, state.exp_avg_sq, buf.flat)
    if n == 0 or n % 2 or any(t.data_ptr() % 16 for t in ptrs):
        return None
    groups = 14 * n // 4
    parts = max(1, min(parts, groups))
    return [(groups * c // parts, groups * (c + 1) // parts) for c in range(parts)]


def rollback_steps(state: TrainState) -> None:
    """Undo the step-counter advance of a skipped update (pipeline.py:182-189)."""
    for slot in state.adam.values():
        slot.step -= 1


def densify_and_prune(state: TrainState, cfg: OptimConfig, scene_extent: float, rng):
    """Clone/split high-gradient Gaussians, prune transparent ones, on the device
    (reference optim.py:132-198; same arguments, return value and random draws).

    One host read of the three counts sizes the new buffers; the split samples
    come from ``rng.standard_normal((2, n_split, 3))`` exactly as in the
    reference so a shared seed reproduces its cloud.  Returns
    (clones, splits, pruned).  A StepEngine driving this state must be
    flushed first (``engine.flush()``): it resizes itself on its next step.
    """
    import numpy as np
    cloud = state.cloud
    n = len(cloud)
    if n == 0:
        return 0, 0, 0
    dev = cloud.device
    st = _lib.stream_handle()
    b = _lib.size_out()
    _lib.call("uws_densify_workspace_size", n, ctypes.byref(b))
    ws = torch.empty(max(b.value, 1), dtype=torch.uint8, device=dev)
    totals = torch.zeros(3, dtype=torch.int64, device=dev)
    _lib.call("uws_densify_classify", _lib.ptr(cloud.flat), n, _lib.ptr(state.grad_accum),
              _lib.ptr(state.obs_count), float(cfg.densify_grad_threshold),
              float(cfg.percent_dense * scene_extent), float(cfg.min_opacity), _lib.ptr(totals),
              _lib.ptr(ws), ws.numel(), st)
    n_keep, n_clone, n_split = (int(v) for v in totals.cpu())
    n_prune = n - n_keep - n_split
    if n_keep == 0 and n_split == 0:
        return 0, 0, 0  # refuse to empty the cloud (optim.py:160-161)
    samples = None
    if n_split:
        draw = np.ascontiguousarray(rng.standard_normal((2, n_split, 3)), dtype=np.float64)
        samples = torch.from_numpy(draw).to(dev)
    n_new = n_keep + n_clone + 2 * n_split
    flat = torch.empty(14 * n_new, dtype=torch.float32, device=dev)
    m = torch.zeros(14 * n_new, dtype=torch.float32, device=dev)
    v = torch.zeros(14 * n_new, dtype=torch.float32, device=dev)
    _lib.call("uws_densify_apply", _lib.ptr(cloud.flat), _lib.ptr(state.exp_avg),
              _lib.ptr(state.exp_avg_sq), n, _lib.ptr(ws), ws.numel(),
              _lib.ptr(samples) if samples is not None else 0,
              float(np.log(cfg.split_scale_factor)), n_keep, n_clone, n_split, _lib.ptr(flat),
              _lib.ptr(m), _lib.ptr(v), st)
    cloud._replace_flat(flat, n_new)
    state._replace_moments(m, v)
    state.reset_densify_stats()
    return n_clone, n_split, n_prune


def reset_opacities(state: TrainState, cfg: OptimConfig) -> None:
    """Set every opacity logit to logit(reset value) and clear its moments
    (reference optim.py:201-207), on the device."""
    import numpy as np
    target = math.log(cfg.opacity_reset_value / (1 - cfg.opacity_reset_value))
    _lib.call("uws_reset_opacities", _lib.ptr(state.cloud.flat), _lib.ptr(state.exp_avg),
              _lib.ptr(state.exp_avg_sq), len(state.cloud), float(np.float32(target)),
              _lib.stream_handle())
