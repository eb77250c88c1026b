"""Helpers shared by the GPU parity tests."""

from types import SimpleNamespace

import numpy as np
import torch

import paper_2411_19588_b200 as uw

FIELDS = ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits")
GRAD_FIELDS = ("d_positions", "d_log_scales", "d_rotations", "d_sh_coeffs", "d_opacity_logits")


def device_scene(g):
    """GaussianCloud / Camera / MediumParams on cuda from a golden or oracle scene."""
    cloud = uw.GaussianCloud(**{k: getattr(g.cloud, k) for k in FIELDS})
    cam = uw.Camera.from_any(g.cam)
    medium = None
    if g.medium is not None:
        m = g.medium
        medium = uw.MediumParams(m.attenuation, m.water_color, m.backscatter,
                                 getattr(m, "water_color_guide", None),
                                 getattr(m, "backscatter_guide", None))
    return cloud, cam, medium


def host_cloud(n, seed=0, spread=4.0, scale_mult=None, opacity=(-1.0, 1.5)):
    """The survey's synthetic generator (reference fixtures.random_cloud)."""
    rng = np.random.default_rng(seed)
    f = (1e4 / n) ** (1.0 / 3.0) if scale_mult is None else scale_mult
    pos = np.stack([rng.uniform(-spread, spread, n), rng.uniform(-spread, spread, n),
                    rng.uniform(4.0, 20.0, n)], axis=1)
    log_scales = np.log(rng.uniform(0.15 * f, 0.6 * f, (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    colors = rng.uniform(0.1, 0.9, (n, 3))
    sh = ((colors - 0.5) / uw.scene.SH_C0)[:, None, :]
    logits = rng.uniform(*opacity, n)
    return SimpleNamespace(positions=pos.astype(np.float32), log_scales=log_scales.astype(np.float32),
                           rotations=q.astype(np.float32), sh_coeffs=sh.astype(np.float32),
                           opacity_logits=logits.astype(np.float32))


def survey_camera(W, H):
    return uw.Camera.look_at((3, -2, -1), (0, 0, 12), width=W, height=H, fx=1.2 * W, fy=1.2 * W)


def survey_medium(guided=True):
    if guided:
        return SimpleNamespace(attenuation=np.array([0.6, 0.45, 0.3], np.float32),
                               water_color=np.array([0.2, 0.35, 0.5], np.float32),
                               backscatter=np.array([0.8, 1.0, 1.2], np.float32),
                               water_color_guide=np.array([0.25, 0.3, 0.45], np.float32),
                               backscatter_guide=np.array([0.9, 1.0, 1.1], np.float32))
    return SimpleNamespace(attenuation=np.array([0.6, 0.45, 0.3], np.float32),
                           water_color=np.array([0.2, 0.35, 0.5], np.float32),
                           backscatter=np.array([0.8, 1.0, 1.2], np.float32),
                           water_color_guide=None, backscatter_guide=None)


def grad_tolerance_ok(got, ref, rel=1e-3, abs_frac=1e-6):
    """SURVEY §8c contract: |g - g_ref| <= rel*|g_ref| + abs_frac*max|g_ref|."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    tol = rel * np.abs(ref) + abs_frac * max(np.abs(ref).max(), 1e-30)
    bad = np.abs(got - ref) > tol
    return int(bad.sum()), float((np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30))[bad].max()
                                 if bad.any() else 0.0)


def np_(t):
    return t.detach().cpu().numpy()


def adam_replay(params, grads, medium, iteration, cfg, moments=None, step=1, spatial_scale=1.0):
    """The reference's apply_gradients (optim.py:98-120) in numpy on float32
    gradients ``grads`` (dict d_<field> / medium (9,)): returns the updated
    (params, medium, moments).  ``moments`` = (m, v, medium m, medium v) or None."""
    from oracle import uwsplat_oracle as O
    lrs = {"positions": uw.position_lr(iteration, cfg, spatial_scale),
           "log_scales": cfg.scaling_lr, "rotations": cfg.rotation_lr,
           "sh_coeffs": cfg.feature_lr, "opacity_logits": cfg.opacity_lr}
    if moments is None:
        moments = ({f: np.zeros_like(v) for f, v in params.items()},
                   {f: np.zeros_like(v) for f, v in params.items()},
                   {f: np.zeros(3, np.float32) for f in MEDIUM_FIELDS},
                   {f: np.zeros(3, np.float32) for f in MEDIUM_FIELDS})
    m, v, mm, mv = moments
    out = {}
    for f in FIELDS:
        out[f], m[f], v[f] = O.adam(params[f], grads["d_" + f], m[f], v[f], step, lrs[f])
    out["rotations"] = O.renormalize(out["rotations"])
    new_med = []
    for j, f in enumerate(MEDIUM_FIELDS):
        lr = getattr(cfg, uw.optim._LR_FIELDS[f])
        q, mm[f], mv[f] = O.adam(medium[f], grads["medium"][3 * j:3 * j + 3], mm[f], mv[f],
                                 step, lr)
        new_med.append(q)
    med = dict(zip(MEDIUM_FIELDS, O.clamp_medium(*new_med)))
    return out, med, (m, v, mm, mv)


MEDIUM_FIELDS = ("attenuation", "water_color", "backscatter")


def host_state(cloud, medium):
    """float32 host copies of a device cloud / medium (for adam_replay)."""
    params = {f: np_(getattr(cloud, f)).copy() for f in FIELDS}
    med = {f: np_(getattr(medium, f)).copy() for f in MEDIUM_FIELDS}
    return params, med


def host_grads(buf):
    g = {f: np_(getattr(buf, f)).copy() for f in GRAD_FIELDS}
    g["medium"] = np_(buf.medium).copy()
    return g
