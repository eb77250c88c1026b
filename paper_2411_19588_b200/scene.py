"""Scene state on the device: Gaussians, cameras, medium, optimizer state.

Mirrors the reference types (reference: scene.py:90-371) with the same field
names and semantics.  Learnable tensors are float32 CUDA tensors; the five
cloud fields are contiguous slices of ONE flat buffer laid out
``[positions 3n | log_scales 3n | rotations 4n | sh_coeffs 3n | opacity n]``
so the fused Adam kernel and the gradient all-reduce see a single array.
The medium is a flat float32[15] device buffer: attenuation, water_color,
backscatter, water_color_guide, backscatter_guide.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib

SH_C0 = 0.28209479177387814
WATER_COLOR_BOUNDS = (0.0, 1.0)
BACKSCATTER_BOUNDS = (0.0, 5.0)
CLOUD_FIELDS = ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits")
MEDIUM_FIELDS = ("attenuation", "water_color", "backscatter")
FIELD_WIDTH = {"positions": 3, "log_scales": 3, "rotations": 4, "sh_coeffs": 3,
               "opacity_logits": 1}
FIELD_OFFSET = {"positions": 0, "log_scales": 3, "rotations": 6, "sh_coeffs": 10,
                "opacity_logits": 13}
PARAMS_PER_GAUSSIAN = 14


def default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2411_19588_b200 needs a CUDA device (sm_100a); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _as_f32(a, shape, device):
    if isinstance(a, torch.Tensor):
        t = a.detach().to(device=device, dtype=torch.float32)
    else:
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float32)), device=device)
    return t.reshape(shape)


def quat_to_rotmat(q):
    """wxyz quaternions -> rotation matrices, normalising first (scene.py:32-48)."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                  2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                  2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], axis=-1)
    return R.reshape(q.shape[:-1] + (3, 3))


def rgb_to_feature(rgb):
    return (np.asarray(rgb, dtype=np.float64) - 0.5) / SH_C0


def feature_to_rgb(f):
    return np.asarray(f, dtype=np.float64) * SH_C0 + 0.5


@dataclass
class Gaussian:
    """One primitive as host float64 values (reference scene.py:61-75)."""

    position: np.ndarray
    log_scale: np.ndarray
    rotation: np.ndarray
    sh_coeffs: np.ndarray
    opacity_logit: float

    def __post_init__(self):
        for name, shape in (("position", (3,)), ("log_scale", (3,)), ("rotation", (4,)),
                            ("sh_coeffs", (-1, 3))):
            v = getattr(self, name)
            if isinstance(v, torch.Tensor):
                v = v.detach().cpu().double().numpy()
            setattr(self, name, np.asarray(v, dtype=np.float64).reshape(shape))
        self.opacity_logit = float(self.opacity_logit)


def covariance(g: Gaussian) -> np.ndarray:
    """World covariance (R diag(e^s)) (R diag(e^s))^T of one primitive (scene.py:78-82).
    Scalar host helper; the device kernels form it per Gaussian in float64."""
    m = quat_to_rotmat(g.rotation) * np.exp(g.log_scale)[None, :]
    return m @ m.T


def opacity(g: Gaussian) -> float:
    """sigmoid(logit) as 1 / (1 + exp(-x)) (scene.py:85-87; scipy expit's formula)."""
    return float(1.0 / (1.0 + np.exp(-g.opacity_logit)))


def flat_views(flat: torch.Tensor, n: int) -> dict:
    """Named per-field views of a [14n(+...)] flat buffer."""
    out = {}
    for name in CLOUD_FIELDS:
        w, o = FIELD_WIDTH[name], FIELD_OFFSET[name]
        v = flat[o * n:(o + w) * n]
        if name == "sh_coeffs":
            v = v.view(n, 1, 3)
        elif name == "opacity_logits":
            v = v.view(n)
        else:
            v = v.view(n, w)
        out[name] = v
    return out


class GaussianCloud:
    """Device-resident structure-of-arrays Gaussians (reference scene.py:90-147).

    ``generation`` is bumped whenever the set of Gaussians changes.
    """

    def __init__(self, positions, log_scales, rotations, sh_coeffs, opacity_logits, device=None):
        device = torch.device(device) if device is not None else default_device()
        pos = _as_f32(positions, (-1, 3), device)
        n = pos.shape[0]
        sh = _as_f32(sh_coeffs, (n, -1, 3) if n else (0, 1, 3), device)
        if sh.shape[1] != 1:
            raise ValueError("only constant (degree-0) color features are supported")
        self._n = n
        self._flat = torch.empty(PARAMS_PER_GAUSSIAN * n, dtype=torch.float32, device=device)
        self._bind()
        self.positions.copy_(pos)
        self.log_scales.copy_(_as_f32(log_scales, (n, 3), device))
        self.rotations.copy_(_as_f32(rotations, (n, 4), device))
        self.sh_coeffs.copy_(sh)
        self.opacity_logits.copy_(_as_f32(opacity_logits, (n,), device))
        self.generation = 0
        if n and not bool(torch.isfinite(self._flat).all()):
            for name in CLOUD_FIELDS:
                if not bool(torch.isfinite(getattr(self, name)).all()):
                    raise ValueError(f"non-finite values in {name}")

    def _bind(self):
        for name, v in flat_views(self._flat, self._n).items():
            object.__setattr__(self, "_v_" + name, v)

    def _replace_flat(self, flat: torch.Tensor, n: int):
        """Adopt a new flat parameter buffer of n Gaussians (densification);
        bumps ``generation`` like the reference (optim.py:187)."""
        object.__setattr__(self, "_flat", flat)
        object.__setattr__(self, "_n", n)
        self._bind()
        self.generation += 1

    # field access mirrors the reference attributes; assignment copies in place
    # when the shape is unchanged, otherwise the flat buffer is rebuilt
    def __getattr__(self, name):
        if name in CLOUD_FIELDS:
            return object.__getattribute__(self, "_v_" + name)
        raise AttributeError(name)

    def __setattr__(self, name, value):
        if name in CLOUD_FIELDS and "_flat" in self.__dict__:
            cur = getattr(self, name)
            t = _as_f32(value, (-1,) + tuple(cur.shape[1:]), self._flat.device)
            if t.shape == cur.shape:
                cur.copy_(t)
            else:
                raise ValueError(f"assigning {name} with a different Gaussian count: rebuild the "
                                 "cloud instead (GaussianCloud(...))")
            return
        object.__setattr__(self, name, value)

    @property
    def device(self):
        return self._flat.device

    @property
    def flat(self) -> torch.Tensor:
        return self._flat

    def __len__(self) -> int:
        return self._n

    @property
    def num_sh_coeffs(self) -> int:
        return 1

    def c_struct(self) -> _lib.CloudC:
        return _lib.CloudC(_lib.ptr(self.positions), _lib.ptr(self.log_scales),
                           _lib.ptr(self.rotations), _lib.ptr(self.sh_coeffs),
                           _lib.ptr(self.opacity_logits), self._n)

    def normalize_rotations(self):
        """q / max(|q|, 1e-12) (scene.py:132-134); fused into Adam on the hot path."""
        q = self.rotations.double()
        nr = torch.sqrt(((q[:, 0] ** 2 + q[:, 1] ** 2) + q[:, 2] ** 2) + q[:, 3] ** 2)
        self.rotations.copy_((q / torch.clamp(nr, min=1e-12)[:, None]).float())

    def base_colors(self) -> torch.Tensor:
        """Clamped degree-0 RGB, float64 (scene.py:136-139)."""
        return torch.clamp(self.sh_coeffs[:, 0, :].double() * SH_C0 + 0.5, min=0.0)

    def gaussian(self, i: int) -> Gaussian:
        """Primitive ``i`` as a host Gaussian (scene.py:122-130)."""
        row = {name: getattr(self, name)[i].detach().cpu().double().numpy()
               for name in CLOUD_FIELDS}
        return Gaussian(row["positions"], row["log_scales"], row["rotations"],
                        row["sh_coeffs"], float(row["opacity_logits"]))

    def copy(self) -> "GaussianCloud":
        c = type(self).__new__(type(self))
        object.__setattr__(c, "_n", self._n)
        object.__setattr__(c, "_flat", self._flat.clone())
        c._bind()
        object.__setattr__(c, "generation", self.generation)
        return c

    def numpy(self) -> dict:
        return {name: getattr(self, name).cpu().numpy() for name in CLOUD_FIELDS}


class MediumParams:
    """Water parameters + optional guidance anchors (scene.py:150-187), on device."""

    def __init__(self, attenuation, water_color, backscatter, water_color_guide=None,
                 backscatter_guide=None, device=None):
        device = torch.device(device) if device is not None else default_device()
        self._flat = torch.zeros(15, dtype=torch.float32, device=device)
        self._flat[0:3] = _as_f32(attenuation, (3,), device)
        self._flat[3:6] = _as_f32(water_color, (3,), device)
        self._flat[6:9] = _as_f32(backscatter, (3,), device)
        self._has_wg = water_color_guide is not None
        self._has_bg = backscatter_guide is not None
        if self._has_wg:
            self._flat[9:12] = _as_f32(water_color_guide, (3,), device)
        if self._has_bg:
            self._flat[12:15] = _as_f32(backscatter_guide, (3,), device)

    @property
    def flat(self) -> torch.Tensor:
        return self._flat

    @property
    def params(self) -> torch.Tensor:
        """The 9 learnable values (attenuation, water_color, backscatter)."""
        return self._flat[0:9]

    attenuation = property(lambda s: s._flat[0:3], lambda s, v: s._flat[0:3].copy_(
        _as_f32(v, (3,), s._flat.device)))
    water_color = property(lambda s: s._flat[3:6], lambda s, v: s._flat[3:6].copy_(
        _as_f32(v, (3,), s._flat.device)))
    backscatter = property(lambda s: s._flat[6:9], lambda s, v: s._flat[6:9].copy_(
        _as_f32(v, (3,), s._flat.device)))

    @property
    def water_color_guide(self):
        return self._flat[9:12] if self._has_wg else None

    @water_color_guide.setter
    def water_color_guide(self, v):
        self._has_wg = v is not None
        if v is not None:
            self._flat[9:12] = _as_f32(v, (3,), self._flat.device)

    @property
    def backscatter_guide(self):
        return self._flat[12:15] if self._has_bg else None

    @backscatter_guide.setter
    def backscatter_guide(self, v):
        self._has_bg = v is not None
        if v is not None:
            self._flat[12:15] = _as_f32(v, (3,), self._flat.device)

    @property
    def has_guidance(self) -> bool:
        return self._has_wg and self._has_bg

    def mark_guidance(self):
        """Slots 9..14 were written on the device (guidance refresh): make them
        the active guidance anchors."""
        self._has_wg = self._has_bg = True

    def clamp_(self):
        """Project into the boxes (scene.py:174-178); fused into Adam on the hot path."""
        self._flat[0:3].clamp_(min=0.0)
        self._flat[3:6].clamp_(*WATER_COLOR_BOUNDS)
        self._flat[6:9].clamp_(*BACKSCATTER_BOUNDS)

    def copy(self) -> "MediumParams":
        return type(self)(self.attenuation, self.water_color, self.backscatter,
                          self.water_color_guide, self.backscatter_guide,
                          device=self._flat.device)

    @staticmethod
    def zero(device=None) -> "MediumParams":
        return MediumParams(np.zeros(3), np.zeros(3), np.zeros(3), device=device)


@dataclass
class Camera:
    """Pinhole camera (scene.py:190-245): x_view = R x_world + t; pixel centres at +0.5."""

    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    R: np.ndarray
    t: np.ndarray
    near: float = 0.01
    far: float = 100.0

    def __post_init__(self):
        self.R = np.asarray(self.R, dtype=np.float64).reshape(3, 3)
        self.t = np.asarray(self.t, dtype=np.float64).reshape(3)
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if not (0 < self.near < self.far):
            raise ValueError("require 0 < near < far")

    @property
    def tan_fovx(self) -> float:
        return 0.5 * self.width / self.fx

    @property
    def tan_fovy(self) -> float:
        return 0.5 * self.height / self.fy

    def world_to_view(self, points):
        return np.asarray(points, dtype=np.float64) @ self.R.T + self.t

    def camera_center(self):
        return -self.R.T @ self.t

    @staticmethod
    def look_at(eye, target, up=(0.0, 1.0, 0.0), *, width, height, fx, fy, cx=None, cy=None,
                near=0.01, far=100.0) -> "Camera":
        eye = np.asarray(eye, dtype=np.float64)
        fwd = np.asarray(target, dtype=np.float64) - eye
        fwd = fwd / np.linalg.norm(fwd)
        right = np.cross(np.asarray(up, dtype=np.float64), fwd)
        right = right / np.linalg.norm(right)
        down = np.cross(fwd, right)
        R = np.stack([right, down, fwd], axis=0)
        return Camera(width=width, height=height, fx=fx, fy=fy,
                      cx=width / 2 if cx is None else cx, cy=height / 2 if cy is None else cy,
                      R=R, t=-R @ eye, near=near, far=far)

    @staticmethod
    def from_any(cam) -> "Camera":
        """Accept the reference's Camera (or any duck-typed equivalent)."""
        if isinstance(cam, Camera):
            return cam
        return Camera(width=int(cam.width), height=int(cam.height), fx=float(cam.fx),
                      fy=float(cam.fy), cx=float(cam.cx), cy=float(cam.cy), R=cam.R, t=cam.t,
                      near=float(cam.near), far=float(cam.far))

    def c_struct(self) -> _lib.CameraC:
        return _lib.CameraC(int(self.width), int(self.height), float(self.fx), float(self.fy),
                            float(self.cx), float(self.cy),
                            (_lib.c_double * 9)(*self.R.reshape(-1).tolist()),
                            (_lib.c_double * 3)(*self.t.tolist()), float(self.near),
                            float(self.far))

    @property
    def grid(self):
        return (self.width + 15) // 16, (self.height + 15) // 16


class AdamSlot:
    """Moments + step counter of one tensor (scene.py:248-259); views into TrainState buffers."""

    def __init__(self, m: torch.Tensor, v: torch.Tensor):
        self.m = m
        self.v = v
        self.step = 0


class TrainState:
    """Everything the trainer mutates (scene.py:262-281), device resident."""

    def __init__(self, cloud: GaussianCloud, medium: MediumParams, iteration: int = 0):
        self.cloud = cloud
        self.medium = medium
        self.iteration = iteration
        n = len(cloud)
        dev = cloud.device
        self.exp_avg = torch.zeros(PARAMS_PER_GAUSSIAN * n, dtype=torch.float32, device=dev)
        self.exp_avg_sq = torch.zeros_like(self.exp_avg)
        self.medium_exp_avg = torch.zeros(9, dtype=torch.float32, device=dev)
        self.medium_exp_avg_sq = torch.zeros(9, dtype=torch.float32, device=dev)
        mv, vv = flat_views(self.exp_avg, n), flat_views(self.exp_avg_sq, n)
        self.adam = {name: AdamSlot(mv[name], vv[name]) for name in CLOUD_FIELDS}
        for j, name in enumerate(MEDIUM_FIELDS):
            self.adam[name] = AdamSlot(self.medium_exp_avg[3 * j:3 * j + 3],
                                       self.medium_exp_avg_sq[3 * j:3 * j + 3])
        self.grad_accum = torch.zeros(n, dtype=torch.float32, device=dev)
        self.obs_count = torch.zeros(n, dtype=torch.int32, device=dev)

    def _replace_moments(self, exp_avg: torch.Tensor, exp_avg_sq: torch.Tensor):
        """Adopt new moment buffers for the cloud's current size; the step
        counters are kept (optim.py:190-195)."""
        n = len(self.cloud)
        self.exp_avg, self.exp_avg_sq = exp_avg, exp_avg_sq
        mv, vv = flat_views(self.exp_avg, n), flat_views(self.exp_avg_sq, n)
        for name in CLOUD_FIELDS:
            slot = self.adam[name]
            slot.m, slot.v = mv[name], vv[name]

    def reset_densify_stats(self):
        n = len(self.cloud)
        self.grad_accum = torch.zeros(n, dtype=torch.float32, device=self.cloud.device)
        self.obs_count = torch.zeros(n, dtype=torch.int32, device=self.cloud.device)
