"""Screen-space projection on the device (reference: projection.py).

``project_cloud`` runs the sm_100a preprocess kernel (EWA covariance,
opacity-aware radius, tile rectangle, compaction of the visible set in source
order) and returns a :class:`ProjectedCloud` whose fields carry the
reference's names.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .scene import Camera, GaussianCloud

TILE_SIZE = 16
COV2D_DILATION = 0.3
ALPHA_FLOOR = 1.0 / 255.0
MIN_RADIUS_SIGMA = 3.0
SPLAT_FLOATS = 12  # uws_splat is 48 bytes


@dataclass
class Projected2D:
    """One footprint as host float64 values (reference projection.py:29-37)."""

    mean2d: np.ndarray     # (2,) pixels
    cov2d: np.ndarray      # (2, 2), dilation included
    depth: float           # view z
    radius: float          # footprint radius, pixels
    source_index: int


class ProjectedCloud:
    """Device form of the reference ProjectedCloud (projection.py:40-86).

    Rows are the K visible Gaussians in ascending source order.  Field views:
    ``source_index`` (K,) int32, ``mean2d`` (K,2) f64, ``conic`` (K,3) f64,
    ``opacity`` (K,) f64, ``depth`` (K,) f64, ``color`` (K,3) f32,
    ``rect`` (K,4) int16 inclusive tile rectangle, and -- when requested --
    ``cov2d`` (K,3) f64 and ``radius`` (K,) f64.  The backward context of the
    reference (t_view, rotmat, cov3d, ...) is recomputed on the device from
    the cloud instead of being stored.
    """

    def __init__(self, n_source: int, device, with_geometry: bool = True):
        cap = max(n_source, 1)
        self.n_source = n_source
        self.device = device
        self._source_index = torch.empty(cap, dtype=torch.int32, device=device)
        self._splat = torch.empty(cap, SPLAT_FLOATS, dtype=torch.float32, device=device)
        self._exact = torch.empty(cap, 4, dtype=torch.float64, device=device)
        self._depth = torch.empty(cap, dtype=torch.float64, device=device)
        self._rect = torch.empty(cap, 4, dtype=torch.int16, device=device)
        self._cov2d = torch.empty(cap, 3, dtype=torch.float64, device=device) if with_geometry else None
        self._radius = torch.empty(cap, dtype=torch.float64, device=device) if with_geometry else None
        self._num_visible = torch.zeros(1, dtype=torch.int32, device=device)
        # {~min, max} of the visible depths' high words (preprocess -> binning)
        self._depth_range = torch.zeros(2, dtype=torch.int32, device=device)
        self._k = 0 if n_source == 0 else None   # host copy of K, read lazily

    def c_struct(self) -> _lib.ProjectedC:
        return _lib.ProjectedC(_lib.ptr(self._source_index), _lib.ptr(self._splat),
                               _lib.ptr(self._exact), _lib.ptr(self._depth), _lib.ptr(self._rect),
                               _lib.ptr(self._cov2d), _lib.ptr(self._radius),
                               _lib.ptr(self._num_visible), _lib.ptr(self._depth_range))

    @property
    def k(self) -> int:
        """Number of visible rows (one device-to-host read on first use)."""
        if self._k is None:
            self._k = int(self._num_visible.item())
        return self._k

    def invalidate(self):
        """Forget the host copy of K (the buffers are being re-filled)."""
        self._k = 0 if self.n_source == 0 else None

    @property
    def num_visible(self) -> torch.Tensor:
        return self._num_visible

    def __len__(self) -> int:
        return self.k

    # -- reference field names ------------------------------------------------
    @property
    def source_index(self):
        return self._source_index[:self.k]

    @property
    def mean2d(self):
        return self._splat[:self.k].view(torch.float64)[:, 0:2]

    @property
    def conic(self):
        return self._exact[:self.k, 0:3]

    @property
    def opacity(self):
        return self._exact[:self.k, 3]

    @property
    def depth(self):
        return self._depth[:self.k]

    @property
    def color(self):
        return self._splat[:self.k, 8:11]

    @property
    def rect(self):
        return self._rect[:self.k]

    @property
    def cov2d(self):
        return None if self._cov2d is None else self._cov2d[:self.k]

    @property
    def radius(self):
        return None if self._radius is None else self._radius[:self.k]

    @property
    def color_clamped(self):
        return self.color <= 0.0

    def item(self, i: int) -> Projected2D:
        """Row ``i`` as a host Projected2D (needs the geometry fields)."""
        if self._cov2d is None:
            raise ValueError("projected without geometry (with_geometry=False)")
        a, b, c = (float(v) for v in self._cov2d[i].tolist())
        return Projected2D(mean2d=self.mean2d[i].cpu().numpy().astype(np.float64),
                           cov2d=np.array([[a, b], [b, c]]), depth=float(self.depth[i]),
                           radius=float(self.radius[i]), source_index=int(self.source_index[i]))


def preprocess_into(proj: ProjectedCloud, cloud: GaussianCloud, cam, workspace=None) -> None:
    """Run the preprocess kernel into an existing ProjectedCloud (no host sync)."""
    proj.invalidate()
    if len(cloud) == 0:
        proj._num_visible.zero_()
        return
    if workspace is None:
        ws_bytes = _lib.size_out()
        _lib.call("uws_preprocess_workspace_size", len(cloud), ctypes.byref(ws_bytes))
        workspace = torch.empty(ws_bytes.value, dtype=torch.uint8, device=cloud.device)
    cl, cc, pc = cloud.c_struct(), cam.c_struct(), proj.c_struct()
    _lib.call("uws_preprocess_fwd", ctypes.byref(cl), ctypes.byref(cc), ctypes.byref(pc),
              _lib.ptr(workspace), workspace.numel(), _lib.stream_handle())


def project_cloud(cloud: GaussianCloud, cam, with_geometry: bool = True) -> ProjectedCloud:
    """Project every Gaussian, dropping those that cannot touch the image
    (reference projection.py:100-199).  K is read from the device lazily."""
    cam = Camera.from_any(cam)
    proj = ProjectedCloud(len(cloud), cloud.device, with_geometry)
    preprocess_into(proj, cloud, cam)
    return proj


def project_gaussian(g, cam) -> Optional[Projected2D]:
    """Project one primitive through the device kernel; None when culled
    (reference projection.py:202-211)."""
    from .scene import GaussianCloud
    cloud = GaussianCloud(g.position[None, :], g.log_scale[None, :], g.rotation[None, :],
                          np.asarray(g.sh_coeffs, np.float64).reshape(1, -1, 3),
                          np.array([g.opacity_logit]))
    proj = project_cloud(cloud, cam)
    return proj.item(0) if len(proj) else None


def tile_span(p, tile_size: int = TILE_SIZE, grid=None):
    """Inclusive tile rectangle of one footprint ``p`` (mean2d, radius), None when
    no pixel centre is reached (projection.py:214-226).

    Host-side helper (float64, same formula as the device kernel)."""
    mx, my = float(p.mean2d[0]), float(p.mean2d[1])
    r = float(p.radius)
    s = [np.floor(np.ceil(mx - r - 0.5 - 1e-9) / tile_size),
         np.floor(np.ceil(my - r - 0.5 - 1e-9) / tile_size),
         np.floor(np.floor(mx + r - 0.5 + 1e-9) / tile_size),
         np.floor(np.floor(my + r - 0.5 + 1e-9) / tile_size)]
    x0, y0, x1, y1 = (int(v) for v in s)
    if grid is not None:
        gx, gy = grid
        x0, y0 = min(max(x0, 0), gx - 1), min(max(y0, 0), gy - 1)
        x1, y1 = max(min(max(x1, -1), gx - 1), x0 - 1), max(min(max(y1, -1), gy - 1), y0 - 1)
    if x1 < x0 or y1 < y0:
        return None
    return x0, y0, x1, y1
