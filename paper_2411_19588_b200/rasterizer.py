"""Tile binning and forward compositing on the device (reference: rasterizer.py).

``bin_and_sort`` and ``render`` keep the reference signatures; all per-tile
work runs in the sm_100a kernels (depth radix sort, tile-key emission, tile
radix sort, tile ranges, per-tile front-to-back compositing with the medium
epilogue).  Outputs are float32 CUDA tensors.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .medium import logistic_remap
from .projection import ALPHA_FLOOR, TILE_SIZE, ProjectedCloud, project_cloud
from .scene import Camera, GaussianCloud, MediumParams

ALPHA_CLAMP = 0.99
T_EARLY_STOP = 1e-4
WEIGHT_EPS = 1e-8


class TileBins:
    """CSR tile lists (rasterizer.py:32-47): ``offsets`` (tiles+1,) and
    ``entries`` (E,) int32 device tensors; entries are ProjectedCloud rows
    sorted by (tile, depth, source index)."""

    def __init__(self, grid_x: int, grid_y: int, offsets: torch.Tensor, entries: torch.Tensor):
        self.grid_x = grid_x
        self.grid_y = grid_y
        self.offsets = offsets
        self.entries = entries

    def tile_entries(self, tx: int, ty: int) -> torch.Tensor:
        tid = ty * self.grid_x + tx
        a, b = (int(v) for v in self.offsets[tid:tid + 2].tolist())
        return self.entries[a:b]


def bin_and_sort(proj: ProjectedCloud, width: int, height: int,
                 tile_size: int = TILE_SIZE) -> TileBins:
    """Assign footprints to tiles and depth-sort each list (rasterizer.py:50-85).

    Standalone form: reads the entry counts once and allocates exactly.  The
    training engine (engine.py) uses capacity buffers instead and never syncs.
    """
    if tile_size != TILE_SIZE:
        raise ValueError("the device kernels use 16x16 tiles")
    cam = Camera(width=width, height=height, fx=1.0, fy=1.0, cx=0.0, cy=0.0, R=[[1, 0, 0],
                 [0, 1, 0], [0, 0, 1]], t=[0, 0, 0])
    gx, gy = cam.grid
    dev = proj.device
    offsets = torch.zeros(gx * gy + 1, dtype=torch.int32, device=dev)
    k_cap = proj.n_source
    if k_cap == 0:
        return TileBins(gx, gy, offsets, torch.empty(0, dtype=torch.int32, device=dev))
    cb, eb = _lib.size_out(), _lib.size_out()
    _lib.call("uws_bin_workspace_size", k_cap, 0, gx, gy, ctypes.byref(cb), ctypes.byref(eb))
    count_ws = torch.empty(cb.value, dtype=torch.uint8, device=dev)
    totals = torch.zeros(2, dtype=torch.int64, device=dev)
    overflow = torch.zeros(1, dtype=torch.int32, device=dev)
    pc, cc = proj.c_struct(), cam.c_struct()
    st = _lib.stream_handle()
    _lib.call("uws_bin_count", ctypes.byref(pc), k_cap, ctypes.byref(cc), _lib.ptr(totals),
              _lib.ptr(count_ws), cb.value, st)
    e, s = (int(v) for v in totals.tolist())
    entries = torch.empty(max(e, 1), dtype=torch.int32, device=dev)
    _lib.call("uws_bin_workspace_size", k_cap, s, gx, gy, ctypes.byref(cb), ctypes.byref(eb))
    emit_ws = torch.empty(eb.value, dtype=torch.uint8, device=dev)
    _lib.call("uws_bin_emit", ctypes.byref(pc), k_cap, e, s, ctypes.byref(cc), _lib.ptr(totals),
              _lib.ptr(offsets), _lib.ptr(entries), _lib.ptr(overflow), 0, _lib.ptr(count_ws),
              cb.value, _lib.ptr(emit_ws), eb.value, st)
    return TileBins(gx, gy, offsets, entries[:e])


class RowLists:
    """Tile-ROW lists: for every tile row, the depth-ordered 8-byte items
    ``(row, x0 | x1 << 16)`` of the Gaussians whose rectangle spans it.  The
    list of tile (tx, ty) is the subsequence of row ty's list whose column span
    contains tx, so the compositing kernels filter it on the fly."""

    def __init__(self, grid_x: int, grid_y: int, row_start: torch.Tensor, items: torch.Tensor):
        self.grid_x = grid_x
        self.grid_y = grid_y
        self.row_start = row_start
        self.items = items


def bin_rows(proj: ProjectedCloud, width: int, height: int) -> RowLists:
    """First level of bin_and_sort (rasterizer.py:50-85): the stable depth order
    bucketed into tile-row lists (one host read of the item count)."""
    cam = Camera(width=width, height=height, fx=1.0, fy=1.0, cx=0.0, cy=0.0, R=[[1, 0, 0],
                 [0, 1, 0], [0, 0, 1]], t=[0, 0, 0])
    gx, gy = cam.grid
    dev = proj.device
    row_start = torch.zeros(gy + 1, dtype=torch.int32, device=dev)
    k_cap = proj.n_source
    if k_cap == 0:
        return RowLists(gx, gy, row_start, torch.zeros(1, 2, dtype=torch.int32, device=dev))
    cb, eb = _lib.size_out(), _lib.size_out()
    _lib.call("uws_bin_workspace_size", k_cap, 0, gx, gy, ctypes.byref(cb), ctypes.byref(eb))
    count_ws = torch.empty(cb.value, dtype=torch.uint8, device=dev)
    totals = torch.zeros(2, dtype=torch.int64, device=dev)
    overflow = torch.zeros(1, dtype=torch.int32, device=dev)
    pc, cc = proj.c_struct(), cam.c_struct()
    st = _lib.stream_handle()
    _lib.call("uws_bin_count", ctypes.byref(pc), k_cap, ctypes.byref(cc), _lib.ptr(totals),
              _lib.ptr(count_ws), cb.value, st)
    s = int(totals[1].item())
    items = torch.empty(max(s, 1), 2, dtype=torch.int32, device=dev)
    _lib.call("uws_bin_rows", ctypes.byref(pc), k_cap, max(s, 1), ctypes.byref(cc),
              _lib.ptr(totals), _lib.ptr(row_start), _lib.ptr(items), _lib.ptr(overflow), 0,
              _lib.ptr(count_ws), cb.value, st)
    return RowLists(gx, gy, row_start, items)


class _LazyTileBins(TileBins):
    """TileBins materialised on first access (render() composites from row
    lists; the full CSR tile lists exist only if someone asks for them)."""

    def __init__(self, proj: ProjectedCloud, width: int, height: int):
        self._args = (proj, width, height)
        self._bins = None
        gx, gy = (width + TILE_SIZE - 1) // TILE_SIZE, (height + TILE_SIZE - 1) // TILE_SIZE
        self.grid_x, self.grid_y = gx, gy

    def _get(self) -> TileBins:
        if self._bins is None:
            self._bins = bin_and_sort(*self._args)
        return self._bins

    offsets = property(lambda self: self._get().offsets)
    entries = property(lambda self: self._get().entries)


@dataclass
class RenderOutput:
    """Forward buffers (rasterizer.py:132-145); proj/bins retained for backward."""

    color: torch.Tensor
    depth: torch.Tensor
    weight: torch.Tensor
    final_transmittance: torch.Tensor
    count: torch.Tensor
    mode: str
    color_clean: Optional[torch.Tensor] = None
    proj: Optional[ProjectedCloud] = None
    bins: Optional[TileBins] = None
    camera: Optional[Camera] = None
    last: Optional[torch.Tensor] = None          # per-pixel consumed list prefix
    attenuation_map: Optional[torch.Tensor] = None
    backscatter_map: Optional[torch.Tensor] = None
    rows: Optional[RowLists] = None               # row lists the forward composited from
    # backward context of the row-list path: the rows each tile staged (first
    # TILE_ROWS_CAP per tile) and how many were stored
    tile_rows: Optional[torch.Tensor] = None
    tile_nrows: Optional[torch.Tensor] = None
    # exact T >= 1e-4 decisions: scratch list of the pixels re-walked in float64
    # and its {count, ticket} pair (zero between calls)
    fix_pixels: Optional[torch.Tensor] = None
    fix_count: Optional[torch.Tensor] = None
    # compositing schedule (heaviest tiles first), kept by the engine's buffer sets
    tile_order: Optional[torch.Tensor] = None

    def c_struct(self) -> _lib.RasterOutC:
        cap = self.tile_rows.shape[1] if self.tile_rows is not None else 0
        return _lib.RasterOutC(_lib.ptr(self.color), _lib.ptr(self.color_clean),
                               _lib.ptr(self.depth), _lib.ptr(self.weight),
                               _lib.ptr(self.final_transmittance), _lib.ptr(self.count),
                               _lib.ptr(self.last), _lib.ptr(self.attenuation_map),
                               _lib.ptr(self.backscatter_map), _lib.ptr(self.tile_rows),
                               _lib.ptr(self.tile_nrows), cap, _lib.ptr(self.fix_pixels),
                               _lib.ptr(self.fix_count), _lib.ptr(self.tile_order))


# staged rows kept per tile for the backward (the consumed prefix is ~140 rows on
# average at 1M Gaussians 1080p; tiles that consumed more re-filter the row lists)
TILE_ROWS_CAP = 1024


def _alloc_output(H, W, dev, mode, medium_maps, tile_rows=True):
    f = dict(dtype=torch.float32, device=dev)
    out = RenderOutput(color=torch.empty(H, W, 3, **f), depth=torch.empty(H, W, **f),
                       weight=torch.empty(H, W, **f), final_transmittance=torch.empty(H, W, **f),
                       count=torch.empty(H, W, dtype=torch.int32, device=dev), mode=mode,
                       last=torch.empty(H, W, dtype=torch.int32, device=dev),
                       fix_pixels=torch.empty(H * W, dtype=torch.int32, device=dev),
                       fix_count=torch.zeros(3, dtype=torch.int32, device=dev))
    if tile_rows:
        tiles = ((H + TILE_SIZE - 1) // TILE_SIZE) * ((W + TILE_SIZE - 1) // TILE_SIZE)
        out.tile_rows = torch.empty(tiles, TILE_ROWS_CAP, dtype=torch.int32, device=dev)
        out.tile_nrows = torch.empty(tiles, dtype=torch.int32, device=dev)
    if mode == "underwater":
        out.color_clean = torch.empty(H, W, 3, **f)
        if medium_maps:
            out.attenuation_map = torch.empty(H, W, 3, **f)
            out.backscatter_map = torch.empty(H, W, 3, **f)
    return out


def composite(proj: ProjectedCloud, bins: TileBins, cam, medium: Optional[MediumParams] = None,
              mode: str = "clean", medium_maps: bool = False) -> RenderOutput:
    """Run the compositing kernel on existing projection + bins."""
    cam = Camera.from_any(cam)
    out = _alloc_output(cam.height, cam.width, proj.device, mode, medium_maps, tile_rows=False)
    pc, cc, oc = proj.c_struct(), cam.c_struct(), out.c_struct()
    med = _lib.ptr(medium.flat) if mode == "underwater" else 0
    _lib.call("uws_raster_fwd", ctypes.byref(pc), _lib.ptr(bins.offsets), _lib.ptr(bins.entries),
              ctypes.byref(cc), med, ctypes.byref(oc), _lib.stream_handle())
    out.proj, out.bins, out.camera = proj, bins, cam
    return out


def render(cloud: GaussianCloud, cam, medium: Optional[MediumParams] = None,
           mode: str = "clean", workers: int = 1, retain: bool = True,
           medium_maps: bool = False) -> RenderOutput:
    """Render a full frame (rasterizer.py:188-241).  ``workers`` is accepted
    for signature compatibility and ignored.  ``medium_maps=True``
    additionally returns the per-pixel attenuation exp(-B_d z) and
    backscatter B_inf (1 - exp(-B_b z)) images."""
    if mode not in ("clean", "underwater"):
        raise ValueError(f"unknown render mode {mode!r}")
    if mode == "underwater" and medium is None:
        raise ValueError("underwater mode requires medium parameters")
    cam = Camera.from_any(cam)
    proj = project_cloud(cloud, cam, with_geometry=False)
    rows = bin_rows(proj, cam.width, cam.height)
    # the per-tile staged rows are kept even when not retained: the float64
    # fix-up pass of the T >= 1e-4 decisions reads them
    out = _alloc_output(cam.height, cam.width, proj.device, mode, medium_maps)
    pc, cc, oc = proj.c_struct(), cam.c_struct(), out.c_struct()
    med = _lib.ptr(medium.flat) if mode == "underwater" else 0
    _lib.call("uws_raster_fwd_rows", ctypes.byref(pc), _lib.ptr(rows.row_start),
              _lib.ptr(rows.items), ctypes.byref(cc), med, ctypes.byref(oc),
              _lib.stream_handle())
    out.proj, out.rows, out.camera = proj, rows, cam
    # the reference's CSR tile lists, built only when accessed (same order and
    # indices as the filtered row lists)
    out.bins = _LazyTileBins(proj, cam.width, cam.height)
    if not retain:
        out.proj = None
        out.bins = None
        out.rows = None
        out.tile_rows = out.tile_nrows = None
    return out


def render_naive(cloud: GaussianCloud, cam, medium: Optional[MediumParams] = None,
                 mode: str = "clean", row_chunk: int = 16) -> RenderOutput:
    """Every visible Gaussian against every pixel, no tile culling
    (rasterizer.py:254-296): the global (depth, source) order of all K visible
    rows is each tile's list, composited by the same device kernel as the tiled
    path (uws_raster_fwd + the float64 transmittance fix-up).  Tiled == naive
    therefore checks that binning drops no contributor.  Lists hold K entries
    per tile, so this is for oracle-sized scenes as in the reference;
    ``row_chunk`` is accepted and ignored."""
    if mode not in ("clean", "underwater"):
        raise ValueError(f"unknown render mode {mode!r}")
    if mode == "underwater" and medium is None:
        raise ValueError("underwater mode requires medium parameters")
    cam = Camera.from_any(cam)
    proj = project_cloud(cloud, cam, with_geometry=False)
    k = proj.k
    gx, gy = cam.grid
    # rows are in ascending source order: a stable sort by depth is the
    # reference's lexsort((source_index, depth))
    order = torch.sort(proj.depth, stable=True).indices.to(torch.int32)
    entries = order.repeat(gx * gy) if k else torch.zeros(1, dtype=torch.int32, device=proj.device)
    offsets = (torch.arange(gx * gy + 1, device=proj.device, dtype=torch.int64) * k).to(torch.int32)
    out = composite(proj, TileBins(gx, gy, offsets, entries), cam, medium, mode)
    out.proj = out.bins = None
    return out


def alpha_at(p, opacity_logit: float, pixel_center) -> float:
    """Opacity of one footprint at a pixel centre, float64 (rasterizer.py:88-101):
    sigmoid(logit) exp(-d^T cov^-1 d / 2), clamped at 0.99, 0 below 1/255.
    Scalar host helper; the kernels evaluate the same expression per pair."""
    d = np.asarray(pixel_center, dtype=np.float64) - np.asarray(p.mean2d, dtype=np.float64)
    q = float(d @ np.linalg.inv(np.asarray(p.cov2d, dtype=np.float64)) @ d)
    a = min(float(1.0 / (1.0 + np.exp(-opacity_logit)) * np.exp(-0.5 * q)), ALPHA_CLAMP)
    return a if a >= ALPHA_FLOOR else 0.0


def composite_pixel(contributors, pixel, far: float):
    """Front-to-back blend of one pixel's depth-sorted (Projected2D, logit, rgb)
    list (rasterizer.py:104-129); returns (color, depth, weight, T_final, count).
    Scalar host helper mirroring the compositing kernel's rules."""
    color = np.zeros(3)
    weight = depth_num = 0.0
    t = 1.0
    count = 0
    for p, logit, rgb in contributors:
        if t < T_EARLY_STOP:
            break
        a = alpha_at(p, logit, pixel)
        if a == 0.0:
            continue
        w = a * t
        color += w * np.asarray(rgb, dtype=np.float64)
        depth_num += w * p.depth
        weight += w
        t *= 1.0 - a
        count += 1
    return color, (depth_num / weight if weight > WEIGHT_EPS else far), weight, t, count


def apply_water(color_clean: torch.Tensor, depth_raw: torch.Tensor,
                medium: MediumParams) -> torch.Tensor:
    """Attenuate a clean render and add backscatter (rasterizer.py:244-251).

    Utility outside the hot path (the render kernel fuses this epilogue)."""
    dev = medium.flat.device
    color_clean = torch.as_tensor(np.asarray(color_clean) if not isinstance(
        color_clean, torch.Tensor) else color_clean).to(dev)
    depth_raw = torch.as_tensor(np.asarray(depth_raw) if not isinstance(
        depth_raw, torch.Tensor) else depth_raw).to(dev)
    z = logistic_remap(depth_raw)[..., None]
    att = torch.exp(-medium.attenuation.double() * z)
    bsc = medium.water_color.double() * (1.0 - torch.exp(-medium.backscatter.double() * z))
    return color_clean.double() * att + bsc
