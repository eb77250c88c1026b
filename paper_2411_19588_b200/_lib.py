"""ctypes binding of the sm_100a C-ABI library (include/uwsplat_b200.h).

The library is built in-tree (``make`` / ``__graft_entry__.build()``) as
``paper_2411_19588_b200/libuwsplat_b200.so``.  There is no fallback: if the
library is missing, every hot-path call raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, c_char_p, c_double, c_float, c_int, c_int16, c_int32, c_int64,
                    c_size_t, c_void_p)

import torch

from .errors import DataError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libuwsplat_b200.so")

UWS_OK, UWS_EINVAL, UWS_ECUDA, UWS_ECAPACITY = 0, 1, 2, 3


class CameraC(ctypes.Structure):
    _fields_ = [("width", c_int32), ("height", c_int32), ("fx", c_double), ("fy", c_double),
                ("cx", c_double), ("cy", c_double), ("R", c_double * 9), ("t", c_double * 3),
                ("near_plane", c_double), ("far_plane", c_double)]


class CloudC(ctypes.Structure):
    _fields_ = [("positions", c_void_p), ("log_scales", c_void_p), ("rotations", c_void_p),
                ("sh_coeffs", c_void_p), ("opacity_logits", c_void_p), ("n", c_int64)]


class ProjectedC(ctypes.Structure):
    _fields_ = [("source_index", c_void_p), ("splat", c_void_p), ("exact", c_void_p),
                ("depth", c_void_p), ("rect", c_void_p), ("cov2d", c_void_p),
                ("radius", c_void_p), ("num_visible", c_void_p), ("depth_range", c_void_p)]


class RasterOutC(ctypes.Structure):
    _fields_ = [("color", c_void_p), ("color_clean", c_void_p), ("depth", c_void_p),
                ("weight", c_void_p), ("final_T", c_void_p), ("count", c_void_p),
                ("last", c_void_p), ("attenuation", c_void_p), ("backscatter", c_void_p),
                ("tile_rows", c_void_p), ("tile_nrows", c_void_p), ("tile_rows_cap", c_int32),
                ("fix_pixels", c_void_p), ("fix_count", c_void_p), ("tile_order", c_void_p)]


class AdamParamsC(ctypes.Structure):
    _fields_ = [("lr", c_double * 8), ("bias1", c_double * 8), ("bias2", c_double * 8),
                ("inv_bias1", c_double * 8), ("inv_bias2", c_double * 8),
                ("beta1", c_double), ("beta2", c_double), ("one_minus_beta1", c_double),
                ("one_minus_beta2", c_double), ("eps", c_double)]


class BackscatterCfgC(ctypes.Structure):
    _fields_ = [("p_dark", c_double), ("intervals_num", c_int32), ("resized_height", c_int32),
                ("edges_num", c_int32), ("pad", c_int32)]


_SIGS = {
    "uws_version": (c_char_p, []),
    "uws_last_error": (c_char_p, []),
    "uws_kernel_launches": (ctypes.c_uint64, []),
    "uws_preprocess_workspace_size": (c_int, [c_int64, POINTER(c_size_t)]),
    "uws_preprocess_fwd": (c_int, [POINTER(CloudC), POINTER(CameraC), POINTER(ProjectedC),
                                   c_void_p, c_size_t, c_void_p]),
    "uws_bin_workspace_size": (c_int, [c_int64, c_int64, c_int32, c_int32, POINTER(c_size_t),
                                       POINTER(c_size_t)]),
    "uws_bin_count": (c_int, [POINTER(ProjectedC), c_int64, POINTER(CameraC), c_void_p,
                              c_void_p, c_size_t, c_void_p]),
    "uws_bin_emit": (c_int, [POINTER(ProjectedC), c_int64, c_int64, c_int64, POINTER(CameraC),
                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                             c_size_t, c_void_p, c_size_t, c_void_p]),
    "uws_bin_rows": (c_int, [POINTER(ProjectedC), c_int64, c_int64, POINTER(CameraC), c_void_p,
                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                             c_void_p]),
    "uws_raster_fwd": (c_int, [POINTER(ProjectedC), c_void_p, c_void_p, POINTER(CameraC),
                               c_void_p, POINTER(RasterOutC), c_void_p]),
    "uws_tile_order": (c_int, [c_void_p, c_int32, c_void_p, c_void_p]),
    "uws_raster_fwd_rows": (c_int, [POINTER(ProjectedC), c_void_p, c_void_p, POINTER(CameraC),
                                    c_void_p, POINTER(RasterOutC), c_void_p]),
    "uws_loss_workspace_size": (c_int, [c_int32, c_int32, c_int32, POINTER(c_size_t)]),
    "uws_loss_fwd_bwd": (c_int, [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p,
                                 c_int32, c_double, c_double, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_size_t, c_void_p]),
    "uws_raster_bwd": (c_int, [POINTER(ProjectedC), c_void_p, c_void_p, POINTER(CameraC),
                               c_void_p, POINTER(RasterOutC), c_void_p, c_void_p, c_void_p,
                               c_void_p]),
    "uws_raster_bwd_rows": (c_int, [POINTER(ProjectedC), c_void_p, c_void_p, POINTER(CameraC),
                                    c_void_p, POINTER(RasterOutC), c_void_p, c_void_p, c_void_p,
                                    c_void_p]),
    "uws_raster_bwd_det_prefix": (c_int, [POINTER(CameraC), POINTER(RasterOutC), c_void_p,
                                          c_void_p, c_void_p]),
    "uws_raster_bwd_det_workspace_size": (c_int, [c_int32, c_int64, c_int64, POINTER(c_size_t)]),
    "uws_raster_bwd_det": (c_int, [POINTER(ProjectedC), c_void_p, c_void_p, c_void_p, c_void_p,
                                   POINTER(CameraC), c_void_p, POINTER(RasterOutC), c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p,
                                   c_size_t, c_void_p]),
    "uws_preprocess_bwd": (c_int, [POINTER(CloudC), POINTER(CameraC), POINTER(ProjectedC),
                                   c_int64, c_void_p, c_void_p, c_void_p, c_int32, c_double,
                                   c_void_p, c_void_p, c_int32, c_void_p]),
    "uws_adam_step": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                              c_void_p, c_void_p, c_void_p, POINTER(AdamParamsC), c_void_p,
                              c_void_p, c_void_p, c_int32, c_void_p]),
    "uws_adam_step_range": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                    POINTER(AdamParamsC), c_void_p, c_void_p, c_void_p, c_int32,
                                    c_int64, c_int64, c_void_p]),
    "uws_densify_workspace_size": (c_int, [c_int64, POINTER(c_size_t)]),
    "uws_densify_classify": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_double, c_double,
                                     c_double, c_void_p, c_void_p, c_size_t, c_void_p]),
    "uws_densify_apply": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_size_t,
                                  c_void_p, c_double, c_int64, c_int64, c_int64, c_void_p,
                                  c_void_p, c_void_p, c_void_p]),
    "uws_reset_opacities": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_float, c_void_p]),
    "uws_backscatter_workspace_size": (c_int, [c_int32, c_int32, POINTER(BackscatterCfgC),
                                               POINTER(c_size_t)]),
    "uws_estimate_backscatter": (c_int, [c_void_p, c_void_p, c_int32, c_int32, c_int32,
                                         POINTER(BackscatterCfgC),
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                         c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"CUDA library {path} not found: build it with `make` or __graft_entry__.build(); "
            "this package has no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name, *args):
    """Invoke an entry point and map its status to the reference's exceptions."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != UWS_OK:
        msg = lib.uws_last_error().decode(errors="replace")
        if rc == UWS_EINVAL:
            if "smaller than" in msg or "shape" in msg:
                raise DataError(msg)
            raise ValueError(msg)
        raise RuntimeError(f"{name} failed ({rc}): {msg}")


def ptr(t) -> int:
    """Raw device pointer of a CUDA tensor (0 for None)."""
    if t is None:
        return 0
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return t.data_ptr()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def size_out():
    return c_size_t(0)
