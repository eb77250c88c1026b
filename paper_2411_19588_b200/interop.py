"""numpy interop at the drop-in boundary.

The reference's callers (pipeline.train / evaluate / render_novel, dataset,
fixtures, cli -- reference pipeline.py:178-290, dataset.py:392-412,
fixtures.py:47-71, cli.py:198-227) treat what ``render`` /
``backward_render`` / ``TrainState`` hand them as numpy arrays:
``buf.mean2d_grad_norm[buf.observed].astype(np.float32)`` (pipeline.py:191),
``np.clip(out.color, 0, 1)`` (pipeline.py:259), ``write_pfm(path,
logistic_remap(out.depth))`` (pipeline.py:287), ``jostle.positions +
rng.normal(...)`` (fixtures.py:64-67).  :class:`DeviceArray` is a
``torch.Tensor`` subclass that keeps the data on the GPU and adds the numpy
protocol those call sites use:

* ``astype(dtype)`` -- a device cast (numpy dtype names accepted);
* torch operators with numpy operands move the operand to the tensor's
  device (``DeviceArray + ndarray`` stays on the GPU);
* numpy functions and ufuncs applied to a DeviceArray (``np.clip``,
  ``np.exp``, ``np.asarray``, ``ndarray + DeviceArray``) see it through
  ``__array__``: one explicit device-to-host copy, then host numpy -- the
  caller asked for a host computation.

Only the drop-in layer (dropin.py) returns DeviceArrays; the package's own
API and the training engine use plain tensors.
"""

from __future__ import annotations

import numpy as np
import torch

_NP_TO_TORCH = {
    np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
    np.dtype(np.float16): torch.float16, np.dtype(np.int64): torch.int64,
    np.dtype(np.int32): torch.int32, np.dtype(np.int16): torch.int16,
    np.dtype(np.int8): torch.int8, np.dtype(np.uint8): torch.uint8,
    np.dtype(np.bool_): torch.bool,
}


def torch_dtype(dtype) -> torch.dtype:
    if isinstance(dtype, torch.dtype):
        return dtype
    try:
        return _NP_TO_TORCH[np.dtype(dtype)]
    except (KeyError, TypeError):
        raise TypeError(f"no device dtype for {dtype!r}") from None


def _has_numpy(args) -> bool:
    for a in args:
        if isinstance(a, (np.ndarray, np.generic)):
            return True
        if isinstance(a, (list, tuple)) and _has_numpy(a):
            return True
    return False


def _device_of(args):
    for a in args:
        if isinstance(a, torch.Tensor):
            with torch._C.DisableTorchFunctionSubclass():
                return a.device
        if isinstance(a, (list, tuple)):
            d = _device_of(a)
            if d is not None:
                return d
    return None


def _to_device(x, dev):
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    if isinstance(x, np.generic):
        return x.item()
    if isinstance(x, (list, tuple)) and any(isinstance(v, (np.ndarray, np.generic)) for v in x):
        return type(x)(_to_device(v, dev) for v in x)
    return x


def _to_host(x):
    if isinstance(x, DeviceArray):
        return x.numpy_host()
    if isinstance(x, (list, tuple)):
        return type(x)(_to_host(v) for v in x)
    if isinstance(x, dict):
        return {k: _to_host(v) for k, v in x.items()}
    return x


class DeviceArray(torch.Tensor):
    """A device tensor that numpy-style caller code can use (see module doc)."""

    __array_priority__ = 1000

    @classmethod
    def __torch_function__(cls, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        if _has_numpy(args) or _has_numpy(tuple(kwargs.values())):
            dev = _device_of(args)
            args = tuple(_to_device(a, dev) for a in args)
            kwargs = {k: _to_device(v, dev) for k, v in kwargs.items()}
        return super().__torch_function__(func, types, args, kwargs)

    # -- numpy protocol --------------------------------------------------------
    def numpy_host(self) -> np.ndarray:
        """Device-to-host copy as a numpy array."""
        return torch.Tensor.numpy(self.detach().cpu().as_subclass(torch.Tensor))

    def __array__(self, dtype=None, copy=None):
        a = self.numpy_host()
        return a if dtype is None else a.astype(dtype, copy=False)

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        inputs = _to_host(inputs)
        if "out" in kwargs:
            kwargs["out"] = _to_host(kwargs["out"])
        return getattr(ufunc, method)(*inputs, **kwargs)

    def __array_function__(self, func, types, args, kwargs):
        return func(*_to_host(args), **_to_host(kwargs))

    def astype(self, dtype, copy: bool = True):
        t = self.to(torch_dtype(dtype))
        return t.clone() if (copy and t.data_ptr() == self.data_ptr()) else t

    def copy(self):
        return self.clone()


def as_ref(t):
    """View a tensor as a DeviceArray (no copy); None and non-tensors pass through."""
    if isinstance(t, torch.Tensor) and not isinstance(t, DeviceArray):
        return t.as_subclass(DeviceArray)
    return t


def plain(t):
    """The plain-tensor view of a DeviceArray (no copy)."""
    if isinstance(t, DeviceArray):
        return t.as_subclass(torch.Tensor)
    return t
