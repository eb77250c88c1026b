"""SPLASH01 checkpoints straight from / into device tensors.

Byte-compatible with the reference's ``save_checkpoint`` / ``load_checkpoint``
(scene.py:284-371): magic ``SPLASH01``, ``<IIIIQ`` header (version 1, flags bit
0 = guidance present, n, SH coefficients per Gaussian, iteration), then
little-endian float32 blocks in field order -- the five cloud tensors, the 3x3
medium block, the optional 2x3 guidance block, per learnable tensor a ``<Q``
Adam step followed by its m and v, the densification statistics
(``grad_accum`` float32, ``obs_count`` uint32).

On the device the cloud is one flat buffer already in checkpoint field order
and the Adam moments live in two flat buffers, so saving is a single gather
on the GPU plus one device-to-host copy, and loading one host-to-device copy
per buffer.
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .errors import CheckpointError
from .scene import (CLOUD_FIELDS, FIELD_WIDTH, MEDIUM_FIELDS, GaussianCloud, MediumParams,
                    TrainState)

MAGIC = b"SPLASH01"          # scene.py:28
VERSION = 1                  # scene.py:29
_HEADER = struct.Struct("<IIIIQ")
_STEP = struct.Struct("<Q")


def save_checkpoint(state: TrainState) -> bytes:
    """Serialize a device-resident TrainState (reference scene.py:288-317)."""
    cloud, medium = state.cloud, state.medium
    n = len(cloud)
    k = cloud.num_sh_coeffs
    guided = medium.has_guidance
    # one float32 gather on the device in file order (the step words go in between)
    parts = [cloud.flat, medium.flat[0:9]]
    if guided:
        parts.append(medium.flat[9:15])
    for name in CLOUD_FIELDS + MEDIUM_FIELDS:
        slot = state.adam[name]
        parts += [slot.m.reshape(-1), slot.v.reshape(-1)]
    parts.append(state.grad_accum.reshape(-1))
    if int(n) and bool((state.obs_count < 0).any()):
        raise CheckpointError("negative observation count cannot be stored as uint32")
    parts.append(state.obs_count.reshape(-1).to(torch.int32).view(torch.float32))
    blob = torch.cat([p.reshape(-1).to(torch.float32) if p.dtype != torch.float32 else
                      p.reshape(-1) for p in parts]).cpu().numpy().view(np.uint8)

    out = bytearray()
    out += MAGIC
    out += _HEADER.pack(VERSION, 1 if guided else 0, n, k, int(state.iteration))
    pos = 0

    def take(count):
        nonlocal pos
        b = blob[pos:pos + 4 * count]
        pos += 4 * count
        return b.tobytes()

    out += take(14 * n)
    out += take(9)
    if guided:
        out += take(6)
    for name in CLOUD_FIELDS + MEDIUM_FIELDS:
        slot = state.adam[name]
        width = FIELD_WIDTH[name] * n if name in CLOUD_FIELDS else 3
        out += _STEP.pack(int(slot.step))
        out += take(width)
        out += take(width)
    out += take(n)
    out += take(n)
    return bytes(out)


class _Reader:
    def __init__(self, data: bytes):
        self.data = memoryview(data)
        self.pos = 0

    def take(self, nbytes: int) -> memoryview:
        if self.pos + nbytes > len(self.data):
            raise CheckpointError("truncated checkpoint")
        out = self.data[self.pos:self.pos + nbytes]
        self.pos += nbytes
        return out

    def f32(self, count: int) -> np.ndarray:
        return np.frombuffer(self.take(4 * count), dtype="<f4").astype(np.float32)


def load_checkpoint(data: bytes, device=None) -> TrainState:
    """Parse checkpoint bytes into a device-resident TrainState
    (reference scene.py:338-371); raises CheckpointError on any defect and
    builds nothing until the whole buffer has been validated."""
    r = _Reader(bytes(data))
    if bytes(r.take(len(MAGIC))) != MAGIC:
        raise CheckpointError("bad magic: not a checkpoint file")
    version, flags, n, k, iteration = _HEADER.unpack(r.take(_HEADER.size))
    if version != VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version}")
    if k != 1:
        raise CheckpointError(f"{k} SH coefficients per Gaussian; only degree 0 (1) exists")
    arrays = {}
    for name in CLOUD_FIELDS:
        arrays[name] = r.f32(FIELD_WIDTH[name] * n)
    medium_block = r.f32(9).reshape(3, 3)
    guide = r.f32(6).reshape(2, 3) if flags & 1 else None
    slots = {}
    for name in CLOUD_FIELDS + MEDIUM_FIELDS:
        (step,) = _STEP.unpack(r.take(_STEP.size))
        width = FIELD_WIDTH[name] * n if name in CLOUD_FIELDS else 3
        slots[name] = (step, r.f32(width), r.f32(width))
    grad_accum = r.f32(n)
    obs = np.frombuffer(r.take(4 * n), dtype="<u4")
    if r.pos != len(r.data):
        raise CheckpointError(f"{len(r.data) - r.pos} trailing bytes in checkpoint")
    if n and int(obs.max()) > np.iinfo(np.int32).max:
        raise CheckpointError("observation count exceeds the int32 device counter")

    shapes = {"positions": (n, 3), "log_scales": (n, 3), "rotations": (n, 4),
              "sh_coeffs": (n, 1, 3), "opacity_logits": (n,)}
    cloud = GaussianCloud(**{f: arrays[f].reshape(shapes[f]) for f in CLOUD_FIELDS},
                          device=device)
    medium = MediumParams(medium_block[0], medium_block[1], medium_block[2],
                          None if guide is None else guide[0],
                          None if guide is None else guide[1], device=cloud.device)
    state = TrainState(cloud, medium, iteration=int(iteration))
    for name, (step, m, v) in slots.items():
        slot = state.adam[name]
        slot.step = int(step)
        slot.m.copy_(torch.from_numpy(m).reshape(slot.m.shape))
        slot.v.copy_(torch.from_numpy(v).reshape(slot.v.shape))
    state.grad_accum.copy_(torch.from_numpy(grad_accum))
    state.obs_count.copy_(torch.from_numpy(obs.astype(np.int64)).to(torch.int32))
    return state
