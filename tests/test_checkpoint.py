"""SPLASH01 checkpoints: byte-exact round trip of reference-written files
(tests/golden/make_checkpoint.py) and the reference's error behaviour
(scene.py:320-371).  CPU tensors here; the same code on CUDA in the GPU test."""

import os
import struct

import numpy as np
import pytest
import torch

import paper_2411_19588_b200 as uw
from paper_2411_19588_b200.errors import CheckpointError

HERE = os.path.join(os.path.dirname(__file__), "golden")


def _data(name):
    with open(os.path.join(HERE, name + ".bin"), "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", ["ckpt_guided", "ckpt_plain"])
def test_reference_checkpoint_round_trip(name):
    data = _data(name)
    st = uw.load_checkpoint(data, device="cpu")
    assert uw.save_checkpoint(st) == data
    # independent parse of the header and the first/last blocks
    version, flags, n, k, it = struct.unpack("<IIIIQ", data[8:32])
    assert (version, k, it) == (1, 1, st.iteration) and n == len(st.cloud)
    assert bool(flags & 1) == st.medium.has_guidance
    pos = np.frombuffer(data[32:32 + 12 * n], dtype="<f4").reshape(n, 3)
    np.testing.assert_array_equal(st.cloud.positions.numpy(), pos)
    obs = np.frombuffer(data[-4 * n:], dtype="<u4")
    np.testing.assert_array_equal(st.obs_count.numpy(), obs.astype(np.int32))
    assert all(slot.step == 2 for slot in st.adam.values())


def test_checkpoint_errors():
    data = _data("ckpt_guided")
    with pytest.raises(CheckpointError, match="truncated"):
        uw.load_checkpoint(data[:-1], device="cpu")
    with pytest.raises(CheckpointError, match="magic"):
        uw.load_checkpoint(b"SPLASH02" + data[8:], device="cpu")
    with pytest.raises(CheckpointError, match="version"):
        uw.load_checkpoint(data[:8] + struct.pack("<I", 2) + data[12:], device="cpu")
    with pytest.raises(CheckpointError, match="trailing"):
        uw.load_checkpoint(data + b"\0", device="cpu")
    with pytest.raises(CheckpointError):
        uw.load_checkpoint(b"", device="cpu")
    assert issubclass(CheckpointError, uw.DataError)
