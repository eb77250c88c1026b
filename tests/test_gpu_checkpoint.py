"""SPLASH01 checkpoints from CUDA tensors (GPU)."""

import os

import pytest
import torch

import paper_2411_19588_b200 as uw
from golden_util import load
from gpu_util import device_scene

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(__file__), "golden")


def test_reference_checkpoint_round_trip_on_device():
    with open(os.path.join(HERE, "ckpt_guided.bin"), "rb") as f:
        data = f.read()
    st = uw.load_checkpoint(data)
    assert st.cloud.flat.is_cuda
    assert uw.save_checkpoint(st) == data


def test_checkpoint_after_device_steps_round_trips():
    g = load("survey2k")
    cloud, cam, medium = device_scene(g)
    st = uw.TrainState(cloud, medium, iteration=1)
    eng = uw.StepEngine(st, cam.width, cam.height, uw.OptimConfig())
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    for _ in range(2):
        eng.step([(cam, gt)])
        st.iteration += 1
    data = uw.save_checkpoint(st)
    back = uw.load_checkpoint(data)
    assert torch.equal(back.cloud.flat, st.cloud.flat)
    assert torch.equal(back.exp_avg, st.exp_avg) and torch.equal(back.exp_avg_sq, st.exp_avg_sq)
    assert torch.equal(back.obs_count, st.obs_count)
    assert back.iteration == st.iteration and back.adam["positions"].step == 2
    assert uw.save_checkpoint(back) == data
