"""The engine's NCCL path on the GPU (it had only run with gloo on CPU).

One B200 is available, so the group has one rank; the engine is told it has two
(``engine.world = 2``) so every step takes the multi-GPU branch: the NCCL
all-reduce of the flat gradient buffer -- single, or split into the medium/skip
head and ALLREDUCE_PARTS asynchronous parts with the cloud update launched range
by range behind each part's wait.  On one rank the sum is the identity, so every
variant must equal the engine without a process group bit for bit: this checks
the collective calls, the waits and the ordering of the range-wise Adam launches
against the reductions, on the device.  The engines run the deterministic backward
(the default one merges tiles with float atomics in varying order).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2411_19588_b200 as uw
from golden_util import load
from gpu_util import device_scene, np_

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    if not dist.is_available() or not dist.is_nccl_available():
        pytest.skip("NCCL backend not available")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def _run(parts, use_dist, steps=4):
    from paper_2411_19588_b200.engine import StepEngine
    g = load("survey2k")
    cloud, cam, medium = device_scene(g)
    state = uw.TrainState(cloud, medium, iteration=1)
    eng = StepEngine(state, cam.width, cam.height, uw.OptimConfig())
    eng.deterministic = True               # bit-identical gradients: exact comparison
    if use_dist:
        assert eng.dist is not None
        eng.world = 2                      # take the multi-GPU branch on the one-rank group
    else:
        eng.dist = None
    eng.ALLREDUCE_PARTS = parts
    gt = torch.as_tensor(g.gt, dtype=torch.float32).cuda()
    stats = []
    for _ in range(steps):
        stats.append(eng.step([(cam, gt)]))
        state.iteration += 1
    torch.cuda.synchronize()
    return [np_(t).copy() for t in (state.cloud.flat, state.exp_avg, state.exp_avg_sq,
                                    state.grad_accum, state.obs_count, state.medium.flat)], stats


@pytest.mark.parametrize("parts", [1, 4])
def test_nccl_allreduce_paths_equal_single_process(nccl_group, parts):
    ref, ref_stats = _run(1, use_dist=False)
    got, stats = _run(parts, use_dist=True)
    for a, b in zip(ref, got):
        np.testing.assert_array_equal(a, b)
    assert all(not s.skipped for s in stats)
    assert [s.total for s in stats] == [s.total for s in ref_stats]


def test_engine_deterministic_steps_bit_identical():
    """StepEngine(deterministic) gives bit-identical trajectories run to run, and the
    same values as the default engine to float32 accumulation order."""
    a, _ = _run(1, use_dist=False)
    b, _ = _run(1, use_dist=False)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
