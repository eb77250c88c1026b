"""Kernel timeline of a few pipelined C3 training steps (torch.profiler / CUPTI):
per-kernel device durations and the idle gaps between consecutive kernels.

    python tools/kernel_gaps.py [steps]
"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2411_19588_b200 as uw  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
cloud = uw.GaussianCloud(**bench.synthetic_cloud(bench.N_GAUSS))
state = uw.TrainState(cloud, uw.MediumParams(**bench.MEDIUM), iteration=1)
tr = uw.ViewShardedTrainer(state, uw.OptimConfig(), bench.W, bench.H)
cam = uw.Camera.look_at(bench.view_eye(0), (0, 0, 12), width=bench.W, height=bench.H,
                        fx=1.2 * bench.W, fy=1.2 * bench.W)
gt = torch.from_numpy(bench.gt_image(0)).to(dev)
for _ in range(5):
    tr.step_async([(cam, gt)], sharded=True)
    state.iteration += 1
tr.flush()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        tr.step_async([(cam, gt)], sharded=True)
        state.iteration += 1
    tr.flush()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
busy = 0.0
gaps = []
prev_end = None
for e in ev:
    s, d = e.time_range.start, e.time_range.end
    gap = (s - prev_end) if prev_end is not None else 0.0
    gaps.append(gap)
    busy += d - s
    print(f"{(s - t0):9.1f} us  dur {d - s:8.1f}  gap {gap:6.1f}  {e.name[:70]}")
    prev_end = max(prev_end or d, d)
span = ev[-1].time_range.end - t0
print(f"span {span:.1f} us, busy {busy:.1f} us, idle {span - busy:.1f} us over {steps} steps, "
      f"{len(ev)} device ops")
