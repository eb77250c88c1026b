"""Host time per pipelined training step (StepEngine.step_async through the trainer) vs
the device time per step, at C3: is the launch path the bottleneck?
usage (GPU box): python tools/host_overhead.py"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2411_19588_b200 as uw

cloud = uw.GaussianCloud(**bench.synthetic_cloud(bench.N_GAUSS))
med = uw.MediumParams(**bench.MEDIUM)
state = uw.TrainState(cloud, med, iteration=1)
cam = uw.Camera.look_at(bench.view_eye(0), (0, 0, 12), width=bench.W, height=bench.H,
                        fx=1.2 * bench.W, fy=1.2 * bench.W)
gt = torch.from_numpy(bench.gt_image()).cuda()
eng = uw.StepEngine(state, bench.W, bench.H, uw.OptimConfig())
for _ in range(10):
    eng.step_async([(cam, gt)])
eng.flush()
torch.cuda.synchronize()
n = 50
host = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for _ in range(n):
    a = time.perf_counter()
    eng.step_async([(cam, gt)])
    host.append(time.perf_counter() - a)
t1 = time.perf_counter()
eng.flush()
e1.record()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host per step_async: median %.3f ms, mean %.3f ms (loop %.3f ms/step); device %.3f ms/step; wall %.3f ms/step"
      % (1e3 * np.median(host), 1e3 * np.mean(host), 1e3 * (t1 - t0) / n, e0.elapsed_time(e1) / n,
         1e3 * (t2 - t0) / n))
# pure host launch cost: the GPU idle before each call (step i-1's record is ready)
pure = []
for _ in range(20):
    torch.cuda.synchronize()
    a = time.perf_counter()
    eng.step_async([(cam, gt)])
    pure.append(time.perf_counter() - a)
eng.flush()
print("host launch cost per step (GPU idle before the call): median %.3f ms" % (1e3 * np.median(pure)))
