import sys, torch
sys.path.insert(0, '.')
import bench, paper_2411_19588_b200 as uw
n, W, H = 5_000_000, 3840, 2160
cloud = uw.GaussianCloud(**bench.synthetic_cloud(n))
st = uw.TrainState(cloud, uw.MediumParams(**bench.MEDIUM), iteration=1)
eng = uw.StepEngine(st, W, H, uw.OptimConfig())
cam = uw.Camera.look_at(bench.view_eye(0), (0, 0, 12), width=W, height=H, fx=1.2 * W, fy=1.2 * W)
for _ in range(3): eng.render(cam)
torch.cuda.synchronize()
