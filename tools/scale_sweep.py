import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import bench, paper_2411_19588_b200 as uw
for n, (W, H) in ((1_000_000, (1920, 1080)), (3_000_000, (1920, 1080)), (1_000_000, (3840, 2160)),
                  (5_000_000, (3840, 2160))):
    host = bench.synthetic_cloud(n)
    cloud = uw.GaussianCloud(**host)
    st = uw.TrainState(cloud, uw.MediumParams(**bench.MEDIUM), iteration=1)
    eng = uw.StepEngine(st, W, H, uw.OptimConfig())
    cam = uw.Camera.look_at(bench.view_eye(0), (0, 0, 12), width=W, height=H, fx=1.2 * W, fy=1.2 * W)
    gt = torch.rand(H, W, 3, device='cuda')
    r = eng.step([(cam, gt)]); st.iteration += 1
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(5):
        eng.step_async([(cam, gt)]); st.iteration += 1
    last = eng.flush()
    t1.record(); torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 5
    f0 = torch.cuda.Event(enable_timing=True); f1 = torch.cuda.Event(enable_timing=True)
    for _ in range(4):      # both frame sets allocated and warm
        eng.render_async(cam)
    eng.render_flush(); torch.cuda.synchronize(); f0.record()
    for _ in range(10): eng.render_async(cam)
    eng.render_flush()
    f1.record(); torch.cuda.synchronize()
    print(f"N={n} {W}x{H}: step {ms:.3f} ms ({W*H/ms/1e3:.0f} Mpix/s) reruns={r.reruns} skipped={last.skipped} "
          f"loss={last.total:.4f} render {f0.elapsed_time(f1)/10:.3f} ms, mem {torch.cuda.max_memory_allocated()/1e9:.1f} GB", flush=True)
    del eng, st, cloud; torch.cuda.empty_cache(); torch.cuda.reset_peak_memory_stats()
