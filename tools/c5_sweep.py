"""C5 render-only sweep: N in {0.1, 0.5, 1, 2, 5}e6 Gaussians at 3840x2160,
color + depth (+ weight, T_final) through the engine's queued frame stream, one B200.

    python tools/c5_sweep.py [--out profiles/r02/c5_sweep.txt]

Same generator, camera and medium as bench.py; CUDA-event timing over 20 queued frames after
the frame sets are warm; SM clock sampled with NVML during the timed frames.  Also reports the
workload statistics of one frame (K visible, S row items) next to the FPS."""
import argparse
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2411_19588_b200 as uw  # noqa: E402


def sm_clock_sampler(stop, out):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        while not stop.is_set():
            out.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.005)
    except Exception:  # no NVML: no clock record
        pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--frames", type=int, default=20)
    args = ap.parse_args()
    W, H = 3840, 2160
    lines = [f"C5 render-only sweep, {W}x{H}, underwater color + depth, frame stream "
             f"({torch.cuda.get_device_name(0)})"]
    for n in (100_000, 500_000, 1_000_000, 2_000_000, 5_000_000):
        host = bench.synthetic_cloud(n)
        cloud = uw.GaussianCloud(**host)
        st = uw.TrainState(cloud, uw.MediumParams(**bench.MEDIUM), iteration=1)
        eng = uw.StepEngine(st, W, H, uw.OptimConfig())
        cam = uw.Camera.look_at(bench.view_eye(0), (0, 0, 12), width=W, height=H, fx=1.2 * W,
                                fy=1.2 * W)
        for _ in range(6):  # every frame set allocated and warm
            eng.render_async(cam)
        eng.render_flush()
        torch.cuda.synchronize()
        clocks, stop = [], threading.Event()
        th = threading.Thread(target=sm_clock_sampler, args=(stop, clocks))
        th.start()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.frames):
            eng.render_async(cam)
        eng.render_flush()
        f1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = f0.elapsed_time(f1) / args.frames
        out = uw.render(cloud, cam, uw.MediumParams(**bench.MEDIUM), "underwater")
        k = len(out.proj) if out.proj is not None else -1
        clk = sorted(clocks)[len(clocks) // 2] if clocks else None
        lines.append(f"N={n/1e6:.1f}M: {ms:.3f} ms/frame = {1000.0 / ms:.0f} FPS "
                     f"({W * H / ms / 1e3:.0f} Mpix/s), K={k}, SM clock median {clk} MHz, "
                     f"peak mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB")
        print(lines[-1], flush=True)
        del eng, st, cloud, out
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
    if args.out:
        with open(args.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
