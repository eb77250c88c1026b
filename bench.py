"""Benchmark of the underwater-3DGS training step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[2], the config the headline metric is quoted
on): 1M Gaussians, 1920x1080, one full training step = render (underwater)
+ L1/D-SSIM loss + backward + Adam, synthetic scene from the survey generator
(SURVEY §8d), random-init parameters, U(0,1) ground truth.  With N GPUs
(torchrun, one process per GPU) every rank renders its own view of the
replicated 1M-Gaussian cloud, gradients are summed with one NCCL all-reduce
and every rank applies the same Adam step: weak scaling, value = all ranks'
pixels / max-over-ranks step time.

``--impl reference`` times the reference's CPU algorithm (the float64 numpy
oracle port in oracle/, the reference itself being pure Python that cannot be
shipped to the GPU box) on the host cores, on a bounded per-step sample of the
same workload, extrapolated to a full step.
"""

from __future__ import annotations

import argparse
import re
import glob
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd Mpixels/s at 1M Gaussians 1080p"
N_GAUSS = 1_000_000
W, H = 1920, 1080
MEDIUM = dict(attenuation=(0.6, 0.45, 0.3), water_color=(0.2, 0.35, 0.5),
              backscatter=(0.8, 1.0, 1.2), water_color_guide=(0.25, 0.3, 0.45),
              backscatter_guide=(0.9, 1.0, 1.1))


def synthetic_cloud(n, seed=0):
    """reference fixtures.random_cloud with the survey's scale rule."""
    rng = np.random.default_rng(seed)
    f = (1e4 / n) ** (1.0 / 3.0)
    pos = np.stack([rng.uniform(-4, 4, n), rng.uniform(-4, 4, n), rng.uniform(4, 20, n)], axis=1)
    log_scales = np.log(rng.uniform(0.15 * f, 0.6 * f, (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    colors = rng.uniform(0.1, 0.9, (n, 3))
    sh = ((colors - 0.5) / 0.28209479177387814)[:, None, :]
    return dict(positions=pos.astype(np.float32), log_scales=log_scales.astype(np.float32),
                rotations=q.astype(np.float32), sh_coeffs=sh.astype(np.float32),
                opacity_logits=rng.uniform(-1.0, 1.5, n).astype(np.float32))


def view_eye(rank):
    # rank 0 is the survey camera; other ranks orbit slightly (equal workload)
    th = 2 * np.pi * rank / 64.0
    return (3.0 + 0.3 * (1 - np.cos(th)), -2.0 + 0.3 * np.sin(th), -1.0)


def gt_image(seed=0):
    return np.random.default_rng(seed).uniform(0, 1, (H, W, 3)).astype(np.float32)


def kernel_traffic(stage):
    """DRAM bytes (read + write) per launch of the stage's dominant kernel, from the committed
    `ncu --set full` capture summary under profiles/ (None when no capture is on file)."""
    kern = {"uws_raster_bwd": "k_raster_bwd", "uws_raster_fwd": "k_raster_fwd",
            "uws_preprocess_fwd": "k_preprocess", "uws_preprocess_bwd": "k_preprocess_bwd",
            "uws_adam_step": "k_adam_cloud", "uws_loss_fwd_bwd": "k_ssim"}.get(stage)
    if kern is None:
        return None
    def version(path):  # (round, capture) numerically: r01/kernel_traffic_v10 after _v9
        nums = [int(x) for x in re.findall(r"\d+", os.path.relpath(path, ROOT))]
        return nums

    caps = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "kernel_traffic*.json")),
                  key=version)
    if not caps:
        return None
    try:
        data = json.load(open(caps[-1]))
    except (OSError, ValueError):
        return None
    tot = [v["dram_bytes"] for k, v in data.items()
           if k.split("<")[0].split("::")[-1] == kern or (kern == "k_ssim" and "k_ssim" in k)]
    return {"bytes": sum(tot), "source": os.path.relpath(caps[-1], ROOT)} if tot else None


# ----------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


class ClockSampler:
    """Samples SM clock + clock-event reasons through NVML every ~2 ms while active."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.err = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
        return self

    def _run(self):
        nv, h = self.nv, self.h
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, rs))
            except Exception as e:  # noqa: BLE001
                self.err = repr(e)
                return
            time.sleep(0.002)

    def __exit__(self, *exc):
        self.stop.set()
        if hasattr(self, "thread"):
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"],
                    "samples": 0, "error": self.err}
        reasons = set()
        for _, r in self.samples:
            for bit, name in REASON_BITS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s for s, _ in self.samples),
                "sm_max_mhz": self.max_sm, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------
class StageTimer:
    """CUDA events around selected C-ABI entry points on the launching stream."""

    def __init__(self, torch):
        self.torch = torch
        self.events = {}
        self.order = []      # (name, start, end) in launch order
        self.enabled = False

    def wrap(self, lib_mod):
        orig = lib_mod.call
        timer = self

        def call(name, *args):
            if not timer.enabled or name.endswith("_size"):
                return orig(name, *args)
            s = timer.torch.cuda.Event(enable_timing=True)
            e = timer.torch.cuda.Event(enable_timing=True)
            s.record()
            r = orig(name, *args)
            e.record()
            timer.events.setdefault(name, []).append((s, e))
            timer.order.append((name, s, e))
            return r

        lib_mod.call = call

    def totals(self):
        return {k: sum(s.elapsed_time(e) for s, e in v) for k, v in self.events.items()}

    def gaps(self):
        """Device time between consecutive timed calls (other launches, memsets,
        host-side stalls), summed per preceding stage."""
        out = {}
        for (n0, _, e0), (_, s1, _) in zip(self.order, self.order[1:]):
            out[n0] = out.get(n0, 0.0) + max(e0.elapsed_time(s1), 0.0)
        return out


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import paper_2411_19588_b200 as uw
    from paper_2411_19588_b200 import _lib

    timer = StageTimer(torch)
    timer.wrap(_lib)
    lib = _lib.load()

    host = synthetic_cloud(N_GAUSS)
    cloud = uw.GaussianCloud(**host)
    medium = uw.MediumParams(**MEDIUM)
    state = uw.TrainState(cloud, medium, iteration=1)
    cfg = uw.OptimConfig()
    trainer = uw.ViewShardedTrainer(state, cfg, W, H)
    cam = uw.Camera.look_at(view_eye(rank), (0, 0, 12), width=W, height=H, fx=1.2 * W, fy=1.2 * W)
    gt_host = torch.from_numpy(gt_image(rank)).pin_memory()
    gt_dev = gt_host.to(dev)

    # Steps are pipelined (StepEngine.step_async): step i is launched before the
    # host reads step i-1's result record (loss, finite/overflow flags, list sizes),
    # so the GPU never waits for the host; the last record is read by flush().
    def step_resident():
        trainer.step_async([(cam, gt_dev)], sharded=True)
        state.iteration += 1

    def step_e2e():
        # ground truth from pinned host memory every step: the engine copies it on
        # its copy stream while the previous step's kernels run
        trainer.step_async([(cam, gt_host)], sharded=True)
        state.iteration += 1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, k, stage_timer=False):
        trainer.flush()
        barrier()
        launches0 = lib.uws_kernel_launches()
        timer.enabled = stage_timer
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(k):
            fn()
        trainer.flush()      # host read of the last step's result record
        end.record()
        timer.enabled = False
        barrier()
        ms = start.elapsed_time(end)
        launches = lib.uws_kernel_launches() - launches0
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, launches

    for _ in range(args.warmup):
        step_resident()
    clocks = ClockSampler(local)
    with clocks:
        ms, launches = timed(step_resident, args.steps)
    # per-stage breakdown from a separate run with CUDA events around every C-ABI
    # call (kept out of the timed region above)
    timed(step_resident, args.steps, stage_timer=True)
    stages = timer.totals()
    gaps = timer.gaps()
    for _ in range(max(2, args.warmup // 2)):   # both pipeline slots warm
        step_e2e()
    ms_e2e, _ = timed(step_e2e, args.steps)
    trainer.flush()

    # render FPS (BASELINE.json's second metric): the forward alone -- preprocess,
    # depth sort, tile-row lists, compositing with the medium epilogue -- per frame
    # through StepEngine.render_async (a frame stream: each frame's overflow flag is
    # read once the next frame is queued), at C3 and at C5's 1M Gaussians @ 3840x2160
    render_fps = {}
    for name, (rw, rh) in ((("C3 1M 1920x1080", (W, H)), ("C5 1M 3840x2160", (3840, 2160)))
                           if not args.no_render_fps else ()):
        eng = trainer.engine if (rw, rh) == (W, H) else uw.StepEngine(state, rw, rh, cfg)
        rcam = uw.Camera.look_at(view_eye(rank), (0, 0, 12), width=rw, height=rh,
                                 fx=1.2 * rw, fy=1.2 * rw)
        for _ in range(3):
            eng.render(rcam)
        nfr = max(args.steps, 10)
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(nfr):
            eng.render_async(rcam)
        eng.render_flush()
        t1.record()
        barrier()
        fms = t0.elapsed_time(t1) / nfr
        render_fps[name] = {"fps": round(1e3 / fms, 1), "ms_per_frame": round(fms, 4),
                            "mpix_per_s": round(rw * rh / fms / 1e3, 1)}
        if eng is not trainer.engine:
            del eng
    # guidance refresh (pipeline.py:204-208; every refit_period = 500 steps): the
    # dark-pixel estimate from the C3 ground truth and the engine's render depth,
    # including the host read of the 96-byte result record (untimed for the step)
    refresh_ms = None
    if not args.no_render_fps:
        depth_raw = trainer.engine.out.depth
        for _ in range(2):
            uw.estimate_backscatter(gt_dev, depth_raw, depth_is_raw=True)
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(5):
            uw.estimate_backscatter(gt_dev, depth_raw, depth_is_raw=True)
        t1.record()
        barrier()
        refresh_ms = round(t0.elapsed_time(t1) / 5, 4)
    torch.cuda.empty_cache()

    px_step = W * H * world
    value = px_step * args.steps / (ms / 1e3) / 1e6
    e2e = px_step * args.steps / (ms_e2e / 1e3) / 1e6

    # workload statistics for the roofline (untimed)
    out = uw.render(cloud, cam, medium, "underwater")
    k_vis = len(out.proj)
    e_ent = int(out.bins.entries.numel())
    last = out.last.view(-1).long()
    term = (out.final_transmittance.view(-1) < 1e-4)
    offs = out.bins.offsets.long()
    gx = (W + 15) // 16
    ys = torch.arange(H, device=dev).view(H, 1).expand(H, W).reshape(-1) // 16
    xs = torch.arange(W, device=dev).view(1, W).expand(H, W).reshape(-1) // 16
    tid = ys * gx + xs
    m_tile = (offs[1:] - offs[:-1])[tid]
    p_pix = int(torch.where(term, last, m_tile).sum().item())
    per_step = {k: v / args.steps for k, v in stages.items()}
    canon = {k: k.replace("_rows", "") for k in per_step}  # row-list variants: same work
    total_stage = sum(per_step.values())
    fwd_flops = 30.0 * p_pix
    bwd_flops = 60.0 * p_pix
    fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12
    hbm_peak = 6552.0
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak = float(peaks.get("hbm_gbs", hbm_peak))
    except (OSError, ValueError):
        pass
    rb_ms = per_step.get("uws_raster_bwd", float("nan"))
    rf_ms = per_step.get("uws_raster_fwd", float("nan"))
    dominant = max(per_step, key=per_step.get) if per_step else None
    stage_share = {k: round(v / total_stage, 4) for k, v in per_step.items()} if total_stage else {}
    hbm_bytes = {
        "uws_preprocess_fwd": 56 * N_GAUSS + 48 * k_vis,
        "uws_bin_count": 24 * k_vis,
        "uws_bin_emit": 20 * e_ent,
        "uws_bin_rows": 24 * k_vis,
        "uws_loss_fwd_bwd": 36 * W * H,
        "uws_preprocess_bwd": 36 * k_vis + 112 * N_GAUSS,
        "uws_adam_step": 392 * N_GAUSS,
    }
    stage_roofline = {}
    for k, v in per_step.items():
        if canon[k] in hbm_bytes and v > 0:
            gbs = hbm_bytes[canon[k]] / (v / 1e3) / 1e9
            stage_roofline[k] = {"bound": "hbm", "achieved_gbs": round(gbs, 1),
                                 "frac": round(gbs / hbm_peak, 4), "ms": round(v, 4)}
    for k in per_step:
        fl = {"uws_raster_fwd": fwd_flops, "uws_raster_bwd": bwd_flops}.get(canon[k])
        if fl is not None and per_step[k] > 0:
            tf = fl / (per_step[k] / 1e3) / 1e12
            stage_roofline[k] = {"bound": "fp32", "achieved_tflops": round(tf, 3),
                                 "frac": round(tf / fp32_peak, 4), "ms": round(per_step[k], 4)}
    dom = stage_roofline.get(dominant, {})
    traffic = kernel_traffic(canon.get(dominant))
    if canon.get(dominant) in ("uws_raster_fwd", "uws_raster_bwd"):
        fl = bwd_flops if canon[dominant] == "uws_raster_bwd" else fwd_flops
        achieved = fl / (per_step[dominant] / 1e3) / 1e12
        roofline = {"bound": "fp32", "kernel": dominant, "achieved": round(achieved, 3),
                    "peak": round(fp32_peak, 1), "unit": "TFLOP/s",
                    "frac": round(achieved / fp32_peak, 4), "traffic": traffic,
                    "peak_source": "nominal FP32 non-tensor 148 SM x 128 lanes x 2 x 1.965 GHz "
                                   "(no FP32 figure in MEASURED_PEAKS.json; no tensor cores on "
                                   "this path)",
                    "work": f"{fl / 1e9:.2f} GFLOP per launch (SURVEY 8d: "
                            f"{'60' if canon[dominant].endswith('bwd') else '30'} flop x P_pix={p_pix})"}
    elif canon.get(dominant) in hbm_bytes:
        gbs = hbm_bytes[canon[dominant]] / (per_step[dominant] / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": dominant, "achieved": round(gbs, 1),
                    "peak": hbm_peak, "unit": "GB/s", "frac": round(gbs / hbm_peak, 4),
                    "traffic": traffic}
    else:
        roofline = {"bound": "hbm", "kernel": dominant, "achieved": None, "peak": hbm_peak,
                    "unit": "GB/s", "frac": None, "traffic": None}

    result = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mpixels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (survey generator, random-init 1M Gaussians, U(0,1) ground truth)",
        "config": {"workload": "C3: 1M Gaussians 1920x1080 underwater training step "
                               "(render+loss+backward+Adam) per GPU, view-sharded",
                   "gaussians": N_GAUSS, "width": W, "height": H, "views_per_step": world,
                   "parallelism": f"view-sharded dp{world} + NCCL all-reduce",
                   "l2": "working set > L2 (params+Adam 168 MB, tile lists ~"
                         f"{e_ent * 8 / 1e6:.0f} MB); no flush"},
        "e2e": {"value": round(e2e, 3), "unit": "Mpixels/s",
                "h2d_bytes_per_step": H * W * 3 * 4,
                "d2h_bytes_per_step": 4 + 8 + 7 * 8},
        "gpu_launches": int(launches),
        "render_fps": render_fps,
        "guidance_refresh_ms": refresh_ms,
        "roofline": roofline,
        "stages_ms": {k: round(v, 4) for k, v in per_step.items()},
        "gaps_after_stage_ms": {k: round(v / args.steps, 4) for k, v in gaps.items()},
        "stage_share": stage_share,
        "stage_roofline": stage_roofline,
        "workload_stats": {"K": k_vis, "E": e_ent, "P_pix": p_pix},
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args.cpu_tiles, report_only=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result if rank == 0 else None


# ----------------------------------------------------------------------------
# CPU reference arm (oracle port of the reference algorithm)
# ----------------------------------------------------------------------------
def cpu_step_sample(cloud, cam, medium, gt, tiles_sample, workers, state):
    """One sampled reference step; returns (extrapolated full-step seconds, details)."""
    from concurrent.futures import ThreadPoolExecutor
    from types import SimpleNamespace

    from oracle import uwsplat_oracle as O

    t0 = time.perf_counter()
    proj = O.project(cloud, cam)
    t_proj = time.perf_counter() - t0
    gx, gy = O.grid_dims(cam.width, cam.height)
    # binning (rasterizer.py:50-85): the entry emission runs on the full frame;
    # the (tile, depth, source) lexsort runs on the sampled tiles' entries and
    # is extrapolated linearly in E (n log n in reality: favours the CPU)
    t0 = time.perf_counter()
    rect = O.tile_rect(proj.mean2d, proj.radius, (gx, gy))
    wx = rect[:, 2] - rect[:, 0] + 1
    cnt = np.maximum(wx, 0) * np.maximum(rect[:, 3] - rect[:, 1] + 1, 0)
    e_total = int(cnt.sum())
    owner = np.repeat(np.arange(len(cnt)), cnt)
    k = np.arange(e_total) - (np.cumsum(cnt) - cnt)[owner]
    tid = (rect[owner, 1] + k // wx[owner]) * gx + (rect[owner, 0] + k % wx[owner])
    t_emit = time.perf_counter() - t0
    sel = np.isin(tid, tiles_sample)
    owner, tid = owner[sel], tid[sel]
    t0 = time.perf_counter()
    perm = np.lexsort((proj.source_index[owner], proj.depth[owner], tid))
    owner, tid = owner[perm], tid[perm]
    offsets = np.zeros(gx * gy + 1, np.int64)
    offsets[1:] = np.cumsum(np.bincount(tid, minlength=gx * gy))
    entries = owner
    t_sort = time.perf_counter() - t0
    e_sample = int(entries.size)
    t_bin = t_emit + t_sort * e_total / max(e_sample, 1)
    # per-tile forward + backward on the sample (tile-parallel like the reference)
    dL = np.zeros((cam.height, cam.width, 3))

    def fwd(t):
        ty, tx = divmod(int(t), gx)
        _, px, py = O._tile_pixels(tx, ty, cam.width, cam.height)
        rows = entries[offsets[t]:offsets[t + 1]]
        return O.blend(px, py, proj.mean2d[rows], proj.conic[rows], proj.color[rows],
                       proj.opacity[rows], proj.depth[rows], float(cam.far))

    def bwd(t):
        ty, tx = divmod(int(t), gx)
        (x0, x1, y0, y1), px, py = O._tile_pixels(tx, ty, cam.width, cam.height)
        rows = entries[offsets[t]:offsets[t + 1]]
        G = np.full(((y1 - y0) * (x1 - x0), 3), 1e-7)
        return O.tile_grads(px, py, proj.mean2d[rows], proj.conic[rows], proj.color[rows],
                            proj.opacity[rows], G)

    with ThreadPoolExecutor(max_workers=workers) as pool:
        t0 = time.perf_counter()
        list(pool.map(fwd, tiles_sample))
        t_fwd = time.perf_counter() - t0
        t0 = time.perf_counter()
        list(pool.map(bwd, tiles_sample))
        t_bwd = time.perf_counter() - t0
    # full-image loss (the reference evaluates it on the whole frame)
    img = np.random.default_rng(1).uniform(0, 1, gt.shape)
    t0 = time.perf_counter()
    O.total_loss(img, gt, medium, 0.3, 0.1)
    t_loss = time.perf_counter() - t0
    # projection backward over all visible rows + Adam over all parameters
    K = len(proj.depth)
    rng = np.random.default_rng(2)
    t0 = time.perf_counter()
    g = O.world_grads(proj, cam, rng.normal(size=(K, 2)) * 1e-6, rng.normal(size=(K, 3)) * 1e-6,
                      rng.normal(size=(K, 3)) * 1e-6, rng.normal(size=K) * 1e-6,
                      len(cloud.positions))
    t_world = time.perf_counter() - t0
    t0 = time.perf_counter()
    for f in ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits"):
        p = getattr(cloud, f)
        z = state.setdefault(f, (np.zeros_like(p), np.zeros_like(p)))
        O.adam(p, g["d_" + f], z[0], z[1], 1, 1e-3)
    t_adam = time.perf_counter() - t0
    lens = offsets[1:] - offsets[:-1]
    # scale the sampled per-tile work by the full frame's tile-list length
    e_in_sample = max(int(lens[np.asarray(tiles_sample)].sum()), 1)
    scale_tiles = e_total / e_in_sample
    full = t_proj + t_bin + (t_fwd + t_bwd) * scale_tiles + t_loss + t_world + t_adam
    return full, dict(project=t_proj, bin_emit=t_emit, bin_sort_sample=t_sort, fwd_sample=t_fwd,
                      bwd_sample=t_bwd, loss=t_loss, world=t_world, adam=t_adam,
                      e_total=e_total, e_sample=e_sample, scale=scale_tiles)


def cpu_setup():
    from types import SimpleNamespace
    host = synthetic_cloud(N_GAUSS)
    cloud = SimpleNamespace(**host)
    from paper_2411_19588_b200.scene import Camera
    cam = Camera.look_at(view_eye(0), (0, 0, 12), width=W, height=H, fx=1.2 * W, fy=1.2 * W)
    medium = SimpleNamespace(**{k: np.asarray(v, np.float32) for k, v in MEDIUM.items()})
    gt = gt_image(0).astype(np.float64)
    return cloud, cam, medium, gt


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(n_tiles, report_only=False, steps=1):
    cores = cpu_cores()
    cloud, cam, medium, gt = cpu_setup()
    gx, gy = (W + 15) // 16, (H + 15) // 16
    tiles = np.sort(np.random.default_rng(7).choice(gx * gy, n_tiles, replace=False))
    state = {}
    times = []
    for _ in range(steps):
        full, det = cpu_step_sample(cloud, cam, medium, gt, tiles, cores, state)
        times.append(full)
    full = float(np.median(times))
    return {"value": round(W * H / full / 1e6, 6), "unit": "Mpixels/s", "cores": cores,
            "kind": "port",
            "sample": (f"float64 numpy oracle of the reference algorithm; full projection, "
                       f"loss, projection-backward and Adam; binning + per-tile forward/backward "
                       f"on {n_tiles} of {gx * gy} seeded tiles (tile-parallel, {cores} threads), "
                       f"extrapolated by tile-list length (x{det['scale']:.0f})"),
            "extrapolated_step_s": round(full, 2),
            "breakdown_s": {k: round(v, 3) for k, v in det.items() if isinstance(v, float)}}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    cores = cpu_cores()
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    cloud, cam, medium, gt = cpu_setup()
    gx, gy = (W + 15) // 16, (H + 15) // 16
    tiles = np.sort(np.random.default_rng(7).choice(gx * gy, args.cpu_tiles, replace=False))
    state = {}
    for _ in range(args.warmup):
        cpu_step_sample(cloud, cam, medium, gt, tiles, cores, state)
    times = []
    for _ in range(args.steps):
        full, det = cpu_step_sample(cloud, cam, medium, gt, tiles, cores, state)
        times.append(full)
    per_step = float(np.mean(times))
    value = W * H / per_step / 1e6
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Mpixels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(per_step * 1e3, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (survey generator, random-init 1M Gaussians, U(0,1) ground truth)",
        "config": {"workload": "C3: 1M Gaussians 1920x1080 underwater training step "
                               "(render+loss+backward+Adam), reference CPU algorithm",
                   "gaussians": N_GAUSS, "width": W, "height": H},
        "cpu_baseline": {"value": round(value, 6), "unit": "Mpixels/s", "cores": cores,
                         "kind": "port",
                         "sample": f"per step: full projection/loss/projection-backward/Adam, "
                                   f"binning+compositing fwd/bwd on {args.cpu_tiles} of "
                                   f"{gx * gy} tiles, extrapolated (x{det['scale']:.0f})"},
        "e2e": {"value": round(value, 6), "unit": "Mpixels/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--cpu-tiles", type=int, default=12)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-render-fps", action="store_true",
                    help="skip the render-FPS frames (e.g. for a step-only ncu launch list)")
    args = ap.parse_args()
    res = run_reference(args) if args.impl == "reference" else run_gpu(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
