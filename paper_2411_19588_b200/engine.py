"""Device-resident training step without host synchronisation.

The public functions (render / total_loss / backward_render /
apply_gradients) mirror the reference API and therefore read sizes back to
the host (K visible Gaussians, E tile entries) to allocate exact outputs.
The training loop does not need that: :class:`StepEngine` owns persistent
buffers for a fixed cloud size and image size, passes counts between kernels
in device memory, and sizes the tile lists with a capacity.  A step is a
fixed sequence of asynchronous launches --

    per view:  preprocess -> depth sort + tile-row counts -> tile-row
               lists -> forward compositing (each tile filters its row list
               on the fly and stops at saturation: the E-entry tile lists of
               bin_and_sort are never materialised) -> L1/D-SSIM loss ->
               backward compositing (re-derives the same consumed prefix)
               -> projection backward (accumulating)
    then:      [NCCL all-reduce of the flat gradient buffer]
               -> fused Adam (skips itself on non-finite / overflow,
                  accumulates the densification statistics, zeroes grads)

-- followed by ONE small device-to-host read (loss values, flags, list
sizes).  If a view's row lists did not fit their capacity the kernels turn
the whole step into a no-op on the device (Adam skipped); the engine grows
the buffers to the reported sizes and runs the step again.  This is the
loop body of pipeline.train (reference pipeline.py:170-193).
"""

from __future__ import annotations

import ctypes
import logging
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .backward import GradientBuffer
from .losses import total_loss_device
from .optim import OptimConfig, apply_gradients_device, range_chunks, rollback_steps
from .projection import ProjectedCloud, preprocess_into
from .rasterizer import RenderOutput, RowLists, _alloc_output
from .scene import Camera, TrainState

log = logging.getLogger(__name__)

# per-view stats record (float64 slots)
_ST_LOSS = 0      # l1, d_ssim, l_bs, total, finite, reserved  (6)
_ST_TOTALS = 6    # E, S as int64 (2 slots)
_ST_OVF = 8       # overflow flag of this view (int32 in a float64 slot)
_ST_SIZE = 10


@dataclass
class EngineStats:
    l1: float
    d_ssim: float
    l_bs: float
    total: float
    views: int
    skipped: bool
    reruns: int
    max_entries: int


class StepEngine:
    """Persistent-buffer, sync-free training step for one (cloud size, image size)."""

    OVERLAP_VIEWS = True   # default of ``overlap_views``
    # composite the tiles heaviest first (the previous forward of the same buffer set
    # gives the schedule: uws_tile_order); a schedule only, results are unchanged
    TILE_ORDER = os.environ.get("UWS_TILE_ORDER", "1") != "0"
    RENDER_SETS = 3        # frame-stream buffer sets / streams (the engine's own + side sets;
                           # measured: 3 renders 1080p ~2 % faster than 2, 4K the same)

    def __init__(self, state: TrainState, width: int, height: int, cfg: OptimConfig,
                 spatial_scale: float = 1.0, max_views: int = 1, entry_capacity: int = 0,
                 group=None):
        import torch.distributed as dist
        self.state = state
        self.cfg = cfg
        self.spatial_scale = spatial_scale
        self.width, self.height = width, height
        self.max_views = max_views
        self.group = group
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0
        dev = state.cloud.device
        self.dev = dev
        self.gx, self.gy = (width + 15) // 16, (height + 15) // 16
        self.row_start = torch.zeros(self.gy + 1, dtype=torch.int32, device=dev)
        self.out = _alloc_output(height, width, dev, "underwater", False)
        self.out.tile_order = _identity_order(self.out)
        _order_state(self)
        self.dL = torch.empty(height, width, 3, dtype=torch.float32, device=dev)
        b = _lib.size_out()
        _lib.call("uws_loss_workspace_size", height, width, 3, ctypes.byref(b))
        self.loss_ws = torch.empty(b.value, dtype=torch.uint8, device=dev)
        self.med_acc = torch.zeros(9, dtype=torch.float64, device=dev)
        self._entry_capacity = entry_capacity
        self._alloc(len(state.cloud))
        # two in-flight step slots: stats record (device + pinned host copy + event) and
        # device copies of host ground-truth images
        self._slots = [_Slot(max_views, dev) for _ in range(2)]
        self._render_stats = torch.zeros(_ST_SIZE + 2, dtype=torch.float64, device=dev)
        # render_async: two frame records, the pending (queued, unchecked) frame
        nsets = self.RENDER_SETS
        self._async_stats = torch.zeros(nsets, _ST_SIZE + 2, dtype=torch.float64, device=dev)
        self._async_flag = torch.zeros(nsets, 2, dtype=torch.int32).pin_memory()
        self._async_done = [torch.cuda.Event() for _ in range(nsets)]
        self._more_sets = {}     # frame-stream buffer sets beyond the second (RENDER_SETS > 2)
        self._async_frames = 0
        self._async_pending = None
        self._fs = None          # the frame stream's second buffer set (lazy)
        # steps over several views overlap consecutive views on two streams / buffer sets
        self.overlap_views = self.OVERLAP_VIEWS
        self._last_view_set = None  # buffer set holding the last step's last view
        self._latest = None      # buffer set of the most recent frame (None: the engine's)
        self._k = 0
        self._pending = None
        # parity tests: leave the step's summed gradients in ``grads`` after Adam
        # (Adam normally consumes and zeroes them)
        self.keep_gradients = False
        # run-to-run bit-identical gradients (backward.py:334-341's fixed tile-order merge):
        # the deterministic backward, at the cost of one host read per view (slot count)
        self.deterministic = False
        self._det_ws = None
        self.copy_stream = torch.cuda.Stream(device=dev)

    def _alloc(self, n: int):
        """Buffers sized by the number of Gaussians (re-done after densification)."""
        dev = self.dev
        self.n = n
        self.generation = self.state.cloud.generation
        self.proj = ProjectedCloud(n, dev, with_geometry=False)
        b = _lib.size_out()
        _lib.call("uws_preprocess_workspace_size", n, ctypes.byref(b))
        self.pre_ws = torch.empty(max(b.value, 1), dtype=torch.uint8, device=dev)
        cb, eb = _lib.size_out(), _lib.size_out()
        _lib.call("uws_bin_workspace_size", n, 0, self.gx, self.gy, ctypes.byref(cb),
                  ctypes.byref(eb))
        self.count_ws = torch.empty(max(cb.value, 1), dtype=torch.uint8, device=dev)
        self._set_capacity(self._entry_capacity or 12 * n)
        self.screen = torch.zeros(max(n, 1), 9, dtype=torch.float32, device=dev)
        self.grads = GradientBuffer(n, dev)

    def _sync_cloud(self):
        """Follow a topology change of the cloud (densify_and_prune)."""
        cloud = self.state.cloud
        if len(cloud) != self.n or cloud.generation != self.generation:
            if self._pending is not None:
                raise RuntimeError("the cloud changed while a step was in flight: call "
                                   "flush() before densify_and_prune")
            self._alloc(len(cloud))

    # -- capacity management ---------------------------------------------------
    def _set_capacity(self, s_cap: int):
        """Capacity of the tile-row lists (S = sum over visible Gaussians of
        the tile rows their rectangle spans)."""
        self.s_cap = int(max(s_cap, 1))
        # 8-byte items: row index, tile-column span x0 | x1 << 16
        self.row_items = torch.empty(self.s_cap, 2, dtype=torch.int32, device=self.dev)

    # -- forward of one view (render path) ----------------------------------------
    def _forward(self, cam: Camera, stats: torch.Tensor, view: int, mode: str = "underwater",
                 train: bool = True, fs: "_FrameSet" = None):
        """Preprocess, depth order + row lists, compositing of one view into the
        engine's buffers, or into frame set ``fs`` (the frame stream's second set)."""
        b = self if fs is None else fs
        st = _lib.stream_handle()
        cloud, medium = self.state.cloud, self.state.medium
        cc = cam.c_struct()
        preprocess_into(b.proj, cloud, cam, b.pre_ws)
        pc = b.proj.c_struct()
        rec = stats[view * _ST_SIZE:(view + 1) * _ST_SIZE]
        totals = rec[_ST_TOTALS:_ST_TOTALS + 2].view(torch.int64)
        ovf = rec[_ST_OVF:_ST_OVF + 1].view(torch.int32)[:1]
        _lib.call("uws_bin_count", ctypes.byref(pc), self.n, ctypes.byref(cc), _lib.ptr(totals),
                  _lib.ptr(b.count_ws), b.count_ws.numel(), st)
        _lib.call("uws_bin_rows", ctypes.byref(pc), self.n, b.s_cap, ctypes.byref(cc),
                  _lib.ptr(totals), _lib.ptr(b.row_start), _lib.ptr(b.row_items),
                  _lib.ptr(ovf), _lib.ptr(self.grads.nonfinite) if train else 0,
                  _lib.ptr(b.count_ws), b.count_ws.numel(), st)
        out = b.out
        out.camera = cam
        oc = out.c_struct()
        self._order_wait(b)
        med = _lib.ptr(medium.flat) if mode == "underwater" else 0
        _lib.call("uws_raster_fwd_rows", ctypes.byref(pc), _lib.ptr(b.row_start),
                  _lib.ptr(b.row_items), ctypes.byref(cc), med, ctypes.byref(oc), st)
        if self.TILE_ORDER and not train:
            # render-only frame: the schedule for the set's next frame, in stream order
            # (a side stream would only add host work per frame)
            _lib.call("uws_tile_order", _lib.ptr(out.tile_nrows), out.tile_nrows.numel(),
                      _lib.ptr(out.tile_order), st)
        elif self.TILE_ORDER:
            # this forward's tile costs schedule this view's backward and the set's next
            # forward.  The one-CTA sort runs on the set's side stream, overlapping the
            # loss; every reader of the order waits for it (_order_wait).
            cur = torch.cuda.current_stream()
            b.ord_start.record(cur)
            b.ord_stream.wait_event(b.ord_start)
            with torch.cuda.stream(b.ord_stream):
                _lib.call("uws_tile_order", _lib.ptr(out.tile_nrows), out.tile_nrows.numel(),
                          _lib.ptr(out.tile_order), _lib.stream_handle())
                b.ord_done.record(b.ord_stream)
            b.ord_recorded = True
        return cc, pc, oc, rec

    @staticmethod
    def _order_wait(b):
        """The current stream waits for buffer set ``b``'s latest schedule (before a
        forward or backward reads it, or before its output is handed out)."""
        if b.ord_recorded:
            torch.cuda.current_stream().wait_event(b.ord_done)

    def render_async(self, cam, mode: str = "underwater") -> RenderOutput:
        """Queue one render-only frame without waiting for it (a frame stream).

        Consecutive frames rotate over RENDER_SETS buffer sets and streams (the
        engine's own buffers on the current stream, the others on side streams),
        so frame i+1's preprocess and depth order -- latency-bound kernels that
        leave most SMs idle -- run while frame i composites.  The
        row-list overflow flag of the PREVIOUS queued frame is read after this one
        is queued, so the host never idles the GPU between frames.  A frame's
        buffers hold its image only once ``render_flush()`` has returned
        (``last_render()`` then returns the most recent frame; a frame that
        overflowed its row lists is re-rendered there, synchronously).  The
        cloud must not change while frames are queued; ``step_async`` and
        ``refresh_guidance`` flush a pending frame first."""
        cam = Camera.from_any(cam)
        if self._pending is None:
            self._sync_cloud()
        k = self._async_frames % self.RENDER_SETS
        self._async_frames += 1
        cur = torch.cuda.current_stream()
        if self._async_pending is None:
            # a new frame stream: side-stream frames wait for everything queued before
            # it (the parameters they read), not for the frames on the current stream
            self._stream_start = torch.cuda.Event()
            self._stream_start.record(cur)
        if k >= 1:
            fs = self._frame_set() if k == 1 else self._extra_set(k)
            fs.stream.wait_event(self._stream_start)
            stream_ctx = torch.cuda.stream(fs.stream)
        else:
            fs = None
            stream_ctx = torch.cuda.stream(cur)
        with stream_ctx:
            stats = self._async_stats[k]
            stats.zero_()
            self._forward(cam, stats, 0, mode, train=False, fs=fs)
            # the frame's overflow flag to pinned memory, behind the frame's kernels
            self._async_flag[k].copy_(stats[_ST_OVF:_ST_OVF + 1].view(torch.int32),
                                      non_blocking=True)
            self._async_done[k].record()
        (self.out if fs is None else fs.out).mode = mode
        prev, self._async_pending = self._async_pending, (cam, mode, k)
        self._latest = fs
        if prev is not None and self._async_overflowed(prev[2]):
            self.render_flush()
        return self._frame_output(fs)

    def render_flush(self) -> RenderOutput:
        """Wait for the queued frames; re-render the last one if its row lists overflowed.
        Returns the most recent frame."""
        frame, self._async_pending = self._async_pending, None
        for fs in [self._fs] + list(self._more_sets.values()):
            if fs is not None:
                torch.cuda.current_stream().wait_stream(fs.stream)
        if frame is not None and self._async_overflowed(frame[2]):
            self._latest = None
            return self.render(frame[0], frame[1])
        return self._frame_output(self._latest)

    def _frame_set(self, train: bool = False) -> "_FrameSet":
        """The second buffer set (frame stream, overlapped views), (re)built for the
        engine's sizes; ``train`` adds the loss / backward buffers."""
        if self._fs is None or self._fs.n != self.n or self._fs.s_cap != self.s_cap:
            if self._fs is not None:
                self._fs.stream.synchronize()   # its buffers are freed below
                self._fs.ord_stream.synchronize()
                stream = self._fs.stream
            else:
                stream = torch.cuda.Stream(device=self.dev)
            self._fs = None
            self._fs = _FrameSet(self, stream)
        if train:
            self._fs.add_training(self)
        return self._fs

    def _extra_set(self, k: int) -> "_FrameSet":
        fs = self._more_sets.get(k)
        if fs is None or fs.n != self.n or fs.s_cap != self.s_cap:
            stream = fs.stream if fs is not None else torch.cuda.Stream(device=self.dev)
            if fs is not None:
                fs.stream.synchronize()
                fs.ord_stream.synchronize()
            self._more_sets[k] = None
            fs = self._more_sets[k] = _FrameSet(self, stream)
        return fs

    def _frame_output(self, fs) -> RenderOutput:
        if fs is None:
            return self.last_render()
        self._order_wait(fs)
        out = fs.out
        out.proj = fs.proj
        out.bins = None
        out.rows = RowLists(self.gx, self.gy, fs.row_start, fs.row_items)
        return out

    def _async_overflowed(self, k: int) -> bool:
        self._async_done[k].synchronize()   # waits for that frame only
        return int(self._async_flag[k, 0]) != 0

    def render(self, cam, mode: str = "underwater") -> RenderOutput:
        """Render-only path (no host sync before the caller reads the image).
        Overflow of the row-list capacity is detected and the view re-run."""
        cam = Camera.from_any(cam)
        if self._pending is None:
            self._sync_cloud()
        for _ in range(4):
            self._render_stats.zero_()
            self._forward(cam, self._render_stats, 0, mode, train=False)
            rec = self._render_stats[0:_ST_SIZE]
            if int(rec[_ST_OVF:_ST_OVF + 1].view(torch.int32)[0]) == 0:
                break
            need_s = int(rec[_ST_TOTALS:_ST_TOTALS + 2].view(torch.int64)[1])
            self._set_capacity(int(need_s * 1.25) + 1024)
        self.out.mode = mode
        self._latest = None      # the most recent frame is in the engine's own buffers
        return self.last_render()

    # -- one view: forward + loss + backward into self.grads -----------------------
    def _view(self, cam: Camera, gt: torch.Tensor, stats: torch.Tensor, view: int,
              fs: "_FrameSet" = None, after=None):
        """Forward, loss and backward of one view into the engine's buffers (or
        buffer set ``fs``); the projection backward -- the only stage writing the
        shared gradient buffer -- first waits for event ``after`` (the previous
        view's projection backward on the other stream)."""
        b = self if fs is None else fs
        st = _lib.stream_handle()
        cloud, medium = self.state.cloud, self.state.medium
        cc, pc, oc, rec = self._forward(cam, stats, view, fs=fs)
        out = b.out
        total_loss_device(out.color, gt, medium, self.cfg.lambda_ssim, self.cfg.lambda_guide,
                          result=rec[_ST_LOSS:_ST_LOSS + 6], grad=b.dL, workspace=b.loss_ws,
                          nonfinite=self.grads.nonfinite)
        self._order_wait(b)
        if self.deterministic:
            self._raster_bwd_det(pc, cc, oc, medium, st)
        else:
            _lib.call("uws_raster_bwd_rows", ctypes.byref(pc), _lib.ptr(b.row_start),
                      _lib.ptr(b.row_items), ctypes.byref(cc), _lib.ptr(medium.flat),
                      ctypes.byref(oc), _lib.ptr(b.dL), _lib.ptr(b.screen),
                      _lib.ptr(b.med_acc), st)
        if after is not None:
            torch.cuda.current_stream().wait_event(after)
        cl = cloud.c_struct()
        guided = 1 if medium.has_guidance else 0
        _lib.call("uws_preprocess_bwd", ctypes.byref(cl), ctypes.byref(cc), ctypes.byref(pc),
                  self.n, _lib.ptr(b.screen), _lib.ptr(b.med_acc), _lib.ptr(medium.flat),
                  guided, float(self.cfg.lambda_guide), _lib.ptr(self.grads.flat),
                  _lib.ptr(self.grads.nonfinite), 1 if view > 0 else 0, st)
        # (the first view stores: Adam leaves the parameter gradients zeroed)

    def _raster_bwd_det(self, pc, cc, oc, medium, st):
        """Deterministic K8 on the row lists (uws_raster_bwd_det): slot partials summed
        per Gaussian in tile order.  Reads the slot count (one sync per view)."""
        tiles = self.gx * self.gy
        if self._det_ws is None:
            self._det_ws = (torch.empty(tiles, dtype=torch.int32, device=self.dev),
                            torch.empty(tiles + 1, dtype=torch.int32, device=self.dev),
                            torch.empty(1, dtype=torch.uint8, device=self.dev))
        count, base, ws = self._det_ws
        _lib.call("uws_raster_bwd_det_prefix", ctypes.byref(cc), ctypes.byref(oc),
                  _lib.ptr(count), _lib.ptr(base), st)
        r = int(base[tiles].item())
        k = self.proj.k
        nb = _lib.size_out()
        _lib.call("uws_raster_bwd_det_workspace_size", tiles, r, k, ctypes.byref(nb))
        if ws.numel() < nb.value:
            ws = torch.empty(int(nb.value * 1.25) + 1, dtype=torch.uint8, device=self.dev)
            self._det_ws = (count, base, ws)
        _lib.call("uws_raster_bwd_det", ctypes.byref(pc), 0, 0, _lib.ptr(self.row_start),
                  _lib.ptr(self.row_items), ctypes.byref(cc), _lib.ptr(medium.flat),
                  ctypes.byref(oc), _lib.ptr(self.dL), _lib.ptr(self.screen),
                  _lib.ptr(self.med_acc), _lib.ptr(base), r, k, _lib.ptr(ws), ws.numel(), st)

    def last_render(self) -> RenderOutput:
        """Forward buffers of the most recent view (valid until the next step).
        ``bins`` is None: the engine never materialises full tile lists."""
        self._order_wait(self)
        out = self.out
        out.proj = self.proj
        out.bins = None
        out.rows = RowLists(self.gx, self.gy, self.row_start, self.row_items)
        return out

    # -- ground truth staging -------------------------------------------------------
    def _stage(self, views: Sequence, slot: "_Slot"):
        """Device views for a step: host images are copied into the slot's
        device buffers on the copy stream (overlapping the previous step's
        kernels); device images are used in place."""
        if len(views) > self.max_views:
            raise ValueError(f"at most {self.max_views} views per step on this engine")
        out = []
        cs = self.copy_stream
        cs.wait_event(slot.free)        # the slot's previous step no longer reads them
        for i, (cam, gt) in enumerate(views):
            cam = Camera.from_any(cam)
            if isinstance(gt, torch.Tensor) and gt.is_cuda:
                out.append((cam, gt.float()))
                continue
            src = gt if isinstance(gt, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(gt, dtype=np.float32))
            buf = slot.gt_buffer(i, (self.height, self.width, 3))
            other = self._slots[(self._slots.index(slot) + 1) % 2]
            other.gt_buffer(i, (self.height, self.width, 3))  # allocate both now, not mid-pipeline
            with torch.cuda.stream(cs):
                buf.copy_(src, non_blocking=True)
            out.append((cam, buf))
        slot.copied.record(cs)
        return out

    def _launch(self, slot: "_Slot"):
        cur = torch.cuda.current_stream()
        cur.wait_event(slot.copied)
        if len(slot.views) > 1 and self.overlap_views and not self.deterministic:
            self._launch_views_overlapped(slot, cur)
        else:
            for i, (cam, gt) in enumerate(slot.views):
                self._view(cam, gt, slot.stats, i)
            self._last_view_set = None
        chunks = None
        if self.dist is not None and self.world > 1:
            chunks = self._all_reduce_gradients()
        # the skip counters are read by the Adam launch (and kept while non-zero): keep a copy
        slot.stats[-2:].copy_(self.grads.skip_counters)
        saved = self.state.iteration
        self.state.iteration = slot.iteration
        apply_gradients_device(self.state, self.grads, self.cfg, self.spatial_scale,
                               zero_grads=not self.keep_gradients, chunks=chunks)
        self.state.iteration = saved
        slot.host.copy_(slot.stats, non_blocking=True)
        slot.done.record(cur)
        slot.free.record(cur)

    def _launch_views_overlapped(self, slot: "_Slot", cur):
        """Several views in one step: even views on the engine's buffers and the
        current stream, odd views on the second buffer set and its stream, so a
        view's preprocess / depth order / compositing overlap the previous view's
        backward.  The projection backwards (the only writers of the gradient
        buffer; view 0 stores, later views add) stay in view order through events."""
        ts = self._frame_set(train=True)
        ts.stream.wait_stream(cur)      # parameters (previous Adam) and ground-truth copies
        prev = None
        for i, (cam, gt) in enumerate(slot.views):
            fs = ts if i % 2 else None
            with torch.cuda.stream(ts.stream if i % 2 else cur):
                self._view(cam, gt, slot.stats, i, fs=fs, after=prev)
                prev = torch.cuda.Event()
                prev.record()
        cur.wait_stream(ts.stream)
        self._last_view_set = ts if (len(slot.views) - 1) % 2 else None

    # gradient all-reduce: 1 = one NCCL all-reduce of the whole flat buffer, then
    # the single Adam launch (the default: the split form below has only been
    # measured on one GPU); > 1 = split against the range-wise cloud update
    ALLREDUCE_PARTS = 1

    def _all_reduce_gradients(self):
        """Sum the flat gradient buffer over the ranks.  The medium/skip tail and the
        densification statistics are reduced first (the medium update and the skip
        test read them); the 14n parameter gradients follow in ALLREDUCE_PARTS
        asynchronous NCCL all-reduces, and each range of the Adam update waits only
        for its own part, so the update of range c overlaps the reduction of c+1.
        Returns the chunk list for ``apply_gradients_device`` (None when the range
        form does not apply: every part has been waited for, then the single launch)."""
        flat, n, d, g = self.grads.flat, self.n, self.dist, self.group
        if self.ALLREDUCE_PARTS <= 1:
            d.all_reduce(flat, group=g)
            return None
        # the same collectives on every rank (they depend on n only) ...
        parts = [(14 * n * c // self.ALLREDUCE_PARTS // 4, 14 * n * (c + 1) // self.ALLREDUCE_PARTS // 4)
                 for c in range(self.ALLREDUCE_PARTS)]
        parts[-1] = (parts[-1][0], (14 * n + 3) // 4)
        head = [d.all_reduce(flat[16 * n:], group=g, async_op=True),
                d.all_reduce(flat[14 * n:16 * n], group=g, async_op=True)]
        works = [d.all_reduce(flat[4 * g0:min(4 * g1, 14 * n)], group=g, async_op=True)
                 for g0, g1 in parts]
        for w in head:
            w.wait()
        # ... and the range-wise update only where it applies (even n, aligned buffers)
        if range_chunks(self.state, self.grads, 1) is None:
            for w in works:
                w.wait()
            return None
        return [(g0, g1, w.wait) for (g0, g1), w in zip(parts, works)]

    def _read(self, slot: "_Slot"):
        slot.done.synchronize()
        s = slot.host
        nv = len(slot.views)
        need_e = need_s = 0
        for i in range(nv):
            tot = s[i * _ST_SIZE + _ST_TOTALS:i * _ST_SIZE + _ST_TOTALS + 2].view(torch.int64)
            need_e = max(need_e, int(tot[0]))   # tile entries (reported only)
            need_s = max(need_s, int(tot[1]))   # row-list items (capacity)
        return float(s[-2]), float(s[-1]), need_e, need_s

    def _stats(self, slot: "_Slot", skipped: bool, reruns: int, need_e: int) -> EngineStats:
        s, nv = slot.host, len(slot.views)
        loss = [sum(float(s[i * _ST_SIZE + j]) for i in range(nv)) / max(nv, 1) for j in range(4)]
        if skipped:
            log.warning("iteration %d: non-finite loss or gradients, skipping update",
                        slot.iteration)
        return EngineStats(loss[0], loss[1], loss[2], loss[3], nv * self.world, skipped, reruns,
                           need_e)

    def _finalize(self, slot: "_Slot") -> EngineStats:
        """Read a launched step's record.  A step the device skipped (non-finite
        values or a row-list overflow on any rank) leaves the skip counter set,
        which also turns every later launched step into a no-op; the host then
        undoes their step-counter advances, clears the counter, re-runs an
        overflowed step with grown lists and re-launches the later step."""
        nonfinite, overflow, need_e, need_s = self._read(slot)
        if nonfinite == 0 and overflow == 0:
            return self._stats(slot, False, 0, need_e)
        nxt = self._pending if self._pending is not slot else None
        if self.state.cloud.generation != self.generation:
            raise RuntimeError("a skipped step cannot be re-run after the cloud changed: "
                               "call flush() before densify_and_prune")
        torch.cuda.current_stream().synchronize()
        rollback_steps(self.state)
        if nxt is not None:
            rollback_steps(self.state)
        self.grads.skip_counters.zero_()
        reruns = 0
        # a row-list overflow on any rank: grow to the reported size and re-run
        # (a step that is also non-finite is then reported as skipped)
        while overflow > 0 and reruns < 3:
            if need_s > self.s_cap:
                self._set_capacity(int(need_s * 1.25) + 1024)
            reruns += 1
            self.grads.flat.zero_()   # (already zero unless keep_gradients)
            self._launch(slot)
            nonfinite, overflow, need_e, need_s = self._read(slot)
            if nonfinite > 0 or overflow > 0:
                rollback_steps(self.state)
                self.grads.skip_counters.zero_()
        st = self._stats(slot, nonfinite > 0 or overflow > 0, reruns, need_e)
        if nxt is not None:
            if self.keep_gradients:
                self.grads.flat.zero_()
            self._launch(nxt)
        return st

    # -- public stepping ---------------------------------------------------------------
    def step_async(self, views: Sequence):
        """Launch one optimizer step over this rank's (camera, gt) views without
        waiting for it; ground-truth images may be host arrays (copied on a side
        stream while the previous step runs) or device tensors.  Returns the
        stats of the previously launched step (None for the first)."""
        if self._async_pending is not None:
            self.render_flush()      # the frame stream shares the step's buffers
        self._sync_cloud()
        slot = self._slots[self._k % 2]
        self._k += 1
        slot.views = self._stage(views, slot)
        slot.iteration = self.state.iteration
        self._launch(slot)
        prev, self._pending = self._pending, slot
        return self._finalize(prev) if prev is not None else None

    def flush(self):
        """Wait for the last launched step and return its stats (None if none)."""
        slot, self._pending = self._pending, None
        return self._finalize(slot) if slot is not None else None

    def refresh_guidance(self, gt, **kw):
        """Guidance refresh of the training loop (pipeline.py:204-208): the
        dark-pixel estimate from the last step's last view -- its ground truth
        ``gt`` and the engine's render depth of that view -- becomes the
        medium's guidance unless degenerate.  Call after step() / flush()."""
        from .backscatter import refresh_guidance
        if self._pending is not None:
            raise RuntimeError("refresh_guidance reads the last step's render: call flush() first")
        if self._async_pending is not None:
            raise RuntimeError("refresh_guidance reads the last step's render depth, but a "
                               "render_async frame has replaced it")
        if not isinstance(gt, torch.Tensor):
            gt = torch.from_numpy(np.ascontiguousarray(gt, dtype=np.float32))
        out = self.out if self._last_view_set is None else self._last_view_set.out
        return refresh_guidance(self.state.medium, gt, out.depth, **kw)

    def step(self, views: Sequence) -> EngineStats:
        """One optimizer step over this rank's views, synchronously.

        Loss values in the returned stats are this rank's view averages."""
        self.step_async(views)
        return self.flush()


def _order_state(b):
    """Side stream and events of a buffer set's compositing schedule."""
    b.ord_stream = torch.cuda.Stream(device=b.out.tile_nrows.device)
    b.ord_start = torch.cuda.Event()
    b.ord_done = torch.cuda.Event()
    b.ord_recorded = False


def _identity_order(out: RenderOutput) -> torch.Tensor:
    """Raster-order compositing schedule for a buffer set's output."""
    return torch.arange(out.tile_nrows.numel(), dtype=torch.int32, device=out.tile_nrows.device)


class _FrameSet:
    """A second set of forward buffers on a side stream (StepEngine.render_async)."""

    def __init__(self, eng: StepEngine, stream):
        dev = eng.dev
        self.stream = stream
        self.n, self.s_cap = eng.n, eng.s_cap
        self.proj = ProjectedCloud(eng.n, dev, with_geometry=False)
        self.pre_ws = torch.empty_like(eng.pre_ws)
        self.count_ws = torch.empty_like(eng.count_ws)
        self.row_start = torch.zeros_like(eng.row_start)
        self.row_items = torch.empty_like(eng.row_items)
        self.out = _alloc_output(eng.height, eng.width, dev, "underwater", False)
        self.out.tile_order = _identity_order(self.out)
        _order_state(self)
        self.dL = None
        # the zero fills above are queued on the current stream: the set's stream
        # must not run a frame on these buffers before them
        self.stream.wait_stream(torch.cuda.current_stream())

    def add_training(self, eng: StepEngine):
        if self.dL is None:
            self.dL = torch.empty_like(eng.dL)
            self.loss_ws = torch.empty_like(eng.loss_ws)
            self.screen = torch.zeros_like(eng.screen)
            self.med_acc = torch.zeros_like(eng.med_acc)
            self.stream.wait_stream(torch.cuda.current_stream())


class _Slot:
    """Per in-flight step: stats record, its pinned host copy and events, and
    device buffers for host ground-truth images."""

    def __init__(self, max_views: int, dev):
        self.stats = torch.zeros(max_views * _ST_SIZE + 2, dtype=torch.float64, device=dev)
        self.host = torch.zeros_like(self.stats, device="cpu").pin_memory()
        self.done = torch.cuda.Event()
        self.copied = torch.cuda.Event()
        self.free = torch.cuda.Event()
        self.gt = []
        self.views = []
        self.iteration = 0
        self._dev = dev

    def gt_buffer(self, i: int, shape):
        while len(self.gt) <= i:
            self.gt.append(torch.empty(shape, dtype=torch.float32, device=self._dev))
        return self.gt[i]
