"""Training-step glue and view-sharded data parallelism.

``train_step`` is the body of the reference's training loop
(pipeline.py:178-193): render (underwater) -> total_loss -> skip if
non-finite -> backward_render -> skip if non-finite -> densification
statistics -> apply_gradients.  It needs one small device-to-host read per
step (loss values + finite flags) besides the two size reads of the
renderer.

``ViewShardedTrainer`` is the multi-GPU extension: every rank
holds the full cloud and optimizer state, renders and back-propagates its
share of the views into ONE flat gradient buffer, the buffers are summed
with a single NCCL all-reduce, and every rank applies the identical Adam
step.  The batch gradient equals the sum over views of the reference's
per-view ``backward_render`` (guidance subgradient added once per view).
"""

from __future__ import annotations

import logging
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from .backward import GradientBuffer, backward_render
from .losses import LossBreakdown, total_loss_device
from .optim import OptimConfig, apply_gradients
from .rasterizer import render
from .scene import TrainState

log = logging.getLogger(__name__)


@dataclass
class StepStats:
    l1: float
    d_ssim: float
    l_bs: float
    total: float
    views: int
    skipped: bool


GRAD_LAYOUT = (("d_positions", 3), ("d_log_scales", 3), ("d_rotations", 4), ("d_sh_coeffs", 3),
               ("d_opacity_logits", 1), ("mean2d_grad_norm", 1), ("observed", 1))


def pack_gradients(grads: dict, n: int) -> torch.Tensor:
    """Pack per-field gradients (any device, e.g. CPU for tests) into the flat
    GradientBuffer layout ``[14n params | n norm | n observed | 9 medium | pad]``."""
    parts = []
    for name, w in GRAD_LAYOUT:
        t = torch.as_tensor(grads[name]).reshape(n * w).to(torch.float32)
        parts.append(t)
    med = torch.cat([torch.as_tensor(grads[k]).reshape(3).to(torch.float32)
                     for k in ("d_attenuation", "d_water_color", "d_backscatter")])
    parts += [med, torch.zeros(7, dtype=torch.float32)]
    return torch.cat(parts)


def unpack_gradients(flat: torch.Tensor, n: int) -> dict:
    out, o = {}, 0
    for name, w in GRAD_LAYOUT:
        out[name] = flat[o:o + n * w].reshape((n, w) if w > 1 else (n,))
        o += n * w
    for k in ("d_attenuation", "d_water_color", "d_backscatter"):
        out[k] = flat[o:o + 3]
        o += 3
    return out


def shard_views(views: Sequence, rank: int, world: int) -> Sequence:
    """Round-robin assignment of the global view batch to ranks."""
    return views[rank::world]


def _accumulate_stats(state: TrainState, buf: GradientBuffer):
    """grad_accum[observed] += mean2d_grad_norm; obs_count[observed] += views (pipeline.py:191-192)."""
    state.grad_accum += buf.mean2d_grad_norm
    state.obs_count += buf.observed_count.to(torch.int32)


def train_step(state: TrainState, cam, gt, cfg: OptimConfig, spatial_scale: float = 1.0,
               buf: Optional[GradientBuffer] = None) -> StepStats:
    """One training iteration on one view (pipeline.py:178-193)."""
    cloud, medium = state.cloud, state.medium
    out = render(cloud, cam, medium=medium, mode="underwater")
    res, dL = total_loss_device(out.color, gt, medium, cfg.lambda_ssim, cfg.lambda_guide)
    if buf is None:
        buf = GradientBuffer(len(cloud), cloud.device)
    else:
        buf.zero_()
    backward_render(out, dL, cloud, medium, cfg.lambda_guide, buf=buf)
    flags = torch.stack([res[0], res[1], res[2], res[3], res[4],
                         buf.all_finite_device().double()]).tolist()
    l1, ds, lb, total, loss_ok, grad_ok = flags
    if loss_ok < 0.5:
        log.warning("iteration %d: non-finite loss, skipping update", state.iteration)
        return StepStats(l1, ds, lb, total, 1, True)
    if grad_ok < 0.5:
        log.warning("iteration %d: non-finite gradients, skipping update", state.iteration)
        return StepStats(l1, ds, lb, total, 1, True)
    _accumulate_stats(state, buf)
    apply_gradients(state, buf, cfg, spatial_scale)
    return StepStats(l1, ds, lb, total, 1, False)


class ViewShardedTrainer:
    """Data-parallel training over camera views, one process per GPU.

    Every rank holds the full cloud and optimizer state; a batch of views is
    split round-robin over the ranks, each rank renders and back-propagates
    its views into one flat gradient buffer (StepEngine), the buffers are
    summed with one NCCL all-reduce, and every rank applies the identical
    fused Adam step.  No host synchronisation inside the step.
    """

    def __init__(self, state: TrainState, cfg: OptimConfig, width: int, height: int,
                 spatial_scale: float = 1.0, views_per_rank: int = 1, group=None,
                 entry_capacity: int = 0):
        from .engine import StepEngine
        self.state = state
        self.engine = StepEngine(state, width, height, cfg, spatial_scale,
                                 max_views=views_per_rank, entry_capacity=entry_capacity,
                                 group=group)
        self.world, self.rank = self.engine.world, self.engine.rank

    def shard(self, views: Sequence) -> Sequence:
        """Views of this rank: round-robin over the global view list."""
        return shard_views(views, self.rank, self.world)

    def step(self, views: Sequence, sharded: bool = False):
        """One optimizer step over a batch of (camera, gt) views; ``views`` is
        the global batch (sharded here) unless ``sharded=True``.  Ground-truth
        images may be host arrays or device tensors."""
        mine = views if sharded else self.shard(views)
        return self.engine.step(mine)

    def step_async(self, views: Sequence, sharded: bool = False):
        """Pipelined form of :meth:`step`: launches this step (host images are
        copied on a side stream while the previous step's kernels run) and
        returns the stats of the previous one; :meth:`flush` returns the last."""
        mine = views if sharded else self.shard(views)
        return self.engine.step_async(mine)

    def flush(self):
        return self.engine.flush()

    def refresh_guidance(self, gt, **kw):
        """pipeline.py:204-208 for the replicated medium: rank 0 estimates from
        its last view (``gt`` = that view's ground truth) and every rank adopts
        the same float32 anchors (one 7-float broadcast), so the replicas stay
        identical.  Returns rank 0's estimate (None on the other ranks)."""
        eng = self.engine
        med = self.state.medium
        est = eng.refresh_guidance(gt, **kw) if self.rank == 0 else None
        if eng.dist is not None and self.world > 1:
            msg = torch.zeros(7, dtype=torch.float32, device=med.flat.device)
            if self.rank == 0:
                msg[:6] = med.flat[9:15]
                msg[6] = 0.0 if est.degenerate else 1.0
            src = eng.dist.get_global_rank(eng.group, 0) if eng.group is not None else 0
            eng.dist.broadcast(msg, src=src, group=eng.group)
            if self.rank != 0 and float(msg[6]) > 0.5:
                med.flat[9:15].copy_(msg[:6])
                med.mark_guidance()
        return est


@dataclass
class FitResult:
    state: TrainState
    log_rows: list
    engine: object


def fit(state: TrainState, cameras: Sequence, images: Sequence, train_idx: Sequence[int],
        cfg: OptimConfig, spatial_scale: float, rng, engine=None) -> FitResult:
    """The loop of pipeline.train (pipeline.py:169-233) on the sync-free StepEngine.

    Same schedule and random stream as the reference: views are drawn by
    popping a list reshuffled with ``rng`` whenever it runs empty (171-175),
    densify_and_prune every ``densify_interval`` iterations in
    [densify_from, densify_until] with the same ``rng`` (195-200), opacity
    reset every ``opacity_reset_interval`` (201-202) and the guidance refresh
    from the current view every ``refit_period`` (204-208).  Iterations that
    need none of those run pipelined (step i is launched before step i-1's
    record is read); the engine is flushed before each densify / reset /
    refit.  Ground-truth images are host arrays, copied on the engine's copy
    stream.  ``log_rows`` carries the reference's per-iteration log columns
    (pipeline.py:210-225) except the medium values, which are read only at
    flush points (``None`` elsewhere) to keep the loop free of host syncs."""
    from .engine import StepEngine
    from .optim import densify_and_prune, position_lr, reset_opacities
    W, H = int(cameras[0].width), int(cameras[0].height)
    eng = engine or StepEngine(state, W, H, cfg, spatial_scale)
    rows, order, pending = [], [], []

    def record(it, st):
        if st is None:
            return
        rows.append({"iter": it, "l1": st.l1, "d_ssim": st.d_ssim, "l_bs": st.l_bs,
                     "total": st.total, "skipped": st.skipped,
                     "lr_position": position_lr(it, cfg, spatial_scale)})

    for it in range(1, cfg.iterations + 1):
        state.iteration = it
        if not order:
            order = list(train_idx)
            rng.shuffle(order)
        view = order.pop()
        densify = (cfg.densify_from <= it <= cfg.densify_until
                   and it % cfg.densify_interval == 0)
        reset = bool(cfg.opacity_reset_interval) and it % cfg.opacity_reset_interval == 0
        refit = bool(cfg.refit_period) and it % cfg.refit_period == 0
        prev = eng.step_async([(cameras[view], images[view])])
        if pending:
            record(pending.pop(), prev)
        pending.append(it)
        if densify or reset or refit:
            st = eng.flush()
            record(pending.pop(), st)
            if not st.skipped:     # the reference `continue`s past a skipped step
                if densify:
                    densify_and_prune(state, cfg, spatial_scale, rng)
                if reset:
                    reset_opacities(state, cfg)
                if refit:
                    eng.refresh_guidance(images[view])
            m = state.medium.flat[:9].tolist()
            rows[-1].update({"num_gaussians": len(state.cloud), "medium": m})
    st = eng.flush()
    if pending:
        record(pending.pop(), st)
    return FitResult(state, rows, eng)
