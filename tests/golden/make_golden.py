"""Generate golden vectors from the REFERENCE implementation (uwsplat 0.1.0).

Run in the build container, where ``/root/reference`` exists:

    python tests/golden/make_golden.py

It imports the reference package straight from ``/root/reference/pkg/src`` and
runs its own public API (render / total_loss / backward_render /
apply_gradients / project_cloud / bin_and_sort) on small seeded scenes, then
stores inputs and outputs as ``tests/golden/<scene>.npz``.  These fixtures pin
the CPU oracle (``oracle/uwsplat_oracle.py``) and the CUDA path on machines
where the reference is not mounted (the GPU box).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _cloud_arrays(cloud):
    return dict(positions=cloud.positions.copy(), log_scales=cloud.log_scales.copy(),
                rotations=cloud.rotations.copy(), sh_coeffs=cloud.sh_coeffs.copy(),
                opacity_logits=cloud.opacity_logits.copy())


def _cam_arrays(cam):
    return dict(cam_wh=np.array([cam.width, cam.height], np.int64),
                cam_intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near, cam.far]),
                cam_R=cam.R.copy(), cam_t=cam.t.copy())


def _medium_arrays(m, prefix="medium_"):
    if m is None:
        return {}
    d = {prefix + "attenuation": m.attenuation.copy(), prefix + "water_color": m.water_color.copy(),
         prefix + "backscatter": m.backscatter.copy()}
    if m.has_guidance:
        d[prefix + "water_color_guide"] = m.water_color_guide.copy()
        d[prefix + "backscatter_guide"] = m.backscatter_guide.copy()
    return d


def scene_record(uw, name, cloud, cam, medium, gt, mode, lambda_ssim=0.3, lambda_guide=0.1):
    from uwsplat.optim import OptimConfig, apply_gradients
    from uwsplat.scene import TrainState

    rec = {}
    rec.update({"in_" + k: v for k, v in _cloud_arrays(cloud).items()})
    rec.update(_cam_arrays(cam))
    rec.update(_medium_arrays(medium))
    rec["gt"] = gt.astype(np.float64)
    rec["mode"] = np.array(mode)
    rec["lambdas"] = np.array([lambda_ssim, lambda_guide])

    proj = uw.project_cloud(cloud, cam)
    for f in ("source_index", "mean2d", "cov2d", "conic", "depth", "radius", "opacity", "color",
              "color_clamped", "tx_clamped", "ty_clamped", "x_clamp_mask", "y_clamp_mask"):
        rec["proj_" + f] = np.asarray(getattr(proj, f))
    bins = uw.bin_and_sort(proj, cam.width, cam.height)
    rec["bins_offsets"] = bins.offsets.astype(np.int64)
    rec["bins_entries"] = bins.entries.astype(np.int32)

    out = uw.render(cloud, cam, medium=medium if mode == "underwater" else None, mode=mode)
    for f in ("color", "depth", "weight", "final_transmittance", "count"):
        rec["out_" + f] = np.asarray(getattr(out, f))
    if mode == "underwater":
        rec["out_color_clean"] = out.color_clean

    bd, dL = uw.total_loss(out.color, gt, medium, lambda_ssim, lambda_guide)
    rec["loss"] = np.array([bd.l1, bd.d_ssim, bd.l_bs, bd.total])
    rec["dL_dC"] = dL
    buf = uw.backward_render(out, dL, cloud, medium if mode == "underwater" else None,
                             lambda_guide)
    for f in ("d_positions", "d_log_scales", "d_rotations", "d_sh_coeffs", "d_opacity_logits",
              "d_attenuation", "d_water_color", "d_backscatter", "mean2d_grad_norm", "observed"):
        rec["grad_" + f] = np.asarray(getattr(buf, f))

    # one Adam step at iteration 1 with the default config (extent 1.0)
    state = TrainState(cloud.copy(), (medium or uw.MediumParams.zero()).copy())
    state.iteration = 1
    cfg = OptimConfig()
    apply_gradients(state, buf, cfg, spatial_scale=1.0)
    for k, v in _cloud_arrays(state.cloud).items():
        rec["adam_" + k] = v
    for k, v in _medium_arrays(state.medium, "adam_medium_").items():
        rec[k] = v
    for k, slot in state.adam.items():
        rec["adam_m_" + k] = slot.m
        rec["adam_v_" + k] = slot.v

    # the reference's own all-Gaussians oracle on the same scene (tiled == naive)
    naive = uw.render_naive(cloud, cam, medium=medium if mode == "underwater" else None, mode=mode)
    rec["naive_color"] = naive.color
    rec["naive_depth"] = naive.depth

    np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
    print(f"{name}: N={len(cloud)} K={len(proj)} E={bins.entries.size} "
          f"{cam.width}x{cam.height} mode={mode} loss={bd.total:.6f}")


def main():
    sys.path.insert(0, REF)
    import uwsplat as uw
    from uwsplat.fixtures import front_camera, gradient_check_scene, random_cloud
    from uwsplat.scene import Camera, MediumParams

    # 1. the reference's canonical gradient-check scene (fixtures.py:42-72)
    cloud, cam, medium, gt = gradient_check_scene()
    scene_record(uw, "gradcheck", cloud, cam, medium, gt, "underwater")

    # 2. survey generator at a small, ragged size (128x96: partial tiles)
    N = 2000
    f = (1e4 / N) ** (1.0 / 3.0)
    rng = np.random.default_rng(0)
    cloud = random_cloud(N, rng, spread=4.0, scale_range=(0.15 * f, 0.6 * f))
    W, H = 136, 104
    cam = Camera.look_at((3, -2, -1), (0, 0, 12), width=W, height=H, fx=1.2 * W, fy=1.2 * W)
    medium = MediumParams((0.6, 0.45, 0.3), (0.2, 0.35, 0.5), (0.8, 1.0, 1.2),
                          water_color_guide=(0.25, 0.3, 0.45), backscatter_guide=(0.9, 1.0, 1.1))
    gt = np.random.default_rng(0).uniform(0, 1, (H, W, 3))
    scene_record(uw, "survey2k", cloud, cam, medium, gt, "underwater")

    # 3. clean mode, front camera, the reference bench cloud (cli.py:208-227 uses 500)
    rng = np.random.default_rng(3)
    cloud = random_cloud(500, rng)
    cam = front_camera(64, 64, focal=60.0)
    gt = np.random.default_rng(4).uniform(0, 1, (64, 64, 3))
    scene_record(uw, "clean500", cloud, cam, None, gt, "clean")

    # 4. opaque scene: every pixel terminates (crossing contributor blended)
    rng = np.random.default_rng(5)
    cloud = random_cloud(3000, rng, spread=1.5, scale_range=(0.5, 1.0),
                         opacity_range=(3.0, 6.0))
    cam = front_camera(32, 32, focal=40.0)
    medium = MediumParams((0.5, 0.4, 0.3), (0.25, 0.35, 0.45), (0.9, 1.1, 1.3))
    gt = np.random.default_rng(6).uniform(0, 1, (32, 32, 3))
    scene_record(uw, "opaque3k", cloud, cam, medium, gt, "underwater")


if __name__ == "__main__":
    main()
