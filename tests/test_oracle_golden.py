"""Pin the CPU oracle against golden vectors produced by the reference itself.

CPU-only.  The fixtures come from ``tests/golden/make_golden.py`` (which runs
the unmodified reference ``uwsplat`` API).  Integer stages (visible set, tile
rectangles, sorted entries, tile ranges) must match exactly; the float64
oracle must reproduce float64 reference values to ~1e-12.
"""

import os

import numpy as np
import pytest

from golden_util import SCENES, load
from oracle import uwsplat_oracle as O


@pytest.fixture(params=SCENES, scope="module")
def scene(request):
    g = load(request.param)
    g.proj = O.project(g.cloud, g.cam)
    g.bins = O.tile_lists(g.proj, g.cam.width, g.cam.height)
    med = g.medium if g.mode == "underwater" else None
    g.out = O.render(g.cloud, g.cam, med, g.mode, proj=g.proj, bins=g.bins)
    return g


def test_projection_matches_reference(scene):
    d, p = scene.d, scene.proj
    np.testing.assert_array_equal(p.source_index, d["proj_source_index"])
    # feeds integer decisions: identical float64 operation order -> bit-exact
    np.testing.assert_array_equal(p.mean2d, d["proj_mean2d"])
    np.testing.assert_array_equal(p.depth, d["proj_depth"])
    np.testing.assert_array_equal(p.radius, d["proj_radius"])
    np.testing.assert_allclose(p.cov2d, d["proj_cov2d"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(p.conic, d["proj_conic"], rtol=1e-12, atol=0)
    np.testing.assert_array_equal(p.opacity, d["proj_opacity"])
    np.testing.assert_array_equal(p.color, d["proj_color"])
    np.testing.assert_array_equal(p.color_clamped, d["proj_color_clamped"])
    np.testing.assert_array_equal(p.x_clamp_mask, d["proj_x_clamp_mask"])
    np.testing.assert_array_equal(p.y_clamp_mask, d["proj_y_clamp_mask"])


def test_bins_bit_exact(scene):
    offs, ent = scene.bins
    np.testing.assert_array_equal(offs, scene.d["bins_offsets"])
    np.testing.assert_array_equal(ent, scene.d["bins_entries"].astype(np.int64))


def test_render_matches_reference(scene):
    d, out = scene.d, scene.out
    np.testing.assert_allclose(out.color, d["out_color"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(out.depth, d["out_depth"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(out.weight, d["out_weight"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(out.final_transmittance, d["out_final_transmittance"],
                               rtol=1e-10, atol=1e-15)
    np.testing.assert_array_equal(out.count, d["out_count"])
    if scene.mode == "underwater":
        np.testing.assert_allclose(out.color_clean, d["out_color_clean"], rtol=0, atol=1e-12)
    # the reference's all-N oracle agrees with its tiled path (SPEC acceptance 2)
    np.testing.assert_allclose(out.color, d["naive_color"], rtol=0, atol=1e-9)


def test_loss_matches_reference(scene):
    lam_s, lam_g = scene.lambdas
    bd, grad = O.total_loss(scene.d["out_color"], scene.gt, scene.medium, lam_s, lam_g)
    np.testing.assert_allclose([bd["l1"], bd["d_ssim"], bd["l_bs"], bd["total"]],
                               scene.d["loss"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(grad, scene.d["dL_dC"], rtol=1e-9, atol=1e-17)


def test_backward_matches_reference(scene):
    d = scene.d
    med = scene.medium if scene.mode == "underwater" else None
    g = O.backward(scene.out, d["dL_dC"], len(scene.cloud.positions), med, scene.lambdas[1])
    for f in ("d_positions", "d_log_scales", "d_rotations", "d_sh_coeffs", "d_opacity_logits",
              "mean2d_grad_norm", "d_attenuation", "d_water_color", "d_backscatter"):
        ref = d["grad_" + f]
        scale = max(np.abs(ref).max(), 1e-30)
        np.testing.assert_allclose(g[f], ref, rtol=1e-7, atol=1e-10 * scale, err_msg=f)
    np.testing.assert_array_equal(g["observed"], d["grad_observed"])


def test_adam_bit_exact(scene):
    """One apply_gradients step replayed from the reference's own gradients."""
    d = scene.d
    lrs = {"positions": O.position_lr(1), "log_scales": 0.005, "rotations": 0.001,
           "sh_coeffs": 0.0025, "opacity_logits": 0.05}
    new = {}
    for f, lr in lrs.items():
        p = d["in_" + f]
        z = np.zeros_like(p)
        new[f], m, v = O.adam(p, d["grad_d_" + f], z, z, 1, lr)
        np.testing.assert_array_equal(m, d["adam_m_" + f])
        np.testing.assert_array_equal(v, d["adam_v_" + f])
    new["rotations"] = O.renormalize(new["rotations"])
    for f in lrs:
        np.testing.assert_array_equal(new[f], d["adam_" + f], err_msg=f)
    if scene.medium is not None and scene.mode == "underwater":
        med = []
        for f in ("attenuation", "water_color", "backscatter"):
            p = d["medium_" + f]
            z = np.zeros_like(p)
            q, m, v = O.adam(p, d["grad_d_" + f], z, z, 1, 0.0025)
            med.append(q)
            np.testing.assert_array_equal(m, d["adam_m_" + f])
        for f, q in zip(("attenuation", "water_color", "backscatter"), O.clamp_medium(*med)):
            np.testing.assert_array_equal(q, d["adam_medium_" + f], err_msg=f)


def test_spec_kats():
    """Known answers from SPEC.md (§projection/rasterizer/medium examples)."""
    # logistic(10) = 2/(1+e^-1) - 1
    assert abs(O.logistic(10.0) - 0.46211715726000974) < 1e-15
    assert O.logistic(0.0) == 0.0
    # covariance of identity quaternion with log_scale (ln2,0,0) -> diag(4,1,1)
    R = O.rotmat_from_quat(np.array([[1.0, 0, 0, 0]]))[0]
    M = R * np.exp(np.array([np.log(2.0), 0, 0]))[None, :]
    np.testing.assert_allclose(M @ M.T, np.diag([4.0, 1, 1]), atol=1e-14)
    # sigmoid(ln 9) = 0.9
    assert abs(O._sigmoid(np.log(9.0)) - 0.9) < 1e-15
    # tile rect: tiny Gaussian inside one tile -> 1x1 span
    r = O.tile_rect(np.array([[8.0, 8.0]]), np.array([2.0]), (4, 4))[0]
    assert tuple(r) == (0, 0, 0, 0)
    # Gaussian at a 4-tile corner reaching 2 px across each boundary -> 2x2
    r = O.tile_rect(np.array([[16.0, 16.0]]), np.array([2.0]), (4, 4))[0]
    assert tuple(r) == (0, 0, 1, 1)
    # single opaque contributor at the pixel centre: C=(0.99,0,0), z=2
    c, z, w, tf, n = O.blend(np.array([0.5]), np.array([0.5]), np.array([[0.5, 0.5]]),
                             np.array([[1.0, 0, 1.0]]), np.array([[1.0, 0, 0]]),
                             np.array([1.0]), np.array([2.0]), 100.0)
    np.testing.assert_allclose(c[0], [0.99, 0, 0])
    assert z[0] == 2.0 and n[0] == 1
    # empty pixel -> far, water colour B_inf (1 - e^{-B_b z}) with remapped z
    c, z, w, tf, n = O.blend(np.array([0.5]), np.array([0.5]), np.zeros((0, 2)),
                             np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0), np.zeros(0), 100.0)
    assert z[0] == 100.0 and w[0] == 0.0 and tf[0] == 1.0
    # position lr endpoints
    assert abs(O.position_lr(0) - 0.00016 * 0.01) < 1e-18
    assert abs(O.position_lr(30000) - 0.0000016) < 1e-18


def test_opaque_scene_crossing_contributor():
    """The contributor that drives T below 1e-4 is still blended (rasterizer.py:167-171)."""
    g = load("opaque3k")
    tf = g.d["out_final_transmittance"]
    assert (tf < 1e-4).all()
    np.testing.assert_allclose(g.d["out_weight"] + tf, 1.0, atol=1e-13)


def test_densify_matches_reference():
    """oracle.densify_and_prune == reference densify_and_prune (same generator seed)."""
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "densify.npz"))
    f5 = ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits")
    arrays = {f: d["in_" + f] for f in f5}
    m = {f: d["in_m_" + f] for f in f5}
    v = {f: d["in_v_" + f] for f in f5}
    new, nm, nv, counts = O.densify_and_prune(arrays, m, v, d["in_grad_accum"], d["in_obs_count"],
                                              float(d["extent"]),
                                              np.random.default_rng(int(d["seed"])))
    assert counts == tuple(int(c) for c in d["counts"])
    for f in f5:
        np.testing.assert_array_equal(new[f], d["out_" + f], err_msg=f)
        np.testing.assert_array_equal(nm[f], d["out_m_" + f], err_msg=f)
        np.testing.assert_array_equal(nv[f], d["out_v_" + f], err_msg=f)
