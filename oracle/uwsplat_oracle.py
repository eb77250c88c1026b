"""CPU float64 oracle for the underwater-splatting hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the shipped package imports this file:
it is used by ``tests/``, by ``__graft_entry__.smoke()`` as the checker, and by
``bench.py`` for the ``cpu_baseline`` leg / ``--impl reference`` arm.

It is a restatement, in plain numpy, of the algorithm in the reference package
``uwsplat`` 0.1.0 (``/root/reference/pkg/src/uwsplat``).  Every function names
the reference lines it follows.  Arithmetic is float64 throughout, like the
reference, and the order of floating-point operations is kept wherever the
result feeds an integer decision (tile rectangles, depth order), so that the
oracle is bit-identical to the reference on the same machine.  The oracle is
pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``; checked by
``tests/test_oracle_golden.py``).

Third-party arithmetic the reference delegates: numpy (matmul / lexsort /
cumprod / add.at) and scipy (``special.expit`` = 1/(1+exp(-x)),
``ndimage.correlate1d`` with mode="constant").  numpy is used directly with
numpy primitives, except that the oracle calls the same scipy functions
(``expit``, ``correlate1d``) the reference calls, so it stays bit-identical.
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

# ---------------------------------------------------------------------------
# constants (reference: projection.py:21-26, rasterizer.py:27-29,
# scene.py:22,25-26, losses.py:23-26, medium.py:23)
# ---------------------------------------------------------------------------
SH_C0 = 0.28209479177387814
TILE = 16
DILATION = 0.3
FLOOR = 1.0 / 255.0
MIN_SIGMA = 3.0
CLAMP = 0.99
T_STOP = 1e-4
W_EPS = 1e-8
LOGISTIC_K = 0.1
SSIM_N = 11
SSIM_SIGMA = 1.5
SSIM_K1 = 0.01 ** 2
SSIM_K2 = 0.03 ** 2


def _sigmoid(x):
    """Logistic sigmoid as the reference evaluates it (projection.py:116).

    The reference calls ``scipy.special.expit`` (scipy>=1.10; 1.18.1 in this
    image), which is 1/(1+exp(-x)) with the C library ``exp``.  numpy's SIMD
    ``np.exp`` differs from it by 1 ulp on a few percent of inputs, so the
    oracle calls the same scipy function to stay bit-identical.
    """
    from scipy.special import expit
    return expit(np.asarray(x, dtype=np.float64))


def rotmat_from_quat(q):
    """wxyz quaternion -> rotation matrix; normalizes first (scene.py:32-48)."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = (q[..., i] for i in range(4))
    rows = [
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ]
    out = np.empty(q.shape[:-1] + (3, 3))
    for i in range(3):
        for j in range(3):
            out[..., i, j] = rows[i][j]
    return out


def logistic(depth):
    """z = 2 / (1 + exp(-0.1 d)) - 1 (medium.py:26-29)."""
    d = np.asarray(depth, dtype=np.float64)
    return 2.0 / (1.0 + np.exp(-LOGISTIC_K * d)) - 1.0


# ---------------------------------------------------------------------------
# preprocess (projection.py:89-199)
# ---------------------------------------------------------------------------
def _reach_radius(cov, peak):
    """Opacity-aware footprint radius (projection.py:89-97)."""
    a, b, c = cov[:, 0], cov[:, 1], cov[:, 2]
    half_tr = 0.5 * (a + c)
    det = a * c - b * b
    lam = half_tr + np.sqrt(np.maximum(half_tr * half_tr - det, 0.0))
    reach = 2.0 * np.log(np.maximum(255.0 * peak, 1.0))
    return np.sqrt(np.maximum(reach, MIN_SIGMA ** 2) * lam)


def project(cloud, cam):
    """Project every Gaussian; keep the visible ones in ascending source order.

    Follows projection.py:100-199 step for step.  Returns a namespace with the
    same field names as the reference ``ProjectedCloud``.
    """
    n = len(cloud.positions)
    out = SimpleNamespace(n_source=n)
    empty = dict(source_index=np.zeros(0, np.int64), mean2d=np.zeros((0, 2)),
                 cov2d=np.zeros((0, 3)), conic=np.zeros((0, 3)), depth=np.zeros(0),
                 radius=np.zeros(0), opacity=np.zeros(0), color=np.zeros((0, 3)),
                 color_clamped=np.zeros((0, 3), bool), t_view=np.zeros((0, 3)),
                 tx_clamped=np.zeros(0), ty_clamped=np.zeros(0),
                 x_clamp_mask=np.zeros(0, bool), x_clamp_sign=np.zeros(0),
                 y_clamp_mask=np.zeros(0, bool), y_clamp_sign=np.zeros(0),
                 rotmat=np.zeros((0, 3, 3)), scale=np.zeros((0, 3)),
                 cov3d=np.zeros((0, 3, 3)), quat_unit=np.zeros((0, 4)),
                 quat_norm=np.zeros(0))
    out.__dict__.update(empty)
    if n == 0:
        return out
    Rv = np.asarray(cam.R, np.float64)
    tv = np.asarray(cam.t, np.float64)
    xyz = np.asarray(cloud.positions, np.float32).astype(np.float64)
    view = xyz @ Rv.T + tv                                  # projection.py:112
    z_all = view[:, 2]
    peak_all = _sigmoid(np.asarray(cloud.opacity_logits, np.float32).astype(np.float64))
    alive = (z_all > cam.near) & (z_all < cam.far) & (peak_all >= FLOOR)   # :114-117
    cand = np.flatnonzero(alive)
    if cand.size == 0:
        return out

    view = view[cand]
    z = view[:, 2]
    lim_x = 1.3 * (0.5 * cam.width / cam.fx)                # :126-131
    lim_y = 1.3 * (0.5 * cam.height / cam.fy)
    u = view[:, 0] / z
    v = view[:, 1] / z
    u_c = np.clip(u, -lim_x, lim_x)
    v_c = np.clip(v, -lim_y, lim_y)
    xu = u_c * z
    yu = v_c * z

    quat = np.asarray(cloud.rotations, np.float32)[cand].astype(np.float64)   # :137-143
    qn = np.linalg.norm(quat, axis=1)
    qu = quat / qn[:, None]
    Rq = rotmat_from_quat(qu)
    sc = np.exp(np.asarray(cloud.log_scales, np.float32)[cand].astype(np.float64))
    Mq = Rq * sc[:, None, :]
    sig3 = Mq @ np.transpose(Mq, (0, 2, 1))

    rz = 1.0 / z                                            # :146-158
    rz2 = rz * rz
    Jac = np.zeros((cand.size, 2, 3))
    Jac[:, 0, 0] = cam.fx * rz
    Jac[:, 0, 2] = -cam.fx * xu * rz2
    Jac[:, 1, 1] = cam.fy * rz
    Jac[:, 1, 2] = -cam.fy * yu * rz2
    TJ = Jac @ Rv
    sig2 = TJ @ sig3 @ np.transpose(TJ, (0, 2, 1))
    ca = sig2[:, 0, 0] + DILATION
    cb = 0.5 * (sig2[:, 0, 1] + sig2[:, 1, 0])
    cc = sig2[:, 1, 1] + DILATION
    cov = np.stack([ca, cb, cc], axis=1)

    m2 = np.stack([cam.fx * u + cam.cx, cam.fy * v + cam.cy], axis=1)    # :160 (unclamped)
    rad = _reach_radius(cov, peak_all[cand])

    hit = ((m2[:, 0] + rad >= -0.5) & (m2[:, 0] - rad <= cam.width + 0.5)      # :164-169
           & (m2[:, 1] + rad >= -0.5) & (m2[:, 1] - rad <= cam.height + 0.5))
    keep = np.flatnonzero(hit)
    if keep.size == 0:
        return out

    det = ca * cc - cb * cb                                  # :174-175
    con = np.stack([cc / det, -cb / det, ca / det], axis=1)
    rows = cand[keep]
    feat = np.asarray(cloud.sh_coeffs, np.float32).reshape(n, -1, 3)[:, 0, :]
    rgb = np.maximum(feat.astype(np.float64) * SH_C0 + 0.5, 0.0)[rows]   # scene.py:136-139

    out.source_index = rows.astype(np.int64)
    out.mean2d = m2[keep]
    out.cov2d = cov[keep]
    out.conic = con[keep]
    out.depth = z[keep]
    out.radius = rad[keep]
    out.opacity = peak_all[cand][keep]
    out.color = rgb
    out.color_clamped = rgb <= 0.0
    out.t_view = view[keep]
    out.tx_clamped = xu[keep]
    out.ty_clamped = yu[keep]
    out.x_clamp_mask = (u != u_c)[keep]
    out.x_clamp_sign = np.sign(u[keep])
    out.y_clamp_mask = (v != v_c)[keep]
    out.y_clamp_sign = np.sign(v[keep])
    out.rotmat = Rq[keep]
    out.scale = sc[keep]
    out.cov3d = sig3[keep]
    out.quat_unit = qu[keep]
    out.quat_norm = qn[keep]
    return out


# ---------------------------------------------------------------------------
# tile rectangles + binning (projection.py:229-249, rasterizer.py:50-85)
# ---------------------------------------------------------------------------
def tile_rect(mean2d, radius, grid=None):
    """Inclusive tile rectangle (x0, y0, x1, y1) per footprint (projection.py:229-249)."""
    mean2d = np.asarray(mean2d, np.float64).reshape(-1, 2)
    radius = np.asarray(radius, np.float64).reshape(-1)
    lo_x = np.ceil(mean2d[:, 0] - radius - 0.5 - 1e-9)
    hi_x = np.floor(mean2d[:, 0] + radius - 0.5 + 1e-9)
    lo_y = np.ceil(mean2d[:, 1] - radius - 0.5 - 1e-9)
    hi_y = np.floor(mean2d[:, 1] + radius - 0.5 + 1e-9)
    r = np.stack([lo_x // TILE, lo_y // TILE, hi_x // TILE, hi_y // TILE], axis=1).astype(np.int64)
    if grid is not None:
        gx, gy = grid
        r[:, 0] = np.clip(r[:, 0], 0, gx - 1)
        r[:, 1] = np.clip(r[:, 1], 0, gy - 1)
        r[:, 2] = np.maximum(np.clip(r[:, 2], -1, gx - 1), r[:, 0] - 1)
        r[:, 3] = np.maximum(np.clip(r[:, 3], -1, gy - 1), r[:, 1] - 1)
    return r


def grid_dims(width, height):
    return (width + TILE - 1) // TILE, (height + TILE - 1) // TILE


def tile_lists(proj, width, height, tiles=None):
    """CSR tile lists sorted by (tile, depth, source) (rasterizer.py:50-85).

    Returns (offsets int64 (tiles+1,), entries int64 (E,)).  ``tiles``
    optionally restricts the emitted entries to a subset of tile ids (used
    for sampled CPU timing; offsets then describe only that subset).
    """
    gx, gy = grid_dims(width, height)
    n_tiles = gx * gy
    K = len(proj.depth)
    if K == 0:
        return np.zeros(n_tiles + 1, np.int64), np.zeros(0, np.int64)
    r = tile_rect(proj.mean2d, proj.radius, (gx, gy))
    rows_of = np.arange(K)
    if tiles is not None:
        # only footprints whose rectangle covers a requested tile can emit an
        # entry for it: enumerate those (same entries, same order, a fraction
        # of the memory at 4K)
        tl = np.asarray(tiles, np.int64)
        txs, tys = tl % gx, tl // gx
        hit = np.zeros(K, bool)
        for tx_, ty_ in zip(txs, tys):
            hit |= (r[:, 0] <= tx_) & (tx_ <= r[:, 2]) & (r[:, 1] <= ty_) & (ty_ <= r[:, 3])
        rows_of = np.nonzero(hit)[0]
        r = r[rows_of]
    wx = r[:, 2] - r[:, 0] + 1
    wy = r[:, 3] - r[:, 1] + 1
    cnt = np.maximum(wx, 0) * np.maximum(wy, 0)
    total = int(cnt.sum())
    if total == 0:
        return np.zeros(n_tiles + 1, np.int64), np.zeros(0, np.int64)
    local = np.repeat(np.arange(len(r)), cnt)
    first = np.cumsum(cnt) - cnt
    k = np.arange(total) - first[local]
    tid = (r[local, 1] + k // wx[local]) * gx + (r[local, 0] + k % wx[local])
    owner = rows_of[local]
    if tiles is not None:
        sel = np.isin(tid, np.asarray(tiles))
        owner, tid = owner[sel], tid[sel]
    perm = np.lexsort((proj.source_index[owner], proj.depth[owner], tid))
    owner = owner[perm]
    tid = tid[perm]
    counts = np.bincount(tid, minlength=n_tiles)
    offsets = np.zeros(n_tiles + 1, np.int64)
    offsets[1:] = np.cumsum(counts)
    return offsets, owner.astype(np.int64)


# ---------------------------------------------------------------------------
# forward compositing (rasterizer.py:148-251)
# ---------------------------------------------------------------------------
def _tile_pixels(tx, ty, width, height):
    x0, y0 = tx * TILE, ty * TILE
    x1, y1 = min(x0 + TILE, width), min(y0 + TILE, height)
    gy_, gx_ = np.meshgrid(np.arange(y0, y1) + 0.5, np.arange(x0, x1) + 0.5, indexing="ij")
    return (x0, x1, y0, y1), gx_.ravel(), gy_.ravel()


def _alpha_block(px, py, mean2d, conic, opac):
    """Raw and gated alpha for a (pixel x contributor) block (rasterizer.py:159-165)."""
    dx = px[:, None] - mean2d[None, :, 0]
    dy = py[:, None] - mean2d[None, :, 1]
    q = (-0.5 * (conic[None, :, 0] * dx * dx + conic[None, :, 2] * dy * dy)
         - conic[None, :, 1] * dx * dy)
    raw = opac[None, :] * np.exp(q)
    a = np.minimum(raw, CLAMP)
    a[raw < FLOOR] = 0.0
    return dx, dy, raw, a


def _transmittance(a):
    """T_i = prod_{j<i}(1 - a_j), T_1 = 1, and the live mask T_i >= 1e-4 (:166-169)."""
    om = 1.0 - a
    T = np.ones_like(a)
    if a.shape[1] > 1:
        T[:, 1:] = np.cumprod(om, axis=1)[:, :-1]
    return om, T, T >= T_STOP


def blend(px, py, mean2d, conic, color, opac, depth, far):
    """Front-to-back blend of one contributor list (rasterizer.py:148-178)."""
    P = px.shape[0]
    if mean2d.shape[0] == 0:
        return (np.zeros((P, 3)), np.full(P, far), np.zeros(P), np.ones(P),
                np.zeros(P, np.int32))
    _, _, _, a = _alpha_block(px, py, mean2d, conic, opac)
    om, T, live = _transmittance(a)
    w = a * T * live
    col = w @ color
    wsum = w.sum(axis=1)
    dnum = w @ depth
    tfin = np.prod(np.where(live, om, 1.0), axis=1)
    cnt = ((a > 0.0) & live).sum(axis=1).astype(np.int32)
    z = np.where(wsum > W_EPS, dnum / np.maximum(wsum, 1e-300), far)
    return col, z, wsum, tfin, cnt


def water(color_clean, depth_raw, attenuation, water_color, backscatter):
    """Attenuation + backscatter epilogue (rasterizer.py:244-251)."""
    zz = logistic(depth_raw)[..., None]
    att = np.exp(-np.asarray(attenuation, np.float32).astype(np.float64) * zz)
    bs = np.asarray(water_color, np.float32).astype(np.float64) * (
        1.0 - np.exp(-np.asarray(backscatter, np.float32).astype(np.float64) * zz))
    return color_clean * att + bs


def render(cloud, cam, medium=None, mode="clean", tiles=None, proj=None, bins=None):
    """Tiled render (rasterizer.py:188-241).  ``tiles`` restricts to a tile subset."""
    if mode not in ("clean", "underwater"):
        raise ValueError(f"unknown render mode {mode!r}")
    if mode == "underwater" and medium is None:
        raise ValueError("underwater mode requires medium parameters")
    H, W = cam.height, cam.width
    if proj is None:
        proj = project(cloud, cam)
    if bins is None:
        bins = tile_lists(proj, W, H, tiles=tiles)
    offsets, entries = bins
    gx, gy = grid_dims(W, H)
    color = np.zeros((H, W, 3))
    depth = np.full((H, W), float(cam.far))
    weight = np.zeros((H, W))
    tfin = np.ones((H, W))
    count = np.zeros((H, W), np.int32)
    tile_ids = range(gx * gy) if tiles is None else tiles
    for t in tile_ids:
        ty, tx = divmod(int(t), gx)
        (x0, x1, y0, y1), px, py = _tile_pixels(tx, ty, W, H)
        rows = entries[offsets[t]:offsets[t + 1]]
        c, z, w, tf, n = blend(px, py, proj.mean2d[rows], proj.conic[rows], proj.color[rows],
                               proj.opacity[rows], proj.depth[rows], float(cam.far))
        sh = (y1 - y0, x1 - x0)
        color[y0:y1, x0:x1] = c.reshape(sh + (3,))
        depth[y0:y1, x0:x1] = z.reshape(sh)
        weight[y0:y1, x0:x1] = w.reshape(sh)
        tfin[y0:y1, x0:x1] = tf.reshape(sh)
        count[y0:y1, x0:x1] = n.reshape(sh)
    out = SimpleNamespace(color=color, depth=depth, weight=weight, final_transmittance=tfin,
                          count=count, mode=mode, color_clean=None, proj=proj, bins=bins,
                          camera=cam)
    if mode == "underwater":
        out.color_clean = color
        out.color = water(color, depth, medium.attenuation, medium.water_color,
                          medium.backscatter)
    return out


def eval_pairs(proj, bins, width, height, tiles=None):
    """Number of (pixel, contributor) pairs up to each pixel's termination.

    P_pix in SURVEY §8(d): sum over pixels of the live-mask length, and R =
    sum over tiles of the max over its pixels of the consumed list prefix.
    """
    offsets, entries = bins
    gx, gy = grid_dims(width, height)
    p_pix = 0
    r_sum = 0
    for t in (range(gx * gy) if tiles is None else tiles):
        ty, tx = divmod(int(t), gx)
        _, px, py = _tile_pixels(tx, ty, width, height)
        rows = entries[offsets[t]:offsets[t + 1]]
        if rows.size == 0:
            continue
        _, _, _, a = _alpha_block(px, py, proj.mean2d[rows], proj.conic[rows], proj.opacity[rows])
        _, _, live = _transmittance(a)
        p_pix += int(live.sum())
        used = (a > 0) & live
        last = np.where(used.any(axis=1), used.shape[1] - np.argmax(used[:, ::-1], axis=1), 0)
        r_sum += int(last.max())
    return p_pix, r_sum


# ---------------------------------------------------------------------------
# losses (losses.py:40-160)
# ---------------------------------------------------------------------------
def _gauss_taps():
    x = np.arange(SSIM_N, dtype=np.float64) - (SSIM_N - 1) / 2.0
    k = np.exp(-0.5 * (x / SSIM_SIGMA) ** 2)
    return k / k.sum()


TAPS = _gauss_taps()


def _corr_axis(img, axis):
    """correlate1d(img, TAPS, axis, mode="constant") -- the scipy.ndimage call the
    reference makes (losses.py:64-65, scipy>=1.10; 1.18.1 here)."""
    from scipy.ndimage import correlate1d
    return correlate1d(img, TAPS, axis=axis, mode="constant")


def window_filter(img):
    """Valid-window separable Gaussian filter (losses.py:61-66)."""
    r = SSIM_N // 2
    return _corr_axis(_corr_axis(img, 0), 1)[r:-r, r:-r]


def window_adjoint(g, shape):
    """Adjoint of window_filter (losses.py:68-74)."""
    r = SSIM_N // 2
    full = np.zeros(shape)
    full[r:-r, r:-r] = g
    return _corr_axis(_corr_axis(full, 0), 1)


def l1(a, b):
    """Mean |a-b| and sign(a-b)/size (losses.py:40-49)."""
    d = np.asarray(a, np.float64) - np.asarray(b, np.float64)
    return float(np.mean(np.abs(d))), np.sign(d) / d.size


def dssim(a, b):
    """1 - mean SSIM and its gradient w.r.t. a (losses.py:83-123)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    flat = a.ndim == 2
    if flat:
        a, b = a[..., None], b[..., None]
    mu_a, mu_b = window_filter(a), window_filter(b)
    e_aa, e_bb, e_ab = window_filter(a * a), window_filter(b * b), window_filter(a * b)
    n1 = 2.0 * mu_a * mu_b + SSIM_K1
    n2 = 2.0 * (e_ab - mu_a * mu_b) + SSIM_K2
    d1 = mu_a * mu_a + mu_b * mu_b + SSIM_K1
    d2 = (e_aa - mu_a * mu_a) + (e_bb - mu_b * mu_b) + SSIM_K2
    S = (n1 * n2) / (d1 * d2)
    val = 1.0 - float(np.mean(S))
    g = -1.0 / S.size
    t_mu = (2.0 * mu_b * (n2 - n1)) / (d1 * d2) - 2.0 * mu_a * S * (1.0 / d1 - 1.0 / d2)
    t_aa = -S / d2
    t_ab = 2.0 * n1 / (d1 * d2)
    grad = window_adjoint(g * t_mu, a.shape)
    grad += 2.0 * a * window_adjoint(g * t_aa, a.shape)
    grad += b * window_adjoint(g * t_ab, a.shape)
    if flat:
        grad = grad[..., 0]
    return val, grad


def guidance(medium):
    """l1 distance of water params from their anchors (losses.py:126-137)."""
    if medium is None or getattr(medium, "water_color_guide", None) is None \
            or getattr(medium, "backscatter_guide", None) is None:
        return 0.0, np.zeros(3), np.zeros(3), False
    dw = np.asarray(medium.water_color, np.float32).astype(np.float64) - \
        np.asarray(medium.water_color_guide, np.float32).astype(np.float64)
    db = np.asarray(medium.backscatter, np.float32).astype(np.float64) - \
        np.asarray(medium.backscatter_guide, np.float32).astype(np.float64)
    return float(np.sum(np.abs(dw)) + np.sum(np.abs(db))), np.sign(dw), np.sign(db), True


def total_loss(rendered, gt, medium, lambda_ssim=0.3, lambda_guide=0.1):
    """Objective and dL/d(rendered) (losses.py:140-160); guidance not in the image grad."""
    v1, g1 = l1(rendered, gt)
    vs, gs = dssim(rendered, gt)
    lb, _, _, present = guidance(medium)
    total = (1.0 - lambda_ssim) * v1 + lambda_ssim * vs + lambda_guide * lb
    grad = (1.0 - lambda_ssim) * g1 + lambda_ssim * gs
    return dict(l1=v1, d_ssim=vs, l_bs=lb, total=total, lambda_ssim=lambda_ssim,
                lambda_guide=lambda_guide, guidance_present=present), grad


# ---------------------------------------------------------------------------
# backward (backward.py:124-344)
# ---------------------------------------------------------------------------
def tile_grads(px, py, mean2d, conic, color, opac, G):
    """Per-contributor screen-space gradients of one tile (backward.py:124-163)."""
    dx, dy, raw, a = _alpha_block(px, py, mean2d, conic, opac)
    om, T, live = _transmittance(a)
    w = a * T * live
    d_col = w.T @ G
    U = G @ color.T
    wU = w * U
    later = np.cumsum(wU[:, ::-1], axis=1)[:, ::-1] - wU     # sum_{j>i} w_j U_j
    d_a = U * T - later / om
    gate = live & (raw >= FLOOR) & (raw < CLAMP)
    dp = d_a * raw * gate
    ca, cb, cc = conic[:, 0][None, :], conic[:, 1][None, :], conic[:, 2][None, :]
    d_logit_raw = dp.sum(axis=0)
    d_m = np.stack([((ca * dx + cb * dy) * dp).sum(axis=0),
                    ((cb * dx + cc * dy) * dp).sum(axis=0)], axis=1)
    d_k = np.stack([(-0.5 * dx * dx * dp).sum(axis=0), (-dx * dy * dp).sum(axis=0),
                    (-0.5 * dy * dy * dp).sum(axis=0)], axis=1)
    return d_col, (1.0 - opac) * d_logit_raw, d_m, d_k


def _quat_chain(qu, qn, dR):
    """d rotation-matrix -> d raw quaternion (backward.py:166-181)."""
    w, x, y, z = qu[:, 0], qu[:, 1], qu[:, 2], qu[:, 3]
    g = lambda i, j: dR[:, i, j]  # noqa: E731
    dw = 2 * (z * (g(1, 0) - g(0, 1)) + y * (g(0, 2) - g(2, 0)) + x * (g(2, 1) - g(1, 2)))
    dx = 2 * (y * (g(0, 1) + g(1, 0)) + z * (g(0, 2) + g(2, 0)) + w * (g(2, 1) - g(1, 2))
              - 2 * x * (g(1, 1) + g(2, 2)))
    dy = 2 * (x * (g(0, 1) + g(1, 0)) + w * (g(0, 2) - g(2, 0)) + z * (g(1, 2) + g(2, 1))
              - 2 * y * (g(0, 0) + g(2, 2)))
    dz = 2 * (w * (g(1, 0) - g(0, 1)) + x * (g(0, 2) + g(2, 0)) + y * (g(1, 2) + g(2, 1))
              - 2 * z * (g(0, 0) + g(1, 1)))
    dq = np.stack([dw, dx, dy, dz], axis=1)
    radial = np.sum(dq * qu, axis=1, keepdims=True)
    return (dq - qu * radial) / qn[:, None]


def world_grads(proj, cam, d_mean2d, d_conic, d_color, d_logit, n):
    """Chain screen-space grads to the cloud parameters (backward.py:184-258).

    Returns a dict of float64 arrays indexed by source Gaussian.
    """
    g = dict(d_positions=np.zeros((n, 3)), d_log_scales=np.zeros((n, 3)),
             d_rotations=np.zeros((n, 4)), d_sh_coeffs=np.zeros((n, 1, 3)),
             d_opacity_logits=np.zeros(n), mean2d_grad_norm=np.zeros(n),
             observed=np.zeros(n, bool))
    K = len(proj.depth)
    if K == 0:
        return g
    src = proj.source_index
    k0, k1, k2 = proj.conic[:, 0], proj.conic[:, 1], proj.conic[:, 2]
    # conic -> cov2d: dX = -Y dY Y with the symmetric off-diagonal split
    Y = np.stack([np.stack([k0, k1], -1), np.stack([k1, k2], -1)], -2)
    dY = np.stack([np.stack([d_conic[:, 0], 0.5 * d_conic[:, 1]], -1),
                   np.stack([0.5 * d_conic[:, 1], d_conic[:, 2]], -1)], -2)
    dX = -Y @ dY @ Y
    G2 = dX.copy()
    G2[:, 0, 1] = G2[:, 1, 0] = dX[:, 0, 1]
    rz = 1.0 / proj.depth
    rz2 = rz * rz
    rz3 = rz2 * rz
    Jac = np.zeros((K, 2, 3))
    Jac[:, 0, 0] = cam.fx * rz
    Jac[:, 0, 2] = -cam.fx * proj.tx_clamped * rz2
    Jac[:, 1, 1] = cam.fy * rz
    Jac[:, 1, 2] = -cam.fy * proj.ty_clamped * rz2
    Rv = np.asarray(cam.R, np.float64)
    TJ = Jac @ Rv
    d_sig3 = np.transpose(TJ, (0, 2, 1)) @ G2 @ TJ
    dJ = 2.0 * (G2 @ TJ @ proj.cov3d) @ Rv.T
    dM = 2.0 * (d_sig3 @ (proj.rotmat * proj.scale[:, None, :]))
    d_ls = np.einsum("kij,kij->kj", proj.rotmat, dM) * proj.scale
    d_q = _quat_chain(proj.quat_unit, proj.quat_norm, dM * proj.scale[:, None, :])

    tx, ty = proj.t_view[:, 0], proj.t_view[:, 1]
    dxu = dJ[:, 0, 2] * (-cam.fx * rz2)
    dyu = dJ[:, 1, 2] * (-cam.fy * rz2)
    dz = (dJ[:, 0, 0] * (-cam.fx * rz2) + dJ[:, 0, 2] * (2.0 * cam.fx * proj.tx_clamped * rz3)
          + dJ[:, 1, 1] * (-cam.fy * rz2) + dJ[:, 1, 2] * (2.0 * cam.fy * proj.ty_clamped * rz3))
    lim_x = 1.3 * (0.5 * cam.width / cam.fx)
    lim_y = 1.3 * (0.5 * cam.height / cam.fy)
    dtx = np.where(proj.x_clamp_mask, 0.0, dxu)
    dty = np.where(proj.y_clamp_mask, 0.0, dyu)
    dz = dz + np.where(proj.x_clamp_mask, dxu * proj.x_clamp_sign * lim_x, 0.0)
    dz = dz + np.where(proj.y_clamp_mask, dyu * proj.y_clamp_sign * lim_y, 0.0)
    dtx = dtx + d_mean2d[:, 0] * cam.fx * rz
    dty = dty + d_mean2d[:, 1] * cam.fy * rz
    dz = dz - d_mean2d[:, 0] * cam.fx * tx * rz2 - d_mean2d[:, 1] * cam.fy * ty * rz2
    d_pos = np.stack([dtx, dty, dz], axis=1) @ Rv

    np.add.at(g["d_positions"], src, d_pos)
    np.add.at(g["d_log_scales"], src, d_ls)
    np.add.at(g["d_rotations"], src, d_q)
    np.add.at(g["d_opacity_logits"], src, d_logit)
    np.add.at(g["d_sh_coeffs"], src, (SH_C0 * d_color * (~proj.color_clamped))[:, None, :])
    ndc = d_mean2d * np.array([cam.width, cam.height]) * 0.5
    np.add.at(g["mean2d_grad_norm"], src, np.linalg.norm(ndc, axis=1))
    g["observed"][src] = True
    return g


def medium_grads(depth, color_clean, dL_dC, medium, lambda_guide):
    """Medium parameter gradients (backward.py:261-275)."""
    zz = logistic(depth)[..., None]
    bd = np.asarray(medium.attenuation, np.float32).astype(np.float64)
    binf = np.asarray(medium.water_color, np.float32).astype(np.float64)
    bb = np.asarray(medium.backscatter, np.float32).astype(np.float64)
    att = np.exp(-bd * zz)
    ebs = np.exp(-bb * zz)
    d_att = np.sum(dL_dC * color_clean * (-zz) * att, axis=(0, 1))
    d_wat = np.sum(dL_dC * (1.0 - ebs), axis=(0, 1))
    d_bsc = np.sum(dL_dC * binf * zz * ebs, axis=(0, 1))
    _, sw, sb, present = guidance(medium)
    if present and lambda_guide != 0.0:
        d_wat = d_wat + lambda_guide * sw
        d_bsc = d_bsc + lambda_guide * sb
    return d_att, d_wat, d_bsc


def backward(out, dL_dC, n_source, medium=None, lambda_guide=0.0, tiles=None, screen=False):
    """All parameter gradients for one view (backward.py:278-344)."""
    proj, (offsets, entries), cam = out.proj, out.bins, out.camera
    H, W = cam.height, cam.width
    dL_dC = np.asarray(dL_dC, np.float64)
    res = {}
    if out.mode == "underwater":
        if medium is None:
            raise ValueError("underwater backward requires medium parameters")
        zz = logistic(out.depth)[..., None]
        G_img = dL_dC * np.exp(-np.asarray(medium.attenuation, np.float32).astype(np.float64) * zz)
        res["d_attenuation"], res["d_water_color"], res["d_backscatter"] = \
            medium_grads(out.depth, out.color_clean, dL_dC, medium, lambda_guide)
    else:
        G_img = dL_dC
        res["d_attenuation"] = res["d_water_color"] = res["d_backscatter"] = np.zeros(3)
    K = len(proj.depth)
    d_col = np.zeros((K, 3))
    d_log = np.zeros(K)
    d_m = np.zeros((K, 2))
    d_k = np.zeros((K, 3))
    gx, gy = grid_dims(W, H)
    for t in (range(gx * gy) if tiles is None else tiles):
        rows = entries[offsets[t]:offsets[t + 1]]
        if rows.size == 0:
            continue
        ty, tx = divmod(int(t), gx)
        (x0, x1, y0, y1), px, py = _tile_pixels(tx, ty, W, H)
        G = G_img[y0:y1, x0:x1].reshape(-1, 3)
        dc, dl, dm, dk = tile_grads(px, py, proj.mean2d[rows], proj.conic[rows],
                                    proj.color[rows], proj.opacity[rows], G)
        np.add.at(d_col, rows, dc)
        np.add.at(d_log, rows, dl)
        np.add.at(d_m, rows, dm)
        np.add.at(d_k, rows, dk)
    if screen:
        res.update(screen_d_color=d_col, screen_d_logit=d_log, screen_d_mean2d=d_m,
                   screen_d_conic=d_k)
    res.update(world_grads(proj, cam, d_m, d_k, d_col, d_log, n_source))
    return res


# ---------------------------------------------------------------------------
# optimizer (optim.py:55-120, scene.py:132-134, 174-178)
# ---------------------------------------------------------------------------
def position_lr(iteration, lr_init=0.00016, lr_final=0.0000016, delay_mult=0.01,
                max_steps=30000, spatial_scale=1.0):
    """Sine-ramped log-linear position lr (optim.py:55-66)."""
    t = min(max(iteration / max_steps, 0.0), 1.0)
    ramp = delay_mult + (1.0 - delay_mult) * math.sin(0.5 * math.pi * t)
    return ramp * math.exp(math.log(lr_init) * (1 - t) + math.log(lr_final) * t) * spatial_scale


def adam(params, grads, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-15):
    """One bias-corrected Adam step in float64, stored float32 (optim.py:69-83).

    ``step`` is the counter AFTER increment.  Returns (params, m, v) float32.
    """
    g = np.asarray(grads, np.float64).reshape(params.shape)
    mm = beta1 * m.astype(np.float64) + (1 - beta1) * g
    vv = beta2 * v.astype(np.float64) + (1 - beta2) * g * g
    mh = mm / (1 - beta1 ** step)
    vh = vv / (1 - beta2 ** step)
    p = params.astype(np.float64) - lr * mh / (np.sqrt(vh) + eps)
    return p.astype(np.float32), mm.astype(np.float32), vv.astype(np.float32)


def renormalize(rot):
    """Quaternion renormalization with a 1e-12 floor (scene.py:132-134)."""
    nr = np.linalg.norm(rot.astype(np.float64), axis=1, keepdims=True)
    return (rot / np.maximum(nr, 1e-12)).astype(np.float32)


def clamp_medium(att, wat, bsc):
    """Medium box projection (scene.py:174-178)."""
    return (np.maximum(att, np.float32(0.0)).astype(np.float32),
            np.clip(wat, 0.0, 1.0).astype(np.float32),
            np.clip(bsc, 0.0, 5.0).astype(np.float32))


def densify_and_prune(arrays, m, v, grad_accum, obs_count, extent, rng,
                      grad_threshold=0.0002, percent_dense=0.01, min_opacity=0.1,
                      split_scale_factor=1.6):
    """Clone / split / prune (optim.py:132-198) on plain arrays.

    ``arrays``/``m``/``v`` map the five cloud fields to (n, ...) float32 arrays.
    Returns (new_arrays, new_m, new_v, (clones, splits, pruned)); nothing
    changes when the cloud would be emptied (optim.py:160-161).
    """
    n = arrays["positions"].shape[0]
    denom = np.maximum(obs_count.astype(np.float64), 1.0)                       # :143
    mean_grad = grad_accum.astype(np.float64) / denom                           # :144
    candidate = (mean_grad > grad_threshold) & (obs_count > 0)                  # :145
    max_scale = np.exp(arrays["log_scales"].astype(np.float64)).max(axis=1)     # :147
    small = max_scale <= percent_dense * extent                                 # :148
    prune = _sigmoid(arrays["opacity_logits"]) < min_opacity                    # :153-154
    clone = candidate & small & ~prune                                          # :149, 155
    split = candidate & ~small & ~prune                                         # :150, 156
    keep = ~(prune | split)                                                     # :157
    if not keep.any() and not split.any():
        return arrays, m, v, (0, 0, 0)
    fields = ("positions", "log_scales", "rotations", "sh_coeffs", "opacity_logits")
    parts = {f: [arrays[f][keep], arrays[f][clone]] for f in fields}            # :161-166
    n_split = int(split.sum())
    if n_split:                                                                 # :168-182
        idx = np.nonzero(split)[0]
        R = rotmat_from_quat(arrays["rotations"][idx])
        s = np.exp(arrays["log_scales"][idx].astype(np.float64))
        samples = rng.standard_normal((2, n_split, 3))
        for half in range(2):
            vec = samples[half] * s
            offs = np.empty((n_split, 3))
            for r in range(3):   # einsum("nij,nj->ni"): ((R0 v0 + R1 v1) + R2 v2)
                offs[:, r] = (R[:, r, 0] * vec[:, 0] + R[:, r, 1] * vec[:, 1]) + R[:, r, 2] * vec[:, 2]
            parts["positions"].append(
                (arrays["positions"][idx].astype(np.float64) + offs).astype(np.float32))
            parts["log_scales"].append((arrays["log_scales"][idx].astype(np.float64)
                                        - np.log(split_scale_factor)).astype(np.float32))
            for f in ("rotations", "sh_coeffs", "opacity_logits"):
                parts[f].append(arrays[f][idx])
    new = {f: np.concatenate(parts[f]).astype(np.float32) for f in fields}     # :184-186
    n_added = int(clone.sum()) + 2 * n_split                                    # :190-195
    new_m = {f: np.concatenate([m[f][keep], np.zeros((n_added,) + m[f].shape[1:], np.float32)])
             for f in fields}
    new_v = {f: np.concatenate([v[f][keep], np.zeros((n_added,) + v[f].shape[1:], np.float32)])
             for f in fields}
    return new, new_m, new_v, (int(clone.sum()), n_split, int(prune.sum()))


# ---------------------------------------------------------------------------
# guidance refresh: dark-pixel backscatter estimate (backscatter.py:52-270)
# ---------------------------------------------------------------------------
BS_WATER_BOX = (0.0, 1.0)          # backscatter.py:21
BS_BACKSCATTER_BOX = (0.0, 5.0)    # backscatter.py:22
BS_BB_STARTS = (0.1, 0.5, 1.0, 2.0, 4.0)   # backscatter.py:29
BS_LM_ITERS = 200                  # backscatter.py:30
BS_LM_TOL = 1e-10                  # backscatter.py:31


def bs_resize(image, depth, resized_height):
    """Downscale (backscatter.py:52-79, 244-249): bilinear colour, nearest depth,
    half-pixel centres, edge clamp.  Returns float64 (image, depth)."""
    image = np.asarray(image, dtype=np.float64)
    depth = np.asarray(depth, dtype=np.float64)
    h, w = image.shape[:2]
    th = min(resized_height, h)
    if th == h:
        return image, depth
    tw = max(1, round(w * th / h))
    # nearest: truncated centre coordinate, clamped to the last row/column
    rn = np.minimum((np.arange(th) + 0.5) * h / th, h - 1).astype(np.int64)
    cn = np.minimum((np.arange(tw) + 0.5) * w / tw, w - 1).astype(np.int64)
    depth = depth[rn][:, cn]
    # bilinear: source coordinate of each output centre, clipped into the image
    sy = np.clip((np.arange(th) + 0.5) * h / th - 0.5, 0, h - 1)
    sx = np.clip((np.arange(tw) + 0.5) * w / tw - 0.5, 0, w - 1)
    iy0 = np.floor(sy).astype(np.int64)
    ix0 = np.floor(sx).astype(np.int64)
    iy1 = np.minimum(iy0 + 1, h - 1)
    ix1 = np.minimum(ix0 + 1, w - 1)
    wy = (sy - iy0)[:, None, None]
    wx = (sx - ix0)[None, :, None]
    upper = image[iy0][:, ix0] * (1 - wx) + image[iy0][:, ix1] * wx
    lower = image[iy1][:, ix0] * (1 - wx) + image[iy1][:, ix1] * wx
    return upper * (1 - wy) + lower * wy, depth


def bs_linspace_labels(values, lo, hi, num):
    """cluster_range over linspace(lo, hi, num) (backscatter.py:82-97, numpy
    linspace: i*step + lo, last edge = hi).  Returns (labels, degenerate);
    raises ValueError where the reference raises DataError (non-increasing edges)."""
    edges = np.linspace(lo, hi, num)
    if edges.size < 2 or edges[-1] <= edges[0]:
        return np.zeros(np.shape(values), dtype=np.int64), True
    if np.any(np.diff(edges) <= 0):
        raise ValueError("cluster edges must be strictly increasing")
    lab = np.searchsorted(edges, values, side="right") - 1
    return np.clip(lab, 0, edges.size - 2), False


def bs_dark_pixels(image, depth, p_dark=0.01, edges_num=10):
    """select_dark_pixels (backscatter.py:100-132): in every depth cluster the
    ceil(p*size) smallest RGB sums, ties by raster order; returned in raster
    order.  Restated as one stable sort on (cluster, sum)."""
    image = np.maximum(np.asarray(image, dtype=np.float64), 0.0)
    depth = np.maximum(np.asarray(depth, dtype=np.float64), 0.0)
    z = depth.ravel()
    rgb = image.reshape(-1, 3)
    lab, degenerate = bs_linspace_labels(z, z.min(), z.max(), edges_num)
    lab = lab.ravel()
    sums = rgb.sum(axis=1)
    order = np.lexsort((np.arange(z.size), sums, lab))   # cluster, then sum, then index
    size = np.bincount(lab, minlength=1)
    start = np.concatenate([[0], np.cumsum(size)[:-1]])
    quota = np.maximum(1, np.ceil(p_dark * size).astype(np.int64))
    rank = np.arange(z.size) - start[lab[order]]
    pick = np.sort(order[rank < quota[lab[order]]])
    return z[pick], rgb[pick], degenerate


def _bs_sse(b_inf, b_b, z, y):
    r = b_inf * (1.0 - np.exp(-b_b * z)) - y
    return float(r @ r)


def bs_lm(z, y, start, lo, hi):
    """Box-projected Levenberg-Marquardt from one start (backscatter.py:142-175)."""
    p = np.clip(start, lo, hi).astype(np.float64)
    sse = _bs_sse(p[0], p[1], z, y)
    lam = 1e-3
    for _ in range(BS_LM_ITERS):
        ez = np.exp(-p[1] * z)
        jac = np.stack([1.0 - ez, p[0] * z * ez], axis=1)
        res = p[0] * (1.0 - ez) - y
        h = jac.T @ jac
        g = jac.T @ res
        moved = None
        for _ in range(12):
            damp = lam * np.diag(np.maximum(np.diag(h), 1e-12))
            try:
                d = np.linalg.solve(h + damp, -g)
            except np.linalg.LinAlgError:
                lam *= 10.0
                continue
            q = np.clip(p + d, lo, hi)
            q_sse = _bs_sse(q[0], q[1], z, y)
            if q_sse <= sse:
                moved = np.linalg.norm(q - p)
                p, sse = q, q_sse
                lam = max(lam / 3.0, 1e-12)
                break
            lam *= 3.0
        if moved is None:
            return p, sse
        if moved < BS_LM_TOL:
            return p, sse
    return p, sse


def bs_fit(z, y, box_binf=BS_WATER_BOX, box_bb=BS_BACKSCATTER_BOX):
    """fit_saturating_exponential (backscatter.py:178-208):
    (b_inf, b_b, rms, degenerate)."""
    z = np.asarray(z, dtype=np.float64).ravel()
    y = np.asarray(y, dtype=np.float64).ravel()
    lo = np.array([box_binf[0], box_bb[0]])
    hi = np.array([box_binf[1], box_bb[1]])
    if z.size < 3 or np.unique(z).size < 2:
        b_inf = float(np.clip(np.mean(y) if y.size else 0.0, *box_binf))
        rms = float(np.sqrt(np.mean((b_inf * (1 - np.exp(-hi[1] * z)) - y) ** 2))) if y.size else 0.0
        return b_inf, float(hi[1]), rms, True
    if np.max(np.abs(y)) == 0.0:
        return float(lo[0]), float(lo[1]), 0.0, False
    best, best_sse = None, np.inf
    for b0 in (float(np.mean(y)), float(np.max(y))):
        for bb0 in BS_BB_STARTS:
            p, sse = bs_lm(z, y, np.array([b0, bb0]), lo, hi)
            if sse < best_sse - 1e-15:
                best, best_sse = p, sse
    return float(best[0]), float(best[1]), float(np.sqrt(best_sse / z.size)), False


def bs_fit_points(dark_z, colors, intervals_num=25):
    """Per-interval per-channel lower envelope (backscatter.py:251-268): for each
    channel a list of (z, value) in interval order."""
    lab, degenerate = bs_linspace_labels(dark_z, dark_z.min(), dark_z.max(), intervals_num)
    pts = []
    for k in range(3):
        if degenerate:
            j = int(np.argmin(colors[:, k]))
            pts.append((np.array([dark_z[j]]), np.array([colors[j, k]])))
            continue
        zs, ys = [], []
        for i in range(intervals_num - 1):
            idx = np.nonzero(lab == i)[0]
            if idx.size:
                j = idx[int(np.argmin(colors[idx, k]))]
                zs.append(dark_z[j])
                ys.append(colors[j, k])
        pts.append((np.array(zs), np.array(ys)))
    return pts, degenerate


def estimate_backscatter(image, depth, p_dark=0.01, intervals_num=25, resized_height=300,
                         edges_num=10):
    """estimate_backscatter (backscatter.py:211-270).  Returns a namespace with
    water_color_est, backscatter_est, residual (float64 (3,)), degenerate,
    plus the intermediate dark set and fit points for stage checks."""
    image, depth = bs_resize(image, depth, resized_height)
    image = np.maximum(image, 0.0)
    depth = np.maximum(depth, 0.0)
    dz, rgb, degenerate = bs_dark_pixels(image, depth, p_dark, edges_num)
    out = SimpleNamespace(dark_z=dz, dark_rgb=rgb, points=None)
    if dz.size == 0 or degenerate:
        mean = image.reshape(-1, 3).mean(axis=0)
        out.water_color_est = np.clip(mean, *BS_WATER_BOX)
        out.backscatter_est = np.full(3, BS_BACKSCATTER_BOX[1])
        out.residual = np.zeros(3)
        out.degenerate = True
        return out
    pts, any_deg = bs_fit_points(dz, rgb, intervals_num)
    out.points = pts
    fits = [bs_fit(z, y) for z, y in pts]
    out.water_color_est = np.array([f[0] for f in fits])
    out.backscatter_est = np.array([f[1] for f in fits])
    out.residual = np.array([f[2] for f in fits])
    out.degenerate = bool(any_deg or any(f[3] for f in fits))
    return out
