"""Oracle: differentiable splatting S(M, G') forward — PAPER.md §3.1,
§4.1, with the tile rasterizer of [3dgs] the paper renders with (P:728,
P:919).  TEST INFRASTRUCTURE (see oracle/__init__.py).  numpy float64.

Steps; readings R1-R20 are listed in DESIGN.md §3:
  1 activate: s = exp(s'), q = r'/|r'| (w,x,y,z), o = sigmoid(logit)
  2 Sigma = R(q) S S^T R(q)^T                                    (Eq. 2)
  3 p = R_cam X' + t_cam, fixed summation order; cull p.z <= 0.2f  (R6)
  4-5 J of the affine approximation of the projection, x/z, y/z clamped (R4)
  6 Sigma2 = J W Sigma W^T J^T (2x2 block, W = R_cam) + 0.3 I    (Eq. 3; R3, R5)
  7 det, conic = Sigma2^-1; cull det <= 0                         (Eq. 1; R2)
  8 radius = ceil(3 sqrt(lambda_1))                               (R7)
  9 mean2d = (fx x/z + cx, fy y/z + cy)                           (R12)
 10 tile rect [x0,x1) x [y0,y1) (16x16 tiles, truncating rule); cull if empty (R8)
 11 depth key = IEEE bits of fp32(p.z)                            (R13)
 12 colour = max(0, SH(d) + 0.5), d = X' - campos normalised      (R10, R11)
 13 instances (tile, key, index) sorted lexicographically; per-tile ranges (R14)
 14 per pixel, front-to-back over its tile's list:                (Eq. 4; R1, R9)
      power = -1/2 (A dx^2 + C dy^2) - B dx dy ; skip if power > 0
      alpha = min(0.99f, o e^power) ; skip if alpha < 1/255
      T' = T (1 - alpha) ; stop (not added) if T' < 1e-4f
      C += c alpha T ; T = T'          pixel = C + T bg            (R17)
 15 brute force: per pixel over all kept Gaussians sorted by (key, index).
Discontinuous thresholds use the fp32-representable constants (§8(c)).
"""
from __future__ import annotations

import numpy as np

from .sh import sh_to_rgb

TILE = 16
NEAR = float(np.float32(0.2))                 # R6: keep p.z > 0.2f
ALPHA_MIN = float(np.float32(1.0 / 255.0))    # R9: skip alpha < 1/255
T_MIN = float(np.float32(1e-4))               # R9: stop when T' < 1e-4f
ALPHA_MAX = float(np.float32(0.99))           # R9: alpha = min(0.99f, .)
DILATION = 0.3                                # R5: +0.3 px^2 low-pass
LAMBDA_FLOOR = 0.1                            # R7
FOV_CLAMP = 1.3                               # R4
BAND_PX = 1e-5                                # §8(c.5) boundary-Gaussian band
BAND_REL = 1e-4                               # §8(c.5) pixel decision band


def tile_grid(width, height):
    return (width + TILE - 1) // TILE, (height + TILE - 1) // TILE


# ---------------------------------------------------------------- step 1
def activate(log_scales, quats, opacity_logits):
    """s = exp(s'), q = r'/|r'|, o = sigmoid(logit) (reading D7)."""
    s = np.exp(np.asarray(log_scales, np.float64))
    q = np.asarray(quats, np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    o = 1.0 / (1.0 + np.exp(-np.asarray(opacity_logits, np.float64)))
    return s, q, o


# ---------------------------------------------------------------- step 2
def quat_to_rotmat(q):
    """Rotation matrix of a unit quaternion (w, x, y, z) (reading D10). [N,3,3]."""
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((q.shape[0], 3, 3), np.float64)
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def covariance3d(s, q):
    """Sigma = R S S^T R^T (Eq. 2). s [N,3] (activated), q [N,4] unit."""
    R = quat_to_rotmat(q)
    M = R * s[:, None, :]                 # R S
    return M @ np.transpose(M, (0, 2, 1))


# ---------------------------------------------------------------- step 3
def view_transform(X, cam):
    """p = R_cam X + t_cam with p_c = ((r_c0 x + r_c1 y) + r_c2 z) + t_c (§8(c.2) 3).

    X fp32 values promoted; products of fp32 values are exact in fp64, so this
    is the fixed-order definition the depth key is formed from.
    """
    X = np.asarray(X, np.float64)
    R = np.asarray(cam.R, np.float64)
    t = np.asarray(cam.t, np.float64)
    p = np.empty_like(X)
    for c in range(3):
        p[:, c] = ((R[c, 0] * X[:, 0] + R[c, 1] * X[:, 1]) + R[c, 2] * X[:, 2]) + t[c]
    return p


# ---------------------------------------------------------------- steps 4-5
def jacobian(p, cam):
    """J of the affine approximation of the perspective map (Eq. 3).

    x/z and y/z clamped to +-1.3 tan(fov/2) before forming J (reading R4).
    Returns J [N,2,3].
    """
    tan_x = cam.width / (2.0 * cam.fx)
    tan_y = cam.height / (2.0 * cam.fy)
    z = p[:, 2]
    xt = np.clip(p[:, 0] / z, -FOV_CLAMP * tan_x, FOV_CLAMP * tan_x) * z
    yt = np.clip(p[:, 1] / z, -FOV_CLAMP * tan_y, FOV_CLAMP * tan_y) * z
    J = np.zeros((p.shape[0], 2, 3), np.float64)
    J[:, 0, 0] = cam.fx / z
    J[:, 0, 2] = -cam.fx * xt / (z * z)
    J[:, 1, 1] = cam.fy / z
    J[:, 1, 2] = -cam.fy * yt / (z * z)
    return J


# ---------------------------------------------------------------- step 6
def cov2d(J, cam, Sigma):
    """Sigma' = J W Sigma W^T J^T, 2x2 block (Eq. 3; R3), + 0.3 I (R5).

    Returns (a, b, c) = (Sigma2_00 + 0.3, Sigma2_01, Sigma2_11 + 0.3).
    """
    W = np.asarray(cam.R, np.float64)
    T = J @ W                                       # [N,2,3]
    S2 = T @ Sigma @ np.transpose(T, (0, 2, 1))     # [N,2,2]
    return S2[:, 0, 0] + DILATION, S2[:, 0, 1], S2[:, 1, 1] + DILATION



# ---------------------------------------------------------------- steps 8, 10
def radius_from_cov2d(a, b, c):
    """lambda_1 = mid + sqrt(max(0.1, mid^2 - det)); radius = ceil(3 sqrt(lambda_1)) (R7).

    Returns (lambda_1, 3 sqrt(lambda_1), radius) as float64 arrays.
    """
    det = a * c - b * b
    mid = 0.5 * (a + c)
    lam1 = mid + np.sqrt(np.maximum(LAMBDA_FLOOR, mid * mid - det))
    three_sqrt = 3.0 * np.sqrt(lam1)
    return lam1, three_sqrt, np.ceil(three_sqrt)


def tile_rect(mx, my, radius, gx, gy):
    """[3dgs] truncating tile rect of the radius box, clamped to the grid (R8).

    x0 = min(gx, max(0, trunc((m.x - r)/16))), x1 = min(gx, max(0, trunc((m.x + r + 15)/16))).
    """
    def trunc_clamp(v, g):
        v = np.where(np.isfinite(v), v, 0.0)
        return np.minimum(g, np.maximum(0, np.trunc(v))).astype(np.int64)

    return (trunc_clamp((mx - radius) / TILE, gx), trunc_clamp((my - radius) / TILE, gy),
            trunc_clamp((mx + radius + TILE - 1) / TILE, gx),
            trunc_clamp((my + radius + TILE - 1) / TILE, gy))


def sh_colour(X, sh, degree, cam):
    """rgb from SH at d = normalize(X' - campos), campos = -R^T t (R10, R11)."""
    R = np.asarray(cam.R, np.float64)
    t = np.asarray(cam.t, np.float64)
    campos = -R.T @ t
    d = np.asarray(X, np.float64) - campos
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    return sh_to_rgb(sh, d, degree)


def _near_multiple(v, period, band):
    r = np.mod(v, period)
    return (r < band) | (period - r < band)


def preprocess_ref(means, log_scales, quats, opacity_logits, sh, sh_degree, cam):
    """Per-Gaussian projection, culling and binning geometry (steps 1-12).

    Returns a dict of per-Gaussian arrays (length N):
      kept (bool), p (cam-space [N,3]), depth_key (uint32, 0 if culled), radius (int),
      rect (int [N,4] x0,y0,x1,y1), tiles_touched (int), mean2d [N,2], conic [N,3]
      (A, B, C), opacity, rgb [N,3], lambda1, boundary (bool, §8(c.5)).
    Culled Gaussians have radius 0, tiles_touched 0 and rect zeros.
    """
    N = np.asarray(means).shape[0]
    gx, gy = tile_grid(cam.width, cam.height)
    s, q, o = activate(log_scales, quats, opacity_logits)
    Sigma = covariance3d(s, q)
    p = view_transform(means, cam)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        in_front = p[:, 2] > NEAR
        J = jacobian(p, cam)
        a, b, c = cov2d(J, cam, Sigma)
        det = a * c - b * b
        ok = in_front & (det > 0)
        conic = np.stack([c / det, -b / det, a / det], axis=1)
        lam1, three_sqrt, radius = radius_from_cov2d(a, b, c)
        mx = cam.fx * p[:, 0] / p[:, 2] + cam.cx
        my = cam.fy * p[:, 1] / p[:, 2] + cam.cy
        x0, y0, x1, y1 = tile_rect(mx, my, radius, gx, gy)
    touched = (x1 - x0) * (y1 - y0)
    kept = ok & (touched > 0)
    zkey = np.where(kept, p[:, 2], 1.0).astype(np.float32).view(np.uint32)
    rgb = sh_colour(means, sh, sh_degree, cam)
    boundary = (_near_multiple(mx - radius, TILE, BAND_PX) | _near_multiple(mx + radius + TILE - 1, TILE, BAND_PX)
                | _near_multiple(my - radius, TILE, BAND_PX) | _near_multiple(my + radius + TILE - 1, TILE, BAND_PX)
                | _near_multiple(three_sqrt, 1.0, BAND_PX) | (np.abs(p[:, 2] - NEAR) < 1e-6))
    boundary &= in_front | (np.abs(p[:, 2] - NEAR) < 1e-6)
    z = np.zeros(N, np.int64)
    return {
        "kept": kept,
        "p": p,
        "depth_key": np.where(kept, zkey, 0).astype(np.uint32),
        "radius": np.where(kept, radius, 0).astype(np.int64),
        "rect": np.stack([np.where(kept, x0, z), np.where(kept, y0, z),
                          np.where(kept, x1, z), np.where(kept, y1, z)], axis=1),
        "tiles_touched": np.where(kept, touched, 0).astype(np.int64),
        "mean2d": np.stack([mx, my], axis=1),
        "conic": conic,
        "opacity": o,
        "rgb": rgb,
        "lambda1": lam1,
        "cov2d": np.stack([a, b, c], axis=1),
        "boundary": boundary,
    }


# ---------------------------------------------------------------- step 13
def bin_ref(pre, cam):
    """Tile instances (tile = ty*gx + tx, key, index), lexicographically sorted.

    Returns (tiles [M] int64, gids [M] int64, ranges [n_tiles, 2] int64 [start,end)).
    """
    gx, gy = tile_grid(cam.width, cam.height)
    tiles, keys, gids = [], [], []
    idx = np.nonzero(pre["kept"])[0]
    rect = pre["rect"]
    for i in idx:
        x0, y0, x1, y1 = rect[i]
        for ty in range(y0, y1):
            for tx in range(x0, x1):
                tiles.append(ty * gx + tx)
                keys.append(int(pre["depth_key"][i]))
                gids.append(int(i))
    tiles = np.asarray(tiles, np.int64)
    keys = np.asarray(keys, np.int64)
    gids = np.asarray(gids, np.int64)
    order = np.lexsort((gids, keys, tiles))
    tiles, gids = tiles[order], gids[order]
    t_ids = np.arange(gx * gy)
    ranges = np.stack([np.searchsorted(tiles, t_ids, "left"),
                       np.searchsorted(tiles, t_ids, "right")], axis=1)
    return tiles, gids, ranges


def tile_list_ref(pre, cam, tile):
    """Step 13 for ONE tile: the kept Gaussians whose rect contains `tile`, sorted by (depth key,
    index) — the slice bin_ref gives that tile, without building all instances (large configs)."""
    gx, _ = tile_grid(cam.width, cam.height)
    ty, tx = divmod(int(tile), gx)
    r = pre["rect"]
    hit = pre["kept"] & (r[:, 0] <= tx) & (tx < r[:, 2]) & (r[:, 1] <= ty) & (ty < r[:, 3])
    idx = np.nonzero(hit)[0]
    return idx[np.lexsort((idx, pre["depth_key"][idx].astype(np.int64)))]


# ---------------------------------------------------------------- step 14
def composite(pre, order, px, py, bg, flags=None):
    """Front-to-back alpha blending (Eq. 4) of Gaussians `order` at pixels (px, py).

    Vectorised over pixels only; the loop over Gaussians is the sequential
    per-pixel recursion.  Returns (rgb [P,3], T [P], n_contrib [P], flagged [P]).
    `order` is either one list shared by all pixels or, for brute force, a
    list with a per-pixel inclusion mask (tuples (gid, mask)).
    """
    P = px.shape[0]
    T = np.ones(P)
    C = np.zeros((P, 3))
    done = np.zeros(P, bool)
    ncon = np.zeros(P, np.int64)
    flagged = np.zeros(P, bool)
    m, cn, o, rgb = pre["mean2d"], pre["conic"], pre["opacity"], pre["rgb"]
    for item in order:
        if isinstance(item, tuple):
            g, incl = item
        else:
            g, incl = item, None
        dx = m[g, 0] - px
        dy = m[g, 1] - py
        A, B, Cc = cn[g]
        power = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy
        active = ~done if incl is None else (~done & incl)
        with np.errstate(over="ignore"):
            alpha = np.minimum(ALPHA_MAX, o[g] * np.exp(power))
        cand = active & ~(power > 0)
        flagged |= cand & (np.abs(alpha - ALPHA_MIN) <= BAND_REL * ALPHA_MIN)
        use = cand & ~(alpha < ALPHA_MIN)
        test_T = T * (1.0 - alpha)
        flagged |= use & (np.abs(test_T - T_MIN) <= BAND_REL * T_MIN)
        stop = use & (test_T < T_MIN)
        done |= stop
        add = use & ~stop
        C += np.where(add[:, None], rgb[g][None, :] * (alpha * T)[:, None], 0.0)
        T = np.where(add, test_T, T)
        ncon += add
        if done.all():
            break
    return C + T[:, None] * np.asarray(bg, np.float64)[None, :], T, ncon, flagged


def _tile_pixels(tile, gx, W, H):
    ty, tx = divmod(int(tile), gx)
    xs = np.arange(tx * TILE, min(W, tx * TILE + TILE))
    ys = np.arange(ty * TILE, min(H, ty * TILE + TILE))
    py, px = np.meshgrid(ys, xs, indexing="ij")
    return px.ravel(), py.ravel()


def render_ref(deformed, opacity_logits, sh, sh_degree, cam, tiles_subset=None, pre=None, full_bins=True,
               bins=None):
    """I = S(M, G'): preprocess, bin/sort, per-tile blend (tiled oracle).

    deformed: dict with means, log_scales, quats (raw, as written by deform).
    tiles_subset: optional iterable of tile ids to blend (others left NaN).
    Returns dict: image [3,H,W], final_T [H,W], n_contrib [H,W], flagged [H,W]
    (decision within relative 1e-4 of a threshold, or tile touched by a
    boundary Gaussian), plus the preprocess dict and (tiles, gids, ranges).
    full_bins=False (with tiles_subset): per-tile lists from tile_list_ref only, for configs where
    building every instance is too slow; (tiles, gids, ranges) are then None.
    bins: (tiles, gids, ranges) of bin_ref(pre, cam) computed earlier (several processes blending the
    tiles of one frame share one binning); same values as computing them here.
    """
    W, H = cam.width, cam.height
    gx, gy = tile_grid(W, H)
    if pre is None:
        pre = preprocess_ref(deformed["means"], deformed["log_scales"], deformed["quats"],
                             opacity_logits, sh, sh_degree, cam)
    if bins is not None:
        tiles, gids, ranges = bins
    elif full_bins or tiles_subset is None:
        tiles, gids, ranges = bin_ref(pre, cam)
    else:
        tiles = gids = ranges = None
    img = np.full((3, H, W), np.nan)
    fT = np.full((H, W), np.nan)
    ncon = np.full((H, W), -1, np.int64)
    flag = np.zeros((H, W), bool)
    if gids is not None:
        bnd_tiles = set(tiles[pre["boundary"][gids]].tolist()) if gids.size else set()
    todo = range(gx * gy) if tiles_subset is None else tiles_subset
    for tile in todo:
        px, py = _tile_pixels(tile, gx, W, H)
        if gids is not None:
            s, e = ranges[tile]
            lst = gids[s:e]
        else:
            lst = tile_list_ref(pre, cam, tile)
            if pre["boundary"][lst].any():
                bnd_tiles = {tile}
            else:
                bnd_tiles = set()
        rgb, T, nc, fl = composite(pre, lst, px.astype(np.float64), py.astype(np.float64), cam.bg)
        img[:, py, px] = rgb.T
        fT[py, px] = T
        ncon[py, px] = nc
        flag[py, px] = fl | (tile in bnd_tiles)
    return {"image": img, "final_T": fT, "n_contrib": ncon, "flagged": flag, "pre": pre,
            "tiles": tiles, "gids": gids, "ranges": ranges}


# ---------------------------------------------------------------- step 15
def render_ref_bruteforce(deformed, opacity_logits, sh, sh_degree, cam, rect_predicate=True):
    """Per-pixel compositing over ALL kept Gaussians sorted by (depth key, index).

    With rect_predicate, Gaussian i is included at pixel p only if tile(p) is
    in rect_i (the [3dgs] binning rule R8); without it, every kept Gaussian
    is composited at every pixel (valid when truncation cannot bind, §8(c.2) 15).
    Returns image [3,H,W], final_T, n_contrib.
    """
    W, H = cam.width, cam.height
    gx, _ = tile_grid(W, H)
    pre = preprocess_ref(deformed["means"], deformed["log_scales"], deformed["quats"],
                         opacity_logits, sh, sh_degree, cam)
    idx = np.nonzero(pre["kept"])[0]
    order = idx[np.lexsort((idx, pre["depth_key"][idx].astype(np.int64)))]
    py, px = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    px, py = px.ravel(), py.ravel()
    ptx, pty = px // TILE, py // TILE
    if rect_predicate:
        rect = pre["rect"]
        items = [(g, (ptx >= rect[g, 0]) & (ptx < rect[g, 2]) & (pty >= rect[g, 1]) & (pty < rect[g, 3]))
                 for g in order]
    else:
        items = list(order)
    rgb, T, nc, _ = composite(pre, items, px.astype(np.float64), py.astype(np.float64), cam.bg)
    return {"image": rgb.T.reshape(3, H, W), "final_T": T.reshape(H, W),
            "n_contrib": nc.reshape(H, W), "pre": pre}
