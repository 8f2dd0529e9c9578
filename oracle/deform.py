"""Oracle: Gaussian deformation field F = D(H(G, t)) — PAPER.md §4.2.

TEST INFRASTRUCTURE (see oracle/__init__.py).  numpy float64.

Steps:
 1. normalise the canonical mean into the field's AABB (reading D1, D8);
 2. bilinear "interp ... 4 vertices" of every plane R_l(i,j) (Eq. 7, P:786-791,
    reading D2 align-corners knots, D3 temporal res fixed over scales);
 3. f_l = Hadamard product over the 6 planes, f_h = concat over scales
    (Eq. 7 "prod" / "cup", reading D4);
 4. f_d = phi_d(f_h) = ReLU(W_d f_h + b_d) (reading D5);
 5. dX = phi_x(f_d), dr = phi_r(f_d), ds = phi_s(f_d) (reading D6);
 6. (X', r', s') = (X + dX, r + dr, s + ds) (raw space, reading D7).
Opacity and SH are not deformed (G' = {X', s', r', sigma, C}) — unless the model carries the
colour and opacity decoders of P:1232 ("Color and Opacity's Deformation", the variant of Table 5):
 7. dC = phi_C(f_d), dalpha = phi_alpha(f_d); C' = C + dC over all (D+1)^2 x 3 SH coefficients
    and logit' = logit + dalpha (raw space, reading C1 — the same convention as D7).
"""
from __future__ import annotations

import numpy as np

# (i,j) in {(x,y),(x,z),(y,z),(x,t),(y,t),(z,t)}; axis 3 is time.
PLANES = ((0, 1), (0, 2), (1, 2), (0, 3), (1, 3), (2, 3))


def grid_coords(means, bmin, bmax, t):
    """World mean -> [0,1]^3 by the AABB, clamped (reading D1); u_t = t (D9).

    Returns u [N,4] float64 (x, y, z, t).
    """
    means = np.asarray(means, np.float64)
    bmin = np.asarray(bmin, np.float64)
    bmax = np.asarray(bmax, np.float64)
    u = (means - bmin) / (bmax - bmin)
    u = np.clip(u, 0.0, 1.0)
    ut = np.full((u.shape[0], 1), float(t), np.float64)
    return np.concatenate([u, ut], axis=1)


def bilinear(plane, ua, ub):
    """Bilinear interpolation over the 4 vertices (Eq. 7; reading D2).

    plane: [n_b][n_a][h] (knot k of an axis sits at u = k/(n-1)).
    ua, ub: [N] in [0,1].  Returns [N, h] float64.
    """
    P = np.asarray(plane, np.float64)
    nb, na = P.shape[0], P.shape[1]
    ga = np.asarray(ua, np.float64) * (na - 1)
    gb = np.asarray(ub, np.float64) * (nb - 1)
    i0 = np.minimum(np.floor(ga), na - 2).astype(np.int64)
    j0 = np.minimum(np.floor(gb), nb - 2).astype(np.int64)
    fa = (ga - i0)[:, None]
    fb = (gb - j0)[:, None]
    return ((1 - fa) * (1 - fb) * P[j0, i0] + fa * (1 - fb) * P[j0, i0 + 1]
            + (1 - fa) * fb * P[j0 + 1, i0] + fa * fb * P[j0 + 1, i0 + 1])


def hexplane_features(means, t, field):
    """f_h = U_l prod_{(i,j)} interp(R_l(i,j)) at (mu, t) — Eq. 7.

    field: paper_2310_08528_b200.inputs.Field (planes[l][p] = [n_b][n_a][h]).
    Returns f_h [N, h*L] float64, scale-major / channel-minor (reading D4).
    """
    u = grid_coords(means, field.bmin, field.bmax, t)
    feats = []
    for l in range(len(field.planes)):
        f_l = np.ones((u.shape[0], field.feat), np.float64)
        for p, (a, b) in enumerate(PLANES):
            f_l = f_l * bilinear(field.planes[l][p], u[:, a], u[:, b])
        feats.append(f_l)
    return np.concatenate(feats, axis=1)


def phi_d(f_h, mlp):
    """f_d = ReLU(W_d f_h + b_d) (reading D5).  Returns [N, W] float64."""
    W_d = np.asarray(mlp.w_d, np.float64)
    return np.maximum(0.0, f_h @ W_d.T + np.asarray(mlp.b_d, np.float64))


def decoder(f_h, mlp):
    """phi_d then the heads phi_x, phi_r, phi_s (readings D5, D6).

    Returns (dX [N,3], dr [N,4], ds [N,3]) float64.
    """
    f_d = phi_d(f_h, mlp)
    dX = f_d @ np.asarray(mlp.w_x, np.float64).T + np.asarray(mlp.b_x, np.float64)
    dr = f_d @ np.asarray(mlp.w_r, np.float64).T + np.asarray(mlp.b_r, np.float64)
    ds = f_d @ np.asarray(mlp.w_s, np.float64).T + np.asarray(mlp.b_s, np.float64)
    return dX, dr, ds


def colour_opacity_heads(f_h, mlp):
    """dC = phi_C(f_d) [N, 3K] (k-major, channel-minor: the SH layout) and dalpha = phi_alpha(f_d) [N]
    (reading C1: one Linear each).  Either is None when the model has no such head."""
    f_d = phi_d(f_h, mlp)
    dC = dA = None
    if getattr(mlp, "w_c", None) is not None:
        dC = f_d @ np.asarray(mlp.w_c, np.float64).T + np.asarray(mlp.b_c, np.float64)
    if getattr(mlp, "w_a", None) is not None:
        dA = f_d @ np.asarray(mlp.w_a, np.float64).T[:, 0] + np.asarray(mlp.b_a, np.float64)[0]
    return dC, dA


def deform_ref(scene, t, means=None, log_scales=None, quats=None, begin=0, end=None):
    """G' = G + F(G, t).

    Uses the canonical mean as the query position (reading D8).  Returns a dict
    of float64 arrays: means [N,3], quats [N,4] (raw), log_scales [N,3] (log).
    `begin/end` restrict to a contiguous Gaussian range (the sharded form).
    """
    X = np.asarray(scene.means if means is None else means, np.float64)
    r = np.asarray(scene.quats if quats is None else quats, np.float64)
    s = np.asarray(scene.log_scales if log_scales is None else log_scales, np.float64)
    end = X.shape[0] if end is None else end
    X, r, s = X[begin:end], r[begin:end], s[begin:end]
    f_h = hexplane_features(X, t, scene.field)
    dX, dr, ds = decoder(f_h, scene.mlp)
    out = {"means": X + dX, "quats": r + dr, "log_scales": s + ds}
    dC, dA = colour_opacity_heads(f_h, scene.mlp)
    if dC is not None:
        C = np.asarray(scene.sh, np.float64)[begin:end]
        out["sh"] = C + dC.reshape(C.shape)
    if dA is not None:
        out["opacity_logits"] = np.asarray(scene.opacity_logits, np.float64)[begin:end] + dA
    return out
