"""Oracle: the training-side gradients of the 4D-GS frame — PAPER.md §4.3 "L = |I^ - I| +
L_tv", back through the splatting S (the [3dgs] "differentiable" rasterizer) and the
deformation field F (Eq. 7).  TEST INFRASTRUCTURE (see oracle/__init__.py).

How it is computed (the plain route, no hand-derived chain rule): the forward of oracle/deform.py and
oracle/render.py is restated here in PyTorch CPU float64 ops, step for step in the same order, and
torch.autograd differentiates it.  Every discontinuous decision of the forward — the near cull, the
tile rect and therefore the per-tile lists, the depth order, the "power > 0" and "alpha < 1/255" skips,
the "T' < 1e-4" stop, the 0.99 clamp and the colour clamp at 0, the ReLU of phi_d, the AABB clamp of
the grid coordinates and the knot index of every bilinear lookup — is taken on DETACHED values, exactly
as the numpy forward takes it; the gradient is the derivative of the frame with those decisions held
fixed (the [3dgs] convention: "exact for the clamp-inactive region").

Readings (listed in DESIGN.md §3):
  B1  L_tv ("grid-based total-variational loss", garbled otherwise): the mean, over every plane
      of every scale, every channel and both grid directions, of the squared differences of adjacent
      grid entries, pooled into one mean (worked example S:238).
  B2  |I^ - I|: the mean over all pixels and the 3 channels of the absolute difference (SPEC
      S:349 "mean absolute per-channel error"); its derivative is sign(I^ - I) / (3 H W), 0 at equality.
  B3  L = L1 + w_tv L_tv with w_tv a caller parameter (the paper gives no weight).
  B4  gradients flow into the canonical Gaussian parameters (means, log-scales, raw quaternions, opacity
      logits, SH), the six planes of every scale and all MLP weights and biases; t is not a parameter.
      dL/dX has both the additive path X' = X + dX and the query-position path u(X).

Pinned by tests/test_oracle_backward.py: the torch forward equals the numpy forward oracle; every
gradient equals central finite differences of the numpy forward (fp64, no decision flips in the
stencil); TV / L1 worked examples; zero upstream -> zero gradients; plane-gradient sparsity.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import render as R
from .deform import PLANES

DT = torch.float64
LOG2E = 1.0 / math.log(2.0)


def _t(a):
    return torch.as_tensor(np.asarray(a, np.float64), dtype=DT)


# ------------------------------------------------------------------ parameters as leaf tensors
def params_of(scene, deformable=True):
    """Leaf tensors (requires_grad) of every trainable array of `scene` (reading B4)."""
    P = {"means": _t(scene.means), "log_scales": _t(scene.log_scales), "quats": _t(scene.quats),
         "opacity_logits": _t(scene.opacity_logits), "sh": _t(scene.sh)}
    if deformable:
        f = scene.field
        for l in range(len(f.planes)):
            for p in range(6):
                P[f"plane{l}_{p}"] = _t(f.planes[l][p])
        for k in ("w_d", "b_d", "w_x", "b_x", "w_r", "b_r", "w_s", "b_s", "w_c", "b_c", "w_a", "b_a"):
            if getattr(scene.mlp, k, None) is not None:        # phi_C / phi_alpha only when present
                P[k] = _t(getattr(scene.mlp, k))
    for v in P.values():
        v.requires_grad_(True)
    return P


# ------------------------------------------------------------------ F: the deformation field
def _bilinear(P, ua, ub):
    """Eq. 7 "interp ... 4 vertices" (as oracle.deform.bilinear); knot indices from detached u."""
    nb, na = P.shape[0], P.shape[1]
    ga = ua * (na - 1)
    gb = ub * (nb - 1)
    i0 = torch.clamp(torch.floor(ga.detach()), max=na - 2).long()
    j0 = torch.clamp(torch.floor(gb.detach()), max=nb - 2).long()
    fa = (ga - i0.to(DT))[:, None]
    fb = (gb - j0.to(DT))[:, None]
    return ((1 - fa) * (1 - fb) * P[j0, i0] + fa * (1 - fb) * P[j0, i0 + 1]
            + (1 - fa) * fb * P[j0 + 1, i0] + fa * fb * P[j0 + 1, i0 + 1])


def deform_torch(scene, t, P):
    """G' = G + F(G, t) on the leaf tensors P; returns dict means / log_scales / quats."""
    f = scene.field
    bmin, bmax = _t(f.bmin), _t(f.bmax)
    u = (P["means"] - bmin) / (bmax - bmin)
    u = torch.clamp(u, 0.0, 1.0)                  # D1: clamp (zero gradient outside the box)
    ut = torch.full((u.shape[0],), float(t), dtype=DT)
    axes = [u[:, 0], u[:, 1], u[:, 2], ut]
    feats = []
    for l in range(len(f.planes)):
        f_l = torch.ones((u.shape[0], f.feat), dtype=DT)
        for p, (a, b) in enumerate(PLANES):
            f_l = f_l * _bilinear(P[f"plane{l}_{p}"], axes[a], axes[b])
        feats.append(f_l)
    f_h = torch.cat(feats, dim=1)
    f_d = torch.relu(f_h @ P["w_d"].T + P["b_d"])
    G = {"means": P["means"] + f_d @ P["w_x"].T + P["b_x"],
         "quats": P["quats"] + f_d @ P["w_r"].T + P["b_r"],
         "log_scales": P["log_scales"] + f_d @ P["w_s"].T + P["b_s"]}
    if "w_c" in P:       # P:1232 colour decoder: C' = C + dC over all K x 3 coefficients (reading C1)
        G["sh"] = P["sh"] + (f_d @ P["w_c"].T + P["b_c"]).reshape(P["sh"].shape)
    if "w_a" in P:       # P:1232 opacity decoder: logit' = logit + dalpha
        G["opacity_logits"] = P["opacity_logits"] + (f_d @ P["w_a"].T + P["b_a"])[:, 0]
    return G


# ------------------------------------------------------------------ S: the splatting
def _sh_basis(d, degree):
    """Real SH with the CS phase (oracle/sh.py table), as torch ops."""
    from . import sh as S
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    cols = [torch.full_like(x, S.C0)]
    if degree >= 1:
        cols += [-S.C1 * y, S.C1 * z, -S.C1 * x]
    if degree >= 2:
        xx, yy, zz = x * x, y * y, z * z
        cols += [S.C2_K * x * y, -S.C2_K * y * z, S.C2_0 * (2 * zz - xx - yy), -S.C2_K * x * z, S.C2_2 * (xx - yy)]
    if degree >= 3:
        cols += [-S.C3_A * y * (3 * xx - yy), S.C3_B * x * y * z, -S.C3_C * y * (4 * zz - xx - yy),
                 S.C3_E * z * (2 * zz - 3 * xx - 3 * yy), -S.C3_C * x * (4 * zz - xx - yy),
                 0.5 * S.C3_B * z * (xx - yy), -S.C3_A * x * (xx - 3 * yy)]
    return torch.stack(cols, dim=1)


def preprocess_torch(G, opacity_logits, sh, sh_degree, cam):
    """Steps 1-12 of oracle.render.preprocess_ref as torch ops (same formulas, same order).  The
    integer results (kept, rect, depth key) come from the numpy oracle on the detached values."""
    pre_np = R.preprocess_ref(G["means"].detach().numpy(), G["log_scales"].detach().numpy(),
                              G["quats"].detach().numpy(), opacity_logits.detach().numpy(),
                              sh.detach().numpy(), sh_degree, cam)
    s = torch.exp(G["log_scales"])
    q = G["quats"] / torch.linalg.norm(G["quats"], dim=1, keepdim=True)
    o = torch.sigmoid(opacity_logits)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    Rq = torch.stack([
        torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1),
        torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1),
        torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)], 1)
    M = Rq * s[:, None, :]
    Sigma = M @ M.transpose(1, 2)                                          # Eq. 2
    Rc, tc = _t(cam.R), _t(cam.t)
    X = G["means"]
    p = torch.stack([((Rc[c, 0] * X[:, 0] + Rc[c, 1] * X[:, 1]) + Rc[c, 2] * X[:, 2]) + tc[c]
                     for c in range(3)], 1)
    pz = p[:, 2]
    tan_x, tan_y = cam.width / (2.0 * cam.fx), cam.height / (2.0 * cam.fy)
    xt = torch.clamp(p[:, 0] / pz, -R.FOV_CLAMP * tan_x, R.FOV_CLAMP * tan_x) * pz
    yt = torch.clamp(p[:, 1] / pz, -R.FOV_CLAMP * tan_y, R.FOV_CLAMP * tan_y) * pz
    zero = torch.zeros_like(pz)
    J = torch.stack([torch.stack([cam.fx / pz, zero, -cam.fx * xt / (pz * pz)], 1),
                     torch.stack([zero, cam.fy / pz, -cam.fy * yt / (pz * pz)], 1)], 1)
    Tm = J @ Rc
    S2 = Tm @ Sigma @ Tm.transpose(1, 2)                                   # Eq. 3
    a, b, c = S2[:, 0, 0] + R.DILATION, S2[:, 0, 1], S2[:, 1, 1] + R.DILATION
    det = a * c - b * b
    conic = torch.stack([c / det, -b / det, a / det], 1)
    mean2d = torch.stack([cam.fx * p[:, 0] / pz + cam.cx, cam.fy * p[:, 1] / pz + cam.cy], 1)
    campos = -Rc.T @ tc
    dv = X - campos
    d = dv / torch.linalg.norm(dv, dim=1, keepdim=True)
    Y = _sh_basis(d, sh_degree)
    raw = torch.einsum("nk,nkc->nc", Y, sh[:, :Y.shape[1], :]) + 0.5
    rgb = torch.where(raw.detach() > 0, raw, torch.zeros_like(raw))       # clamp at 0 (R10)
    return pre_np, {"mean2d": mean2d, "conic": conic, "opacity": o, "rgb": rgb}


def composite_torch(pre_t, order, px, py, bg):
    """Eq. 4 front to back (oracle.render.composite) with every decision from detached values."""
    P = px.shape[0]
    T = torch.ones(P, dtype=DT)
    C = torch.zeros((P, 3), dtype=DT)
    done = torch.zeros(P, dtype=torch.bool)
    m, cn, o, rgb = pre_t["mean2d"], pre_t["conic"], pre_t["opacity"], pre_t["rgb"]
    for g in order:
        dx = m[g, 0] - px
        dy = m[g, 1] - py
        A, B, Cc = cn[g, 0], cn[g, 1], cn[g, 2]
        power = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy
        raw_a = o[g] * torch.exp(power)
        alpha = torch.where(raw_a.detach() < R.ALPHA_MAX, raw_a, torch.full_like(raw_a, R.ALPHA_MAX))
        al = alpha.detach()
        use = ~done & ~(power.detach() > 0) & ~(al < R.ALPHA_MIN)
        test_T = T * (1.0 - alpha)
        stop = use & (test_T.detach() < R.T_MIN)
        done = done | stop
        add = use & ~stop
        C = C + torch.where(add[:, None], rgb[g][None, :] * (alpha * T)[:, None], torch.zeros_like(C))
        T = torch.where(add, test_T, T)
        if bool(done.all()):
            break
    return C + T[:, None] * _t(bg)[None, :]


def render_torch(G, opacity_logits, sh, sh_degree, cam):
    """I^ = S(M, G') (oracle.render.render_ref, tiled) as torch ops; returns image [3, H, W]."""
    W, H = cam.width, cam.height
    gx, gy = R.tile_grid(W, H)
    pre_np, pre_t = preprocess_torch(G, opacity_logits, sh, sh_degree, cam)
    _, gids, ranges = R.bin_ref(pre_np, cam)
    img = torch.zeros((3, H * W), dtype=DT)
    for tile in range(gx * gy):
        pxn, pyn = R._tile_pixels(tile, gx, W, H)
        s0, e0 = ranges[tile]
        col = composite_torch(pre_t, gids[s0:e0].tolist(), _t(pxn), _t(pyn), cam.bg)
        img = img.index_put((torch.arange(3)[:, None], torch.as_tensor(pyn * W + pxn)[None, :]), col.T)
    return img.reshape(3, H, W)


# ------------------------------------------------------------------ L = |I^ - I| + w L_tv
def l1_loss(image, target):
    """B2: mean over pixels and channels of |I^ - I|."""
    return torch.mean(torch.abs(image - _t(target)))


def tv_loss(planes):
    """B1: pooled mean of the squared differences of horizontally and vertically adjacent entries of
    every plane (list of [n_b][n_a][h] tensors), over all planes, channels and both directions."""
    terms = []
    for Pl in planes:
        terms.append(((Pl[:, 1:, :] - Pl[:, :-1, :]) ** 2).reshape(-1))    # along a (horizontal)
        terms.append(((Pl[1:, :, :] - Pl[:-1, :, :]) ** 2).reshape(-1))    # along b (vertical)
    return torch.mean(torch.cat(terms))


def frame_loss(scene, frame, target, tv_weight, P):
    """L of one (t, camera) frame: deform (leaf tensors P), render, L1 + w_tv L_tv (B3)."""
    G = deform_torch(scene, float(scene.times[frame]), P)
    img = render_torch(G, G.get("opacity_logits", P["opacity_logits"]), G.get("sh", P["sh"]), scene.sh_degree,
                       scene.cameras[frame])
    planes = [P[k] for k in sorted(P) if k.startswith("plane")]
    return l1_loss(img, target) + tv_weight * tv_loss(planes), img


def grads_ref(scene, frame, target, tv_weight=0.0):
    """dL/d(every parameter) of frame_loss (numpy float64 dict) and L."""
    P = params_of(scene)
    L, img = frame_loss(scene, frame, target, tv_weight, P)
    L.backward()
    return {k: v.grad.numpy().copy() for k, v in P.items()}, float(L.detach()), img.detach().numpy()


def render_grads_ref(deformed, opacity_logits, sh, sh_degree, cam, dL_dimage):
    """The splatting alone: gradients of sum(dL_dimage * I^) w.r.t. the deformed attributes (means,
    log_scales, raw quats) and the opacity logits and SH it renders."""
    G = {k: _t(deformed[k]).requires_grad_(True) for k in ("means", "log_scales", "quats")}
    ol = _t(opacity_logits).requires_grad_(True)
    sht = _t(sh).requires_grad_(True)
    img = render_torch(G, ol, sht, sh_degree, cam)
    (img * _t(dL_dimage)).sum().backward()
    out = {k: v.grad.numpy().copy() for k, v in G.items()}
    out["opacity_logits"] = ol.grad.numpy().copy()
    out["sh"] = sht.grad.numpy().copy()
    return out, img.detach().numpy()


def deform_grads_ref(scene, t, dL_ddeformed):
    """The deformation field alone: gradients of sum_k <dL_ddeformed[k], G'[k]> (k = means, log_scales,
    quats, and with the P:1232 decoders sh / opacity_logits) w.r.t. the canonical parameters, the planes
    and the MLP."""
    P = params_of(scene)
    G = deform_torch(scene, t, P)
    sum(((G[k] * _t(dL_ddeformed[k])).sum() for k in G)).backward()
    return {k: (v.grad.numpy().copy() if v.grad is not None else np.zeros(tuple(v.shape)))
            for k, v in P.items() if k in G or k not in ("opacity_logits", "sh")}
