"""Pins for the splatting oracle (oracle/render.py) — CPU only.

Closed forms and worked examples for Eqs. 1-4, the [3dgs]
conventions read in R4-R9, brute-force compositing (§8(c.2) step 15) and the
north_star checks: zero heads -> static render, single isotropic splat,
opaque front occluder, tiled == brute force.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import render as R
from paper_2310_08528_b200.inputs import Camera, look_at, make_scene, with_heads, with_max_opacity

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
G = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))


def _cam(W=64, H=64, eye=(0, 0, 4), target=(0, 0, 0), bg=(0, 0, 0)):
    return look_at(eye, target, W, H, bg)


def _gaussians(means, log_scales, quats, logits, dc):
    n = len(means)
    sh = np.zeros((n, 1, 3), np.float32)
    sh[:, 0, :] = np.asarray(dc, np.float32)
    return dict(means=np.asarray(means, np.float32), log_scales=np.asarray(log_scales, np.float32),
                quats=np.asarray(quats, np.float32)), np.asarray(logits, np.float32), sh


# ------------------------------------------------------------------ Eq. 2
@pytest.mark.parametrize("ex", G["covariance"])
def test_covariance_worked_examples(ex):
    S = R.covariance3d(np.array([ex["scale"]], float), np.array([ex["quat_wxyz"]], float))[0]
    assert np.allclose(S, ex["sigma"], atol=1e-12)


def test_covariance_symmetric_psd_rotation_consistent():
    rng = np.random.default_rng(0)
    s = np.exp(rng.normal(size=(1000, 3)))
    q = rng.normal(size=(1000, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    S = R.covariance3d(s, q)
    assert np.max(np.abs(S - np.transpose(S, (0, 2, 1)))) < 1e-12 * np.max(np.abs(S))
    ev = np.linalg.eigvalsh(S)
    assert np.all(ev >= -1e-12 * ev.max(axis=1, keepdims=True))
    # eigenvalues are s^2 (the rotation does not change them)
    assert np.allclose(np.sort(ev, axis=1), np.sort(s * s, axis=1), rtol=1e-9)
    # quaternion rotation matrices are orthonormal with det +1
    Rm = R.quat_to_rotmat(q)
    assert np.allclose(Rm @ np.transpose(Rm, (0, 2, 1)), np.eye(3), atol=1e-12)
    assert np.allclose(np.linalg.det(Rm), 1.0, atol=1e-12)


@pytest.mark.parametrize("ex", G["activation"])
def test_activation_examples(ex):
    if "log_scale" in ex:
        s, _, _ = R.activate([[ex["log_scale"]] * 3], [[1, 0, 0, 0]], [0.0])
        assert s[0, 0] == ex["scale"]
    elif "opacity_logit" in ex:
        _, _, o = R.activate([[0, 0, 0]], [[1, 0, 0, 0]], [ex["opacity_logit"]])
        assert o[0] == ex["opacity"]
    else:
        _, q, _ = R.activate([[0, 0, 0]], [ex["quat"]], [0.0])
        assert np.array_equal(q[0], ex["unit"])


# ------------------------------------------------------------------ Eq. 3
def test_on_axis_isotropic_projection():
    """on-axis, depth z, Sigma = sigma^2 I -> Sigma2 = (f sigma/z)^2 I + 0.3 I."""
    cam = _cam()
    for sigma, z in ((0.05, 4.0), (0.2, 4.0)):
        g, lg, sh = _gaussians([[0, 0, 4.0 - z]], [[math.log(sigma)] * 3], [[1, 0, 0, 0]], [0.0], [0, 0, 0])
        pre = R.preprocess_ref(g["means"], g["log_scales"], g["quats"], lg, sh, 0, cam)
        s32 = float(np.exp(np.float64(np.float32(math.log(sigma)))))
        want = (cam.fx * s32 / z) ** 2 + 0.3
        a, b, c = pre["cov2d"][0]
        assert abs(a - want) < 1e-10 * want and abs(c - want) < 1e-10 * want and abs(b) < 1e-12
        # principal point
        assert np.allclose(pre["mean2d"][0], [cam.cx, cam.cy], atol=1e-12)


def test_near_plane_cull():
    """SPEC S:128 / R6: p.z <= 0.2f is culled; just in front of it is kept."""
    cam = _cam()
    zs = [4.0 - 0.1, 4.0 - 0.2, 4.0 - 0.25, 4.0 + 1.0]     # cam depth 0.1, 0.2, 0.25, -1
    g, lg, sh = _gaussians([[0, 0, 4.0 - d] for d in (0.1, 0.2, 0.25)] + [[0, 0, 5.0]],
                           [[-3.0] * 3] * 4, [[1, 0, 0, 0]] * 4, [0.0] * 4, [[0, 0, 0]] * 4)
    pre = R.preprocess_ref(g["means"], g["log_scales"], g["quats"], lg, sh, 0, cam)
    assert pre["kept"].tolist() == [False, pre["p"][1, 2] > R.NEAR, True, False]


def test_jacobian_matches_finite_differences():
    """J of the perspective map pi(p) = (fx x/z + cx, fy y/z + cy), inside the clamp."""
    cam = _cam(W=80, H=60)
    rng = np.random.default_rng(1)
    p = np.stack([rng.uniform(-0.5, 0.5, 50), rng.uniform(-0.4, 0.4, 50), rng.uniform(1, 5, 50)], 1)
    J = R.jacobian(p, cam)

    def pi(v):
        return np.stack([cam.fx * v[:, 0] / v[:, 2] + cam.cx, cam.fy * v[:, 1] / v[:, 2] + cam.cy], 1)

    h = 1e-6
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        num = (pi(p + e) - pi(p - e)) / (2 * h)
        assert np.max(np.abs(num - J[:, :, k])) < 1e-5 * np.max(np.abs(J))


def test_jacobian_clamp():
    """R4: outside 1.3 tan(fov/2) the x/z used by J is clamped."""
    cam = _cam(W=64, H=64)
    lim = 1.3 * cam.width / (2 * cam.fx)
    p = np.array([[10.0, 0.0, 1.0]])
    J = R.jacobian(p, cam)
    assert abs(J[0, 0, 2] - (-cam.fx * lim)) < 1e-12


# ------------------------------------------------------------------ radius / rect
def test_radius_rect_hand_calculation():
    ex = G["radius_rect"][0]
    a, b, c = ex["cov2d_dilated"]
    lam, three, r = R.radius_from_cov2d(np.array([a]), np.array([b]), np.array([c]))
    assert abs(lam[0] - ex["lambda1"]) < 1e-12 and r[0] == ex["radius"]
    rect = R.tile_rect(np.array([ex["mean2d"][0]]), np.array([ex["mean2d"][1]]), r, *ex["grid"])
    assert [int(v[0]) for v in rect] == ex["rect"]


def test_rect_clamps_at_border():
    x0, y0, x1, y1 = R.tile_rect(np.array([-30.0, 70.0]), np.array([2.0, 63.0]),
                                 np.array([5.0, 40.0]), 4, 4)
    assert (x0.tolist(), x1.tolist()) == ([0, 1], [0, 4])       # left one fully outside
    assert (y0.tolist(), y1.tolist()) == ([0, 1], [1, 4])


# ------------------------------------------------------------------ Eq. 1 / Eq. 4
def _pre_fragments(frags):
    n = len(frags)
    pre = {"mean2d": np.zeros((n, 2)), "conic": np.zeros((n, 3)), "opacity": np.zeros(n),
           "rgb": np.zeros((n, 3))}
    for i, f in enumerate(frags):
        pre["mean2d"][i] = f.get("mean", (0.0, 0.0))
        cov = np.asarray(f.get("cov2d", [[1.0, 0.0], [0.0, 1.0]]), float)
        inv = np.linalg.inv(cov)
        pre["conic"][i] = [inv[0, 0], inv[0, 1], inv[1, 1]]
        pre["opacity"][i] = f["alpha"]
        pre["rgb"][i] = f["rgb"]
    return pre


@pytest.mark.parametrize("ex", G["density"])
def test_density_worked_examples(ex):
    """Eq. 1 through the blend: pixel = o G(x) with o = 0.5, rgb = 1, black bg."""
    pre = _pre_fragments([{"mean": (ex["offset"][0], ex["offset"][1]), "cov2d": ex["cov2d"],
                           "alpha": 0.5, "rgb": (1, 1, 1)}])
    rgb, T, _, _ = R.composite(pre, [0], np.array([0.0]), np.array([0.0]), [0, 0, 0])
    assert abs(rgb[0, 0] / 0.5 - ex["value"]) < 1e-15


@pytest.mark.parametrize("ex", G["compositing"])
def test_compositing_worked_examples(ex):
    pre = _pre_fragments(ex["fragments"])
    rgb, T, nc, _ = R.composite(pre, list(range(len(ex["fragments"]))), np.array([0.0]),
                                np.array([0.0]), ex["bg"])
    assert np.allclose(rgb[0], ex["pixel"], atol=1e-15)
    assert nc[0] == len(ex["fragments"])


def test_composite_background_and_transmittance():
    """One fragment: c a + (1 - a) bg; T non-increasing."""
    pre = _pre_fragments([{"alpha": 0.3, "rgb": (0.2, 0.4, 0.6)}, {"alpha": 0.6, "rgb": (1, 0, 0)},
                          {"alpha": 0.9, "rgb": (0, 0, 1)}])
    bg = np.array([0.1, 0.7, 0.3])
    rgb1, T1, _, _ = R.composite(pre, [0], np.array([0.0]), np.array([0.0]), bg)
    assert np.allclose(rgb1[0], 0.3 * np.array([0.2, 0.4, 0.6]) + 0.7 * bg, atol=1e-15)
    Ts = [R.composite(pre, list(range(k)), np.array([0.0]), np.array([0.0]), bg)[1][0] for k in range(4)]
    assert all(Ts[i + 1] <= Ts[i] for i in range(3)) and Ts[0] == 1.0


def test_fp32_threshold_constants():
    g = G["fp32_thresholds"]
    assert R.T_MIN == g["t_min_f32"] and R.ALPHA_MIN == g["alpha_min_f32"]
    assert 1.0 - R.ALPHA_MAX == g["one_minus_0p99f"]
    t1 = np.float32(1.0) - np.float32(R.ALPHA_MAX)             # fp32 arithmetic (GPU side)
    assert float(t1 * t1) == g["two_clamped_layers_T"] < R.T_MIN
    assert (1.0 - R.ALPHA_MAX) ** 2 < R.T_MIN                  # fp64 (oracle side) decides the same


def test_alpha_skip_and_stop_rules():
    """R9: alpha < 1/255 skipped; the Gaussian whose T' < 1e-4f stops and is not added."""
    pre = _pre_fragments([{"alpha": R.ALPHA_MIN * 0.999, "rgb": (1, 1, 1)},
                          {"alpha": 0.999, "rgb": (1, 0, 0)}, {"alpha": 0.999, "rgb": (0, 1, 0)},
                          {"alpha": 0.5, "rgb": (0, 0, 1)}])
    rgb, T, nc, _ = R.composite(pre, [0, 1, 2, 3], np.array([0.0]), np.array([0.0]), [0, 0, 0])
    assert nc[0] == 1                       # skip, add (clamped to 0.99f), stop
    assert rgb[0, 0] == R.ALPHA_MAX and rgb[0, 1] == 0.0 and T[0] == 1.0 - R.ALPHA_MAX


# ------------------------------------------------------------------ north_star pins
def test_single_isotropic_splat_closed_form():
    """On-axis isotropic Gaussian (m = principal point, ragged 72x56 image):
    pixel = rgb a(p) + (1 - a(p)) bg, a = min(0.99f, o exp(-|p-m|^2 / (2 s^2))), s^2 = (f sigma/z)^2 + 0.3,
    if a >= 1/255 and tile(p) in rect, else bg."""
    W, H = 72, 56
    cam = _cam(W, H, bg=(0.2, 0.3, 0.4))
    sigma = 0.06
    g, lg, sh = _gaussians([[0.0, 0.0, 0.0]], [[math.log(sigma)] * 3], [[0.3, 0.1, -0.2, 0.9]],
                           [1.2], [[0.7, -0.4, 0.1]])
    out = R.render_ref(g, lg, sh, 0, cam)
    img = out["image"]
    pre = out["pre"]
    s32 = float(np.exp(np.float64(g["log_scales"][0, 0])))
    p = pre["p"][0]
    s2 = (cam.fx * s32 / p[2]) ** 2 + 0.3
    m = pre["mean2d"][0]
    o = 1 / (1 + math.exp(-float(lg[0])))
    rgb = np.maximum(0, np.array([0.7, -0.4, 0.1], np.float32).astype(float) * 0.28209479177387814 + 0.5)
    x0, y0, x1, y1 = pre["rect"][0]
    bg = np.array([0.2, 0.3, 0.4], np.float32).astype(float)
    for py in range(H):
        for px in range(W):
            a = min(R.ALPHA_MAX, o * math.exp(-0.5 * ((px - m[0]) ** 2 + (py - m[1]) ** 2) / s2))
            inrect = x0 <= px // 16 < x1 and y0 <= py // 16 < y1
            want = rgb * a + (1 - a) * bg if (a >= R.ALPHA_MIN and inrect) else bg
            assert np.allclose(img[:, py, px], want, atol=1e-12, rtol=0), (px, py)
    assert abs(m[0] - 35.5) < 1e-12 and abs(m[1] - 27.5) < 1e-12


def test_opaque_front_occluder():
    """A front Gaussian clamped at 0.99f, a second clamped one stops: pixel = rgb1 0.99f + (1-0.99f) bg,
    independent of everything behind (occluder pin)."""
    cam = _cam(64, 64, bg=(0.5, 0.25, 1.0))
    means = [[0, 0, 1.0], [0, 0, 0.5], [0, 0, 0.0], [0.01, 0.0, -0.5]]
    g, lg, sh = _gaussians(means, [[math.log(0.3)] * 3] * 4, [[1, 0, 0, 0]] * 4, [8.0] * 4,
                           [[1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0], [1.0, 1.0, 1.0]])
    out = R.render_ref(g, lg, sh, 0, cam)
    rgb1 = np.maximum(0, np.array([1.0, 0, 0]) * 0.28209479177387814 + 0.5)
    bg = np.array([0.5, 0.25, 1.0])
    want = rgb1 * R.ALPHA_MAX + (1 - R.ALPHA_MAX) * bg
    for (py, px) in ((31, 31), (32, 32), (31, 32)):
        assert np.array_equal(out["image"][:, py, px], want)
        assert out["n_contrib"][py, px] == 1
    # reorder the array: same image (depth order decides)
    perm = [3, 1, 0, 2]
    g2 = {k: v[perm] for k, v in g.items()}
    out2 = R.render_ref(g2, lg[perm], sh[perm], 0, cam)
    assert np.array_equal(out["image"], out2["image"])


def test_empty_scene_is_background():
    """empty set -> background everywhere."""
    cam = _cam(40, 24, bg=(0.1, 0.2, 0.3))
    g, lg, sh = _gaussians(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0), np.zeros((0, 3)))
    out = R.render_ref(g, lg, sh, 0, cam)
    assert np.allclose(out["image"], np.array([0.1, 0.2, 0.3], np.float32).astype(float)[:, None, None])
    assert np.all(out["final_T"] == 1.0) and np.all(out["n_contrib"] == 0)


def test_static_render_when_heads_zero(tiny_scene):
    """north_star: zero heads -> render(deform(G, t)) == render(G) (a static 3D-GS render)."""
    s = with_heads(tiny_scene, 0.0)
    d = oracle.deform_ref(s, 0.37)
    a = R.render_ref(d, s.opacity_logits, s.sh, s.sh_degree, s.cameras[0])
    b = R.render_ref(dict(means=s.means, log_scales=s.log_scales, quats=s.quats), s.opacity_logits,
                     s.sh, s.sh_degree, s.cameras[0])
    assert np.array_equal(a["image"], b["image"])


@pytest.mark.parametrize("W,H", [(64, 64), (70, 50)])
def test_tiled_equals_bruteforce_with_rect_predicate(W, H):
    """§8(c.2) step 15 at the tiny config's real opacities (incl. a ragged tile tail)."""
    s = make_scene("tiny", width=W, height=H)
    d = oracle.deform_ref(s, s.times[0])
    t = R.render_ref(d, s.opacity_logits, s.sh, s.sh_degree, s.cameras[0])
    b = R.render_ref_bruteforce(d, s.opacity_logits, s.sh, s.sh_degree, s.cameras[0], rect_predicate=True)
    assert np.array_equal(t["image"], b["image"])
    assert np.array_equal(t["n_contrib"], b["n_contrib"])


def test_tiled_equals_bruteforce_low_opacity():
    """north_star literal check: with opacities <= 0.017 truncation cannot bind, so tiled ==
    brute force over ALL Gaussians with no rect predicate."""
    s = with_max_opacity(make_scene("tiny", n=600), 0.017)
    d = oracle.deform_ref(s, s.times[0])
    t = R.render_ref(d, s.opacity_logits, s.sh, s.sh_degree, s.cameras[0])
    b = R.render_ref_bruteforce(d, s.opacity_logits, s.sh, s.sh_degree, s.cameras[0], rect_predicate=False)
    assert np.array_equal(t["image"], b["image"])


def test_binning_lists_are_valid(tiny_scene):
    """Per-tile lists hold exactly the Gaussians whose rect covers the tile, sorted by (key, index)."""
    s = tiny_scene
    d = oracle.deform_ref(s, s.times[0])
    cam = s.cameras[0]
    pre = R.preprocess_ref(d["means"], d["log_scales"], d["quats"], s.opacity_logits, s.sh, 0, cam)
    tiles, gids, ranges = R.bin_ref(pre, cam)
    gx, gy = R.tile_grid(cam.width, cam.height)
    assert len(tiles) == int(pre["tiles_touched"].sum())
    for tile in range(gx * gy):
        st, en = ranges[tile]
        lst = gids[st:en]
        ty, tx = divmod(tile, gx)
        r = pre["rect"]
        want = np.nonzero(pre["kept"] & (r[:, 0] <= tx) & (tx < r[:, 2]) & (r[:, 1] <= ty) & (ty < r[:, 3]))[0]
        assert sorted(lst.tolist()) == want.tolist()
        keys = pre["depth_key"][lst].astype(np.int64)
        pairs = list(zip(keys.tolist(), lst.tolist()))
        assert pairs == sorted(pairs)


def test_tile_list_ref_equals_bin_ref_slices(tiny_scene):
    """The single-tile list builder (used for sampled tiles at large configs) gives exactly the
    slice of the full instance sort, and the subset render equals the full render on those tiles."""
    s = make_scene("tiny", width=70, height=50)
    d = oracle.deform_ref(s, s.times[0])
    cam = s.cameras[0]
    pre = R.preprocess_ref(d["means"], d["log_scales"], d["quats"], s.opacity_logits, s.sh, 0, cam)
    tiles, gids, ranges = R.bin_ref(pre, cam)
    gx, gy = R.tile_grid(cam.width, cam.height)
    for tile in range(gx * gy):
        st, en = ranges[tile]
        assert np.array_equal(R.tile_list_ref(pre, cam, tile), gids[st:en])
    sub = [0, 5, gx * gy - 1]
    a = R.render_ref(d, s.opacity_logits, s.sh, 0, cam, tiles_subset=sub, pre=pre)
    b = R.render_ref(d, s.opacity_logits, s.sh, 0, cam, tiles_subset=sub, pre=pre, full_bins=False)
    m = np.isfinite(a["image"][0])
    assert m.sum() > 0 and np.array_equal(a["image"][:, m], b["image"][:, m])
    assert np.array_equal(a["flagged"], b["flagged"])
