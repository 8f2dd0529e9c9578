"""Pins for the deformation oracle (oracle/deform.py) — CPU only.

Each test pins the oracle to something other than itself:
closed forms of bilinear interpolation, invariants of the Hadamard/concat
fusion (Eq. 7), a scalar loop for the MLP, and the additive
update rule.
"""
import json
import math
import os
from dataclasses import replace

import numpy as np
import pytest

import oracle
from oracle.deform import bilinear, decoder, grid_coords, hexplane_features
from paper_2310_08528_b200.inputs import make_scene, with_heads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _bilinear_plane(na, nb, h, coef):
    """Plane holding v(i,j) = a + b i + c j + d i j per channel (knot indices)."""
    j, i = np.meshgrid(np.arange(nb), np.arange(na), indexing="ij")
    a, b, c, d = coef
    return (a[None, None, :] + b[None, None, :] * i[..., None] + c[None, None, :] * j[..., None]
            + d[None, None, :] * (i * j)[..., None])


def test_bilinear_exact_on_bilinear_functions():
    """Eq. 7 'bilinear interpolation ... 4 vertices': exact on a + b i + c j + d i j."""
    rng = np.random.default_rng(0)
    na, nb, h = 33, 17, 5
    coef = [rng.normal(size=h) for _ in range(4)]
    P = _bilinear_plane(na, nb, h, coef)
    ua, ub = rng.uniform(0, 1, 10000), rng.uniform(0, 1, 10000)
    ua[:3] = [0.0, 1.0, 1.0]
    ub[:3] = [1.0, 0.0, 1.0]
    got = bilinear(P, ua, ub)
    ga, gb = ua * (na - 1), ub * (nb - 1)
    want = (coef[0][None] + coef[1][None] * ga[:, None] + coef[2][None] * gb[:, None]
            + coef[3][None] * (ga * gb)[:, None])
    assert np.max(np.abs(got - want)) < 1e-11


def test_bilinear_knots_and_cell_centres():
    """SPEC S:210 (a knot reproduces its value) and S:211 (cell centre = mean of 4)."""
    rng = np.random.default_rng(1)
    na, nb, h = 9, 6, 4
    P = rng.normal(size=(nb, na, h))
    for j in range(nb):
        for i in range(na):
            v = bilinear(P, np.array([i / (na - 1)]), np.array([j / (nb - 1)]))[0]
            assert np.allclose(v, P[j, i], atol=1e-14, rtol=0)
    for j in range(nb - 1):
        for i in range(na - 1):
            v = bilinear(P, np.array([(i + 0.5) / (na - 1)]), np.array([(j + 0.5) / (nb - 1)]))[0]
            want = 0.25 * (P[j, i] + P[j, i + 1] + P[j + 1, i] + P[j + 1, i + 1])
            assert np.allclose(v, want, atol=1e-14, rtol=0)


def test_bilinear_matches_scalar_loop():
    """random queries vs a scalar double-loop bilinear (brute force)."""
    rng = np.random.default_rng(2)
    na, nb, h = 12, 7, 3
    P = rng.normal(size=(nb, na, h))
    ua, ub = rng.uniform(0, 1, 200), rng.uniform(0, 1, 200)
    got = bilinear(P, ua, ub)
    for q in range(200):
        x, y = ua[q] * (na - 1), ub[q] * (nb - 1)
        acc = np.zeros(h)
        for jj in range(nb):
            for ii in range(na):
                w = max(0.0, 1 - abs(x - ii)) * max(0.0, 1 - abs(y - jj))   # tent weights
                acc += w * P[jj, ii]
        assert np.allclose(got[q], acc, atol=1e-13, rtol=0)


def _field_from(scene, planes):
    return replace(scene.field, planes=planes)


def test_hexplane_affine_planes_exact(tiny_scene):
    """north_star pin: planes holding affine functions, the other 5 planes = 1, are exact."""
    s = tiny_scene
    f = s.field
    rng = np.random.default_rng(3)
    for p_idx, (a, b) in enumerate(oracle.deform.PLANES):
        planes = [[np.ones_like(P, dtype=np.float64) for P in f.planes[0]]]
        na = f.planes[0][p_idx].shape[1]
        nb = f.planes[0][p_idx].shape[0]
        coef = [rng.normal(size=f.feat) for _ in range(3)] + [np.zeros(f.feat)]
        planes[0][p_idx] = _bilinear_plane(na, nb, f.feat, coef)
        fld = _field_from(s, planes)
        t = 0.37
        fh = hexplane_features(s.means[:500], t, fld)
        u = grid_coords(s.means[:500], f.bmin, f.bmax, t)
        ga, gb = u[:, a] * (na - 1), u[:, b] * (nb - 1)
        want = coef[0][None] + coef[1][None] * ga[:, None] + coef[2][None] * gb[:, None]
        assert np.max(np.abs(fh - want)) < 1e-11, (a, b)


def test_hexplane_product_and_concat_invariants():
    """SPEC S:219 (all-ones planes -> f_h = 1), S:220 (a zero plane zeroes its scale),
    S:244 (L=2 restricted to l=1 equals the L=1 field)."""
    s = make_scene("dnerf", n=300, width=64, height=64, n_frames=1)
    f = s.field
    ones = [[np.ones_like(P) for P in ps] for ps in f.planes]
    fh = hexplane_features(s.means, 0.3, _field_from(s, ones))
    assert fh.shape == (300, f.feat * 2) and np.max(np.abs(fh - 1.0)) < 1e-14  # weights sum to 1 up to rounding
    for p_idx in range(6):
        planes = [list(ps) for ps in f.planes]
        planes[1][p_idx] = np.zeros_like(planes[1][p_idx])
        fh = hexplane_features(s.means, 0.6, _field_from(s, planes))
        assert np.all(fh[:, f.feat:] == 0.0)
        assert np.all(fh[:, :f.feat] != 0.0)
    full = hexplane_features(s.means, 0.45, f)
    single = hexplane_features(s.means, 0.45, replace(f, planes=[f.planes[0]], res=[f.res[0]]))
    assert np.array_equal(full[:, :f.feat], single)


def test_decoder_matches_scalar_loop(tiny_scene):
    """phi_d = ReLU(W_d f_h + b_d); heads linear (readings D5, D6) — scalar-loop brute force."""
    s = with_heads(tiny_scene, 0.7, seed=5, bias_sigma=0.3)
    fh = hexplane_features(s.means[:20], 0.5, s.field)
    dX, dr, ds = decoder(fh, s.mlp)
    m = s.mlp
    for n in range(20):
        hid = []
        for o in range(m.width):
            acc = float(m.b_d[o])
            for k in range(m.in_dim):
                acc += float(m.w_d[o, k]) * fh[n, k]
            hid.append(max(0.0, acc))
        for W, b, out in ((m.w_x, m.b_x, dX), (m.w_r, m.b_r, dr), (m.w_s, m.b_s, ds)):
            for o in range(W.shape[0]):
                acc = float(b[o]) + sum(float(W[o, k]) * hid[k] for k in range(m.width))
                assert abs(acc - out[n, o]) < 1e-12


def test_zero_heads_identity(tiny_scene):
    """SPEC S:285 / north_star: zero heads -> G' = G exactly (compared by value)."""
    s = with_heads(tiny_scene, 0.0)
    d = oracle.deform_ref(s, 0.37)
    assert np.array_equal(d["means"], s.means.astype(np.float64))
    assert np.array_equal(d["quats"], s.quats.astype(np.float64))
    assert np.array_equal(d["log_scales"], s.log_scales.astype(np.float64))


def test_constant_head_x_shifts(tiny_scene):
    """head_x constant (1,0,0), others zero -> every mean shifts by +x."""
    s = with_heads(tiny_scene, 0.0)
    s = replace(s, mlp=replace(s.mlp, b_x=np.array([1, 0, 0], np.float32)))
    d = oracle.deform_ref(s, 0.8)
    assert np.array_equal(d["means"] - s.means.astype(np.float64),
                          np.tile([1.0, 0.0, 0.0], (s.n, 1)))
    assert np.array_equal(d["quats"], s.quats.astype(np.float64))


def test_permutation_equivariance(tiny_scene):
    """permuting Gaussians before deform equals permuting after."""
    s = with_heads(tiny_scene, 0.5, seed=9)
    perm = np.random.default_rng(4).permutation(s.n)
    d = oracle.deform_ref(s, 0.2)
    dp = oracle.deform_ref(s, 0.2, means=s.means[perm], quats=s.quats[perm],
                           log_scales=s.log_scales[perm])
    for k in d:
        assert np.array_equal(d[k][perm], dp[k])


def test_range_equals_slice(tiny_scene):
    """Sharded form (§8(e2)): deform of [begin,end) equals the slice of the full deform."""
    s = with_heads(tiny_scene, 0.5, seed=9)
    d = oracle.deform_ref(s, 0.6)
    r = oracle.deform_ref(s, 0.6, begin=700, end=1333)
    for k in d:
        assert np.array_equal(d[k][700:1333], r[k])


def test_grid_clamp_outside_aabb(tiny_scene):
    """Reading D1: out-of-box means clamp to the AABB faces."""
    s = tiny_scene
    X = np.array([[5.0, -7.0, 0.0], [1.0, 1.0, 1.0]])
    u = grid_coords(X, s.field.bmin, s.field.bmax, 0.25)
    assert np.array_equal(u[0], [1.0, 0.0, 0.5, 0.25])
    assert np.array_equal(u[1], [1.0, 1.0, 1.0, 0.25])


# ---------------------------------------------------------------- colour / opacity decoders
def test_colour_opacity_heads_match_scalar_loop():
    """dC = phi_C(f_d), dalpha = phi_alpha(f_d), one Linear each (reading C1) — scalar-loop brute force,
    and the SH layout of dC (k-major, channel-minor)."""
    from paper_2310_08528_b200.inputs import with_colour_heads
    s = with_colour_heads(make_scene("dnerf", n=40), 0.3, 0.5, seed=9)
    t = 0.42
    fh = hexplane_features(s.means[:6], t, s.field)
    d = oracle.deform_ref(s, t, begin=0, end=6)
    m = s.mlp
    K = (s.sh_degree + 1) ** 2
    for n in range(6):
        hid = []
        for o in range(m.width):
            acc = float(m.b_d[o]) + sum(float(m.w_d[o, k]) * fh[n, k] for k in range(m.in_dim))
            hid.append(max(0.0, acc))
        for kk in range(K):
            for ch in range(3):
                o = 3 * kk + ch
                acc = float(m.b_c[o]) + sum(float(m.w_c[o, j]) * hid[j] for j in range(m.width))
                assert abs(float(s.sh[n, kk, ch]) + acc - d["sh"][n, kk, ch]) < 1e-12
        acc = float(m.b_a[0]) + sum(float(m.w_a[0, j]) * hid[j] for j in range(m.width))
        assert abs(float(s.opacity_logits[n]) + acc - d["opacity_logits"][n]) < 1e-12


def test_zero_colour_heads_identity_and_constant_shift():
    """Zero phi_C, phi_alpha leave SH and opacity unchanged (exact); a bias-only phi_alpha shifts every
    logit by that bias; models without the heads return no SH / opacity (P:802 G' aliases them)."""
    from paper_2310_08528_b200.inputs import with_colour_heads
    base = make_scene("tiny", n=300)
    assert "sh" not in oracle.deform_ref(base, 0.3) and "opacity_logits" not in oracle.deform_ref(base, 0.3)
    s = with_colour_heads(base, 0.0, 0.0)
    d = oracle.deform_ref(s, 0.3)
    assert np.array_equal(d["sh"], s.sh.astype(np.float64))
    assert np.array_equal(d["opacity_logits"], s.opacity_logits.astype(np.float64))
    s2 = replace(s, mlp=replace(s.mlp, b_a=np.array([0.25], np.float32)))
    d2 = oracle.deform_ref(s2, 0.3)
    assert np.array_equal(d2["opacity_logits"] - s.opacity_logits.astype(np.float64), np.full(s.n, 0.25))
