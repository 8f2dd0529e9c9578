"""Pins for the oracle's geometry that the round-1 pins left handedness/sign-blind — CPU only.

Each pin computes the expected value by an independent route (textbook definitions, not the
oracle's formulas) and each has a mutation test: the named plausible mistake, injected by
monkeypatching the oracle, must make the pin fail.

  * Eq. 2 quaternion handedness: R(q) v == vec(q (0,v) q*) (Hamilton product), and
    the textbook +90 deg turn about z maps x -> y.                      mutation: R <-> R^T
  * Eq. 3 anisotropic Sigma, off-axis, rotated camera: (a, b, c) == J_full Sigma J_full^T
    + 0.3 I where J_full is the central-difference Jacobian of the world->pixel map
    K [R|t] X (homogeneous), and Sigma is built from Hamilton-rotated axes; mean2d == the
    homogeneous projection.                          mutations: W <-> W^T, R <-> R^T, cx <-> cy
  * Eq. 1 / Eq. 4 conic cross term: a tilted 2-D Gaussian through the whole tiled
    render equals rgb a + (1 - a) bg with a = min(0.99f, o exp(-1/2 d^T inv(Sigma2) d)),
    inv by numpy.linalg.inv.                                            mutation: B -> -B
  * P:706 / R11 SH view direction at degree 1: with the camera at a known eye and the
    Gaussian along a known unit direction u from it, colour == the hand value
    +-C1 u_k c_k + 0.5.                          mutations: d -> -d, campos = -t, campos = +R^T t
"""
import math

import numpy as np
import pytest

from oracle import render as R
from paper_2310_08528_b200.inputs import look_at


# ---------------------------------------------------------------- independent helpers
def hamilton(p, q):
    """Quaternion product p q, (w, x, y, z) — the textbook Hamilton rule."""
    pw, pv = p[0], np.asarray(p[1:], float)
    qw, qv = q[0], np.asarray(q[1:], float)
    w = pw * qw - pv @ qv
    v = pw * qv + qw * pv + np.cross(pv, qv)
    return np.concatenate([[w], v])


def rotate(q, v):
    """v' = q (0, v) q^*  for a unit quaternion q."""
    qc = np.array([q[0], -q[1], -q[2], -q[3]])
    return hamilton(hamilton(q, np.concatenate([[0.0], v])), qc)[1:]


def sigma_hamilton(s, q):
    """Sigma = sum_i s_i^2 (q e_i q*)(q e_i q*)^T : the covariance of axes s_i along the rotated
    basis vectors (Eq. 2 read geometrically, no rotation-matrix formula)."""
    S = np.zeros((3, 3))
    for i in range(3):
        e = np.zeros(3)
        e[i] = 1.0
        a = rotate(q, e)
        S += s[i] ** 2 * np.outer(a, a)
    return S


def project_h(cam, X):
    """World -> pixel by the homogeneous pinhole map u = K [R | t] X, pixel = u[:2] / u[2]."""
    K = np.array([[cam.fx, 0.0, cam.cx], [0.0, cam.fy, cam.cy], [0.0, 0.0, 1.0]])
    Rt = np.concatenate([np.asarray(cam.R, float), np.asarray(cam.t, float)[:, None]], axis=1)
    u = K @ Rt @ np.concatenate([np.asarray(X, float), [1.0]])
    return u[:2] / u[2]


def jac_numeric(cam, X, h=1e-5):
    J = np.zeros((2, 3))
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        J[:, k] = (project_h(cam, X + e) - project_h(cam, X - e)) / (2 * h)
    return J


# ---------------------------------------------------------------- fixtures of the pins
def _tilted_scene():
    """A rotated camera (generic eye, ragged W != H) and an anisotropic, rotated Gaussian off-axis,
    well inside the J clamp (R4 does not bind)."""
    cam = look_at((1.5, -0.8, 3.7), (0.2, 0.1, 0.0), 96, 72, (0.2, 0.3, 0.4))
    X = np.array([0.55, 0.35, 0.3], np.float32)
    log_s = np.log(np.array([0.09, 0.025, 0.004])).astype(np.float32)
    q = np.array([0.8, 0.3, -0.4, 0.35])
    q = (q / np.linalg.norm(q)).astype(np.float32)
    return cam, X, log_s, q


def _pre(cam, X, log_s, q, logit=0.8, dc=(0.7, -0.4, 0.1)):
    sh = np.zeros((1, 1, 3), np.float32)
    sh[0, 0] = dc
    return R.preprocess_ref(X[None], log_s[None], q[None], np.array([logit], np.float32), sh, 0, cam), sh


# ---------------------------------------------------------------- the pins (raise AssertionError)
def pin_quaternion_handedness():
    rng = np.random.default_rng(11)
    q = rng.normal(size=(200, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    v = rng.normal(size=(200, 3))
    Rm = R.quat_to_rotmat(q)
    for i in range(200):
        assert np.allclose(Rm[i] @ v[i], rotate(q[i], v[i]), atol=1e-12), i
    # textbook: +90 deg about z (right-handed) sends x to y
    c = math.cos(math.pi / 4)
    Rz = R.quat_to_rotmat(np.array([[c, 0.0, 0.0, c]]))[0]
    assert np.allclose(Rz @ [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], atol=1e-15)
    # Eq. 2 assembled by the oracle == axes rotated by the Hamilton product
    s = np.exp(rng.normal(size=(50, 3)))
    S = R.covariance3d(s, q[:50])
    for i in range(50):
        assert np.allclose(S[i], sigma_hamilton(s[i], q[i]), rtol=1e-12, atol=1e-14), i


def pin_ewa_offaxis_anisotropic():
    cam, X, log_s, q = _tilted_scene()
    pre, _ = _pre(cam, X, log_s, q)
    assert pre["kept"][0]
    Xd = X.astype(float)
    s = np.exp(log_s.astype(float))
    qd = q.astype(float) / np.linalg.norm(q.astype(float))
    Sig = sigma_hamilton(s, qd)
    Jf = jac_numeric(cam, Xd)
    S2 = Jf @ Sig @ Jf.T + 0.3 * np.eye(2)
    a, b, c = pre["cov2d"][0]
    assert abs(S2[0, 1]) > 0.2 * math.sqrt(S2[0, 0] * S2[1, 1]), "the pin needs a real cross term"
    tol = 1e-7 * max(abs(a), abs(c))
    assert abs(a - S2[0, 0]) < tol and abs(b - S2[0, 1]) < tol and abs(c - S2[1, 1]) < tol, (a, b, c, S2)
    m = project_h(cam, Xd)
    assert abs(m[0] - cam.cx) > 5 and abs(m[1] - cam.cy) > 5, "the pin needs an off-axis mean"
    assert np.allclose(pre["mean2d"][0], m, atol=1e-9), (pre["mean2d"][0], m)


def pin_conic_cross_term():
    cam, X, log_s, q = _tilted_scene()
    logit, dc = 0.8, (0.7, -0.4, 0.1)
    g = dict(means=X[None], log_scales=log_s[None], quats=q[None])
    sh = np.zeros((1, 1, 3), np.float32)
    sh[0, 0] = dc
    out = R.render_ref(g, np.array([logit], np.float32), sh, 0, cam)
    Xd = X.astype(float)
    Sig = sigma_hamilton(np.exp(log_s.astype(float)), q.astype(float) / np.linalg.norm(q.astype(float)))
    Jf = jac_numeric(cam, Xd)
    S2inv = np.linalg.inv(Jf @ Sig @ Jf.T + 0.3 * np.eye(2))
    m = project_h(cam, Xd)
    o = 1.0 / (1.0 + math.exp(-float(np.float32(logit))))
    rgb = np.maximum(0.0, np.asarray(dc, np.float32).astype(float) * (0.5 / math.sqrt(math.pi)) + 0.5)
    bg = np.asarray(cam.bg, float)
    x0, y0, x1, y1 = out["pre"]["rect"][0]
    checked = 0
    for py in range(cam.height):
        for px in range(cam.width):
            d = np.array([px - m[0], py - m[1]])
            a = min(R.ALPHA_MAX, o * math.exp(-0.5 * d @ S2inv @ d))
            inrect = x0 <= px // 16 < x1 and y0 <= py // 16 < y1
            if not inrect or abs(a - R.ALPHA_MIN) < 1e-6:
                continue
            want = rgb * a + (1 - a) * bg if a >= R.ALPHA_MIN else bg
            assert np.allclose(out["image"][:, py, px], want, atol=1e-8, rtol=0), (px, py)
            checked += a >= R.ALPHA_MIN
    assert checked > 30


C1 = math.sqrt(3.0 / (4.0 * math.pi))     # textbook |Y_1m| normalisation


def pin_sh_view_direction():
    eye = np.array([2.0, 1.0, 3.0])
    cam = look_at(eye, (0.0, 0.0, 0.0), 64, 48, (0, 0, 0))
    # coefficient k=1 (-C1 y) on red, k=2 (C1 z) on green, k=3 (-C1 x) on blue; DC 0
    sh = np.zeros((1, 4, 3), np.float32)
    sh[0, 1, 0], sh[0, 2, 1], sh[0, 3, 2] = 0.8, -0.6, 0.9
    for u in ([1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0], [0.6, 0.0, -0.8]):
        u = np.asarray(u)
        X = (eye + 2.5 * u).astype(np.float32)[None]
        rgb = R.sh_colour(X, sh, 1, cam)[0]
        want = np.maximum(0.0, [-C1 * u[1] * 0.8 + 0.5, C1 * u[2] * -0.6 + 0.5, -C1 * u[0] * 0.9 + 0.5])
        assert np.allclose(rgb, want, atol=2e-6), (u, rgb, want)


PINS = {"quat": pin_quaternion_handedness, "ewa": pin_ewa_offaxis_anisotropic,
        "conic": pin_conic_cross_term, "sh_dir": pin_sh_view_direction}


@pytest.mark.parametrize("name", sorted(PINS))
def test_pin_holds(name):
    PINS[name]()


# ---------------------------------------------------------------- mutations (each must fail a pin)
def _mut_R_transposed(mp):
    orig = R.quat_to_rotmat
    mp.setattr(R, "quat_to_rotmat", lambda q: np.transpose(orig(q), (0, 2, 1)))


def _mut_W_transposed(mp):
    def cov2d_wt(J, cam, Sigma):
        W = np.asarray(cam.R, np.float64).T
        T = J @ W
        S2 = T @ Sigma @ np.transpose(T, (0, 2, 1))
        return S2[:, 0, 0] + R.DILATION, S2[:, 0, 1], S2[:, 1, 1] + R.DILATION
    mp.setattr(R, "cov2d", cov2d_wt)


def _wrap_pre(mp, f):
    orig = R.preprocess_ref

    def pre(means, log_scales, quats, opacity_logits, sh, sh_degree, cam):
        out = orig(means, log_scales, quats, opacity_logits, sh, sh_degree, cam)
        f(out, cam)
        return out
    mp.setattr(R, "preprocess_ref", pre)


def _mut_B_sign(mp):
    def flip(out, cam):
        out["conic"] = out["conic"] * np.array([1.0, -1.0, 1.0])
    _wrap_pre(mp, flip)


def _mut_cx_cy(mp):
    def swap(out, cam):
        # mean2d = (fx x/z + cy, fy y/z + cx): the ragged W != H camera tells cx and cy apart
        out["mean2d"] = out["mean2d"] + np.array([[cam.cy - cam.cx, cam.cx - cam.cy]])
    _wrap_pre(mp, swap)


def _mut_d_neg(mp):
    orig = R.sh_to_rgb
    mp.setattr(R, "sh_to_rgb", lambda sh, d, deg: orig(sh, -np.asarray(d), deg))


def _mut_campos(sign_t_only):
    def apply(mp):
        def sh_colour(X, sh, degree, cam):
            Rc = np.asarray(cam.R, np.float64)
            t = np.asarray(cam.t, np.float64)
            campos = -t if sign_t_only else Rc.T @ t
            d = np.asarray(X, np.float64) - campos
            d = d / np.linalg.norm(d, axis=1, keepdims=True)
            return R.sh_to_rgb(sh, d, degree)
        mp.setattr(R, "sh_colour", sh_colour)
    return apply


MUTATIONS = [
    ("R_transposed", _mut_R_transposed, ["quat", "ewa"]),
    ("W_transposed", _mut_W_transposed, ["ewa", "conic"]),
    ("B_sign", _mut_B_sign, ["conic"]),
    ("cx_cy_swapped", _mut_cx_cy, ["ewa"]),
    ("d_negated", _mut_d_neg, ["sh_dir"]),
    ("campos_minus_t", _mut_campos(True), ["sh_dir"]),
    ("campos_plus_RTt", _mut_campos(False), ["sh_dir"]),
]


@pytest.mark.parametrize("name,mut,pins", MUTATIONS, ids=[m[0] for m in MUTATIONS])
def test_mutation_is_caught(monkeypatch, name, mut, pins):
    mut(monkeypatch)
    for p in pins:
        with pytest.raises(AssertionError):
            PINS[p]()
