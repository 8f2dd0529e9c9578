"""Pins for the gradient oracle (oracle/backward.py) — CPU only.

The oracle differentiates a torch restatement of the forward with autograd; it is pinned to things
other than itself:
  * its forward equals the numpy forward oracle (deform_ref, render_ref) to 1e-12;
  * every gradient equals central finite differences of the NUMPY forward (fp64 inputs, h = 1e-6),
    with the stencil checked to flip no decision (same contributor count at every pixel) — the SPEC
    S:156/S:162/S:229/S:297 finite-difference oracle;
  * L_tv and L1 worked examples; zero upstream -> zero gradients (S:154,
    S:228); linearity over queries; plane-gradient sparsity.
"""
import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import backward as B  # noqa: E402
from oracle import render as R  # noqa: E402
from paper_2310_08528_b200.inputs import make_scene, with_heads  # noqa: E402


def _small_scene(n=12, W=32, H=28, deg=1, seed=0, log_scale=-1.6, heads=0.3):
    """A few large Gaussians in view of a ragged image, non-trivial heads (so every path carries
    gradient), SH degree `deg`; arrays promoted to float64 (finite differences below fp32 spacing)."""
    s = make_scene("dnerf", n=n, width=W, height=H, n_frames=2, seed=seed)
    rng = np.random.default_rng(100 + seed)
    K = (deg + 1) ** 2
    s = dataclasses.replace(
        s, means=(s.means * 0.6).astype(np.float64),
        log_scales=(log_scale + 0.3 * rng.normal(size=(n, 3))).astype(np.float64),
        quats=s.quats.astype(np.float64), opacity_logits=s.opacity_logits.astype(np.float64),
        sh=np.ascontiguousarray(s.sh[:, :K, :]).astype(np.float64), sh_degree=deg)
    if heads:
        s = with_heads(s, heads, seed=3 + seed, bias_sigma=0.05)
    return s


def _np_render(G, s, frame=0):
    return R.render_ref(G, s.opacity_logits, s.sh, s.sh_degree, s.cameras[frame])


# ------------------------------------------------------------------ forward equals the numpy oracle
def test_torch_forward_equals_numpy_oracle():
    s = _small_scene()
    t = float(s.times[1])
    P = B.params_of(s)
    G = B.deform_torch(s, t, P)
    Gn = oracle.deform_ref(s, t)
    for k in Gn:
        assert np.max(np.abs(G[k].detach().numpy() - Gn[k])) < 1e-12, k
    img = B.render_torch(G, P["opacity_logits"], P["sh"], s.sh_degree, s.cameras[1]).detach().numpy()
    ref = _np_render(Gn, s, 1)["image"]
    assert np.max(np.abs(img - ref)) < 1e-12
    assert np.mean(np.abs(ref - np.asarray(s.cameras[1].bg)[:, None, None])) > 1e-2   # not an empty frame


# ------------------------------------------------------------------ worked examples
def test_tv_worked_examples():
    """a constant plane -> 0; [[0,1],[0,1]] -> horizontal diffs 1,1, vertical 0,0 -> 0.5."""
    assert float(B.tv_loss([torch.full((3, 4, 2), 0.7, dtype=torch.float64)])) == 0.0
    P = torch.tensor([[0.0, 1.0], [0.0, 1.0]], dtype=torch.float64)[:, :, None]
    assert float(B.tv_loss([P])) == 0.5
    # pooled over planes: a second, constant 2x2 plane adds 4 zero terms -> 2 / 8
    assert float(B.tv_loss([P, torch.zeros((2, 2, 1), dtype=torch.float64)])) == 0.25


def test_l1_worked_examples():
    """identical images -> 0; all 1 vs all 0 -> 1; a scalar-loop recomputation."""
    a = np.random.default_rng(0).uniform(size=(3, 5, 7))
    assert float(B.l1_loss(torch.as_tensor(a), a)) == 0.0
    assert float(B.l1_loss(torch.ones((3, 2, 2), dtype=torch.float64), np.zeros((3, 2, 2)))) == 1.0
    b = np.random.default_rng(1).uniform(size=(3, 5, 7))
    loop = sum(abs(a[c, y, x] - b[c, y, x]) for c in range(3) for y in range(5) for x in range(7)) / a.size
    assert abs(float(B.l1_loss(torch.as_tensor(a), b)) - loop) < 1e-15


# ------------------------------------------------------------------ finite differences
def _fd_check(f_np, x, grad, idxs, h=1e-6, rtol=1e-4, decisions=None):
    """Central differences of the numpy scalar function f_np(x) at the flat indices idxs."""
    gmax = float(np.max(np.abs(grad))) if grad.size else 0.0
    checked = 0
    for i in idxs:
        xp = x.copy().reshape(-1)
        xm = x.copy().reshape(-1)
        xp[i] += h
        xm[i] -= h
        (fp, dp), (fm, dm) = f_np(xp.reshape(x.shape)), f_np(xm.reshape(x.shape))
        if decisions is not None and not (decisions(dp) and decisions(dm)):
            continue                                 # a decision flips inside the stencil: excluded
        fd = (fp - fm) / (2 * h)
        an = grad.reshape(-1)[i]
        assert abs(fd - an) <= rtol * max(abs(an), 1e-3 * gmax) + 1e-10, (i, fd, an)
        checked += 1
    return checked


@pytest.mark.parametrize("deg", [0, 1, 3])
def test_render_gradients_match_finite_differences(deg):
    """Splat backward: gradients of sum(w * I^) w.r.t. X', s', r' (raw), opacity logits
    and SH, for random upstream weights w, against central differences of oracle.render.render_ref."""
    s = _small_scene(deg=deg, seed=deg)
    cam = s.cameras[0]
    G = oracle.deform_ref(s, float(s.times[0]))
    w = np.random.default_rng(7).normal(size=(3, cam.height, cam.width))
    grads, img = B.render_grads_ref(G, s.opacity_logits, s.sh, s.sh_degree, cam, w)
    base = _np_render(G, s)
    nc0 = base["n_contrib"]

    def ok(out):            # the stencil flips no skip / stop decision (contributor counts unchanged)
        return np.array_equal(out["n_contrib"], nc0)

    total = 0
    for key in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        x0 = (G[key] if key in G else getattr(s, key)).astype(np.float64)

        def f(x, key=key):
            if key in G:
                out = R.render_ref({**G, key: x}, s.opacity_logits, s.sh, s.sh_degree, cam)
            elif key == "opacity_logits":
                out = R.render_ref(G, x, s.sh, s.sh_degree, cam)
            else:
                out = R.render_ref(G, s.opacity_logits, x, s.sh_degree, cam)
            return float(np.sum(w * out["image"])), out

        idxs = range(x0.size) if x0.size <= 64 else np.random.default_rng(1).choice(x0.size, 64, replace=False)
        total += _fd_check(f, x0, grads[key], idxs, decisions=ok)
        assert np.any(grads[key] != 0), key
    assert total > 150


def test_deform_gradients_match_finite_differences():
    """HexPlane + phi_d + heads backward: gradients of sum <w, G'> w.r.t.
    canonical X (both paths), s, r, the planes (the touched vertices and untouched ones) and the MLP."""
    s = _small_scene(n=6, seed=4, heads=0.5)
    t = float(s.times[1])
    rng = np.random.default_rng(5)
    w = {k: rng.normal(size=v.shape) for k, v in oracle.deform_ref(s, t).items()}
    grads = B.deform_grads_ref(s, t, w)

    def f_of(mutate):
        def f(x):
            s2 = mutate(x)
            G = oracle.deform_ref(s2, t)
            return float(sum(np.sum(w[k] * G[k]) for k in G)), None
        return f

    checked = 0
    for key in ("means", "log_scales", "quats"):
        x0 = getattr(s, key).astype(np.float64)
        checked += _fd_check(f_of(lambda x, key=key: dataclasses.replace(s, **{key: x})), x0, grads[key],
                             range(x0.size))
    f = s.field
    for l in range(len(f.planes)):
        for p in range(6):
            P0 = f.planes[l][p].astype(np.float64)
            g = grads[f"plane{l}_{p}"]
            nz = np.flatnonzero(g)
            idxs = list(rng.choice(nz, min(12, nz.size), replace=False)) + list(rng.choice(P0.size, 4, replace=False))

            def mut(x, l=l, p=p):
                planes = [list(ps) for ps in f.planes]
                planes[l][p] = x
                return dataclasses.replace(s, field=dataclasses.replace(f, planes=planes))
            checked += _fd_check(f_of(mut), P0, g, idxs)
    for k in ("w_d", "b_d", "w_x", "b_x", "w_r", "b_r", "w_s", "b_s"):
        x0 = getattr(s.mlp, k).astype(np.float64)
        idxs = range(x0.size) if x0.size <= 40 else rng.choice(x0.size, 40, replace=False)
        checked += _fd_check(f_of(lambda x, k=k: dataclasses.replace(s, mlp=dataclasses.replace(s.mlp, **{k: x}))),
                             x0, grads[k], idxs)
    assert checked > 300


def test_full_frame_loss_gradients_match_finite_differences():
    """The whole chain: L = |I^ - I| + w L_tv -> render -> deform -> encode -> planes, on a
    16x16 frame of 8 Gaussians, every parameter group sampled, against central differences of the numpy
    forward oracle + the numpy loss."""
    s = _small_scene(n=8, W=16, H=16, deg=1, seed=2, log_scale=-1.3)
    frame, tvw = 1, 0.05
    cam = s.cameras[frame]
    target = np.random.default_rng(9).uniform(size=(3, cam.height, cam.width))
    grads, L, img = B.grads_ref(s, frame, target, tvw)
    t = float(s.times[frame])

    def np_loss(s2):
        G = oracle.deform_ref(s2, t)
        out = R.render_ref(G, s2.opacity_logits, s2.sh, s2.sh_degree, cam)
        tv_terms = []
        for ps in s2.field.planes:
            for Pl in ps:
                Pl = np.asarray(Pl, np.float64)
                tv_terms += [((Pl[:, 1:] - Pl[:, :-1]) ** 2).ravel(), ((Pl[1:] - Pl[:-1]) ** 2).ravel()]
        return float(np.mean(np.abs(out["image"] - target)) + tvw * np.mean(np.concatenate(tv_terms))), out

    base_L, base = np_loss(s)
    assert abs(base_L - L) < 1e-12
    nc0 = base["n_contrib"]

    def ok(out):
        return np.array_equal(out["n_contrib"], nc0)

    rng = np.random.default_rng(11)
    checked = 0
    groups = {"means": lambda x: dataclasses.replace(s, means=x), "log_scales": lambda x: dataclasses.replace(s, log_scales=x),
              "quats": lambda x: dataclasses.replace(s, quats=x),
              "opacity_logits": lambda x: dataclasses.replace(s, opacity_logits=x), "sh": lambda x: dataclasses.replace(s, sh=x)}
    for k, mut in groups.items():
        x0 = getattr(s, k).astype(np.float64)
        idxs = rng.choice(x0.size, min(16, x0.size), replace=False)
        checked += _fd_check(lambda x, mut=mut: np_loss(mut(x)), x0, grads[k], idxs, decisions=ok)
    f = s.field
    for l, p in ((0, 0), (0, 3), (1, 2), (1, 5)):
        P0 = f.planes[l][p].astype(np.float64)
        nz = np.flatnonzero(np.abs(grads[f"plane{l}_{p}"]) > 1e-6 * np.abs(grads[f"plane{l}_{p}"]).max())

        def mut(x, l=l, p=p):
            planes = [list(ps) for ps in f.planes]
            planes[l][p] = x
            return dataclasses.replace(s, field=dataclasses.replace(f, planes=planes))
        checked += _fd_check(lambda x, mut=mut: np_loss(mut(x)), P0, grads[f"plane{l}_{p}"],
                             rng.choice(nz, min(10, nz.size), replace=False), decisions=ok)
    for k in ("w_d", "b_d", "w_x", "w_r", "w_s"):
        x0 = getattr(s.mlp, k).astype(np.float64)

        def mut(x, k=k):
            return dataclasses.replace(s, mlp=dataclasses.replace(s.mlp, **{k: x}))
        checked += _fd_check(lambda x, mut=mut: np_loss(mut(x)), x0, grads[k],
                             rng.choice(x0.size, min(10, x0.size), replace=False), decisions=ok)
    assert checked > 100


# ------------------------------------------------------------------ invariants
def test_zero_upstream_gives_zero_gradients():
    """SPEC S:154 / S:228: dL/dImage = 0 -> every splat gradient 0; dL/dG' = 0 -> every field gradient 0."""
    s = _small_scene(n=5)
    G = oracle.deform_ref(s, float(s.times[0]))
    cam = s.cameras[0]
    g, _ = B.render_grads_ref(G, s.opacity_logits, s.sh, s.sh_degree, cam, np.zeros((3, cam.height, cam.width)))
    assert all(np.all(v == 0) for v in g.values())
    d = B.deform_grads_ref(s, 0.3, {k: np.zeros_like(v) for k, v in G.items()})
    assert all(np.all(v == 0) for v in d.values())


def test_plane_gradient_sparsity_and_linearity():
    """one query writes non-zero gradients to at most 4 vertices of each of the 6 planes of
    each scale; the gradients of a batch are the sum of the per-query gradients."""
    s = _small_scene(n=3, seed=6)
    t = 0.41
    rng = np.random.default_rng(2)
    w = {k: rng.normal(size=v.shape) for k, v in oracle.deform_ref(s, t).items()}
    full = B.deform_grads_ref(s, t, w)
    acc = None
    for i in range(3):
        wi = {k: np.where(np.arange(3)[:, None] == i, v, 0.0) for k, v in w.items()}
        gi = B.deform_grads_ref(s, t, wi)
        for l in range(len(s.field.planes)):
            for p in range(6):
                verts = np.any(gi[f"plane{l}_{p}"] != 0, axis=-1)
                assert verts.sum() <= 4, (i, l, p)
        acc = gi if acc is None else {k: acc[k] + gi[k] for k in acc}
    for k in full:
        assert np.allclose(full[k], acc[k], rtol=0, atol=1e-12 * max(1.0, np.abs(full[k]).max())), k


def test_colour_opacity_decoder_gradients_match_finite_differences():
    """P:1232 decoders: with phi_C / phi_alpha the deformed SH and opacity logits are G' outputs too; their
    gradients w.r.t. W_c, b_c, W_a, b_a, the shared phi_d / W_d / planes and the canonical SH / logits
    against central differences of oracle.deform.deform_ref (which applies the decoders)."""
    from paper_2310_08528_b200.inputs import with_colour_heads
    s = with_colour_heads(_small_scene(n=5, seed=7, heads=0.3), 0.2, 0.3)
    s = dataclasses.replace(s, sh=s.sh.astype(np.float64), opacity_logits=s.opacity_logits.astype(np.float64))
    t = float(s.times[0])
    rng = np.random.default_rng(8)
    w = {k: rng.normal(size=np.shape(v)) for k, v in oracle.deform_ref(s, t).items()}
    assert set(w) == {"means", "log_scales", "quats", "sh", "opacity_logits"}
    grads = B.deform_grads_ref(s, t, w)

    def f_of(mutate):
        def f(x):
            G = oracle.deform_ref(mutate(x), t)
            return float(sum(np.sum(w[k] * G[k]) for k in G)), None
        return f

    checked = 0
    for k in ("w_c", "b_c", "w_a", "b_a", "w_d", "b_d"):
        x0 = getattr(s.mlp, k).astype(np.float64)
        idxs = range(x0.size) if x0.size <= 30 else rng.choice(x0.size, 30, replace=False)
        checked += _fd_check(f_of(lambda x, k=k: dataclasses.replace(s, mlp=dataclasses.replace(s.mlp, **{k: x}))),
                             x0, grads[k], idxs)
    for k in ("sh", "opacity_logits", "means"):
        x0 = getattr(s, k).astype(np.float64)
        idxs = range(x0.size) if x0.size <= 40 else rng.choice(x0.size, 40, replace=False)
        checked += _fd_check(f_of(lambda x, k=k: dataclasses.replace(s, **{k: x})), x0, grads[k], idxs)
    # the canonical SH / logits enter additively: their gradient is the upstream one
    assert np.allclose(grads["sh"], w["sh"], rtol=0, atol=1e-12)
    assert np.allclose(grads["opacity_logits"], w["opacity_logits"], rtol=0, atol=1e-12)
    assert checked > 150
