"""GPU parity of the training side (§4.3) against the autograd
oracle (oracle/backward.py, itself pinned by finite differences in tests/test_oracle_backward.py).

Protocol (reading B5): both sides are fed the same fp32 inputs — for the splat backward
the GPU's own fp32 G' (as the forward parity protocol P3); gradients are compared per tensor as
max |g_gpu - g_ref| <= tol * max |g_ref| (tol 1e-4: fp32 arithmetic with ex2.approx and per-pixel
sums with cancellation against the fp64 oracle; each gradient's scale is its tensor's largest entry).
Discontinuous decisions are held fixed on both sides; scenes are chosen with no pixel in the oracle's
decision band so the two sides hold the same decisions.
"""
import dataclasses

import numpy as np
import pytest

from paper_2310_08528_b200 import fgs
from paper_2310_08528_b200.inputs import make_scene, with_heads

from gpu_util import ensure_lib

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    ensure_lib()


def _scene(n=40, W=48, H=40, deg=1, seed=0, log_scale=-2.6, heads=0.3, feat=None):
    s = make_scene("dnerf", n=n, width=W, height=H, n_frames=2, seed=seed)
    rng = np.random.default_rng(200 + seed)
    K = (deg + 1) ** 2
    f32 = np.float32
    s = dataclasses.replace(s, means=(s.means * 0.6).astype(f32),
                            log_scales=(log_scale + 0.3 * rng.normal(size=(n, 3))).astype(f32),
                            sh=np.ascontiguousarray(s.sh[:, :K, :]).astype(f32), sh_degree=deg)
    if heads:
        s = with_heads(s, heads, seed=5 + seed, bias_sigma=0.05)
    return s


def _rel(a, b):
    m = float(np.max(np.abs(b)))
    return float(np.max(np.abs(a - b))) / m if m > 0 else float(np.max(np.abs(a)))


def _forward(ds, s, frame):
    import torch
    outs, tens = ds.alloc_deformed(1)
    fgs.fgs_deform(ds.g, ds.field, ds.mlp, float(s.times[frame]), outs[0])
    cam = s.cameras[frame]
    ws = ds.alloc_workspace(1)
    img = torch.empty((3, cam.height, cam.width), device="cuda")
    fgs.fgs_render(ds.cams[frame], outs[0], img, ws)
    fgs.fgs_render_status(ws)
    return outs[0], tens[0], img, ws


@pytest.mark.parametrize("deg,seed", [(0, 0), (1, 1), (3, 2)])
def test_render_backward_matches_oracle(deg, seed):
    import torch

    from oracle import backward as B
    from oracle import render as R
    s = _scene(deg=deg, seed=seed)
    ds = fgs.DeviceScene(s)
    d, tens, img, ws = _forward(ds, s, 0)
    cam = s.cameras[0]
    w = np.random.default_rng(7 + seed).normal(size=(3, cam.height, cam.width)).astype(np.float32)
    wt = torch.from_numpy(w).cuda()
    dg, gt = ds.alloc_gaussian_grads()
    scratch = torch.empty(fgs.fgs_render_backward_scratch_bytes(s.n), dtype=torch.uint8, device="cuda")
    fgs.fgs_render_backward(ds.cams[0], d, img, wt, ws, scratch, dg)
    torch.cuda.synchronize()
    G = {k: v.cpu().numpy() for k, v in tens.items()}
    ref, ref_img = B.render_grads_ref(G, s.opacity_logits, s.sh, s.sh_degree, cam, w)
    out = R.render_ref(G, s.opacity_logits, s.sh, s.sh_degree, cam)
    assert not out["flagged"].any()
    assert np.max(np.abs(img.cpu().numpy() - ref_img)) < 2e-3
    for k in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        assert np.any(ref[k] != 0), k
        err = _rel(gt[k].cpu().numpy(), ref[k])
        assert err <= TOL, (k, err)


def test_deform_backward_matches_oracle():
    import torch

    from oracle import backward as B
    s = _scene(n=500, seed=3, heads=0.5)
    ds = fgs.DeviceScene(s)
    t = float(s.times[1])
    rng = np.random.default_rng(9)
    up = {"means": rng.normal(size=(s.n, 3)), "log_scales": rng.normal(size=(s.n, 3)),
          "quats": rng.normal(size=(s.n, 4))}
    up = {k: v.astype(np.float32) for k, v in up.items()}
    dd, dt = ds.alloc_gaussian_grads()
    for k, v in up.items():
        dt[k].copy_(torch.from_numpy(v))
    dc, ct = ds.alloc_gaussian_grads()
    df, ft = ds.alloc_field_grads()
    scratch = torch.empty(fgs.fgs_deform_backward_scratch_bytes(ds.field, ds.mlp), dtype=torch.uint8, device="cuda")
    fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, t, dd, dc, df, scratch)
    torch.cuda.synchronize()
    ref = B.deform_grads_ref(s, t, up)
    for k in ("means", "log_scales", "quats"):
        err = _rel(ct[k].cpu().numpy(), ref[k])
        assert err <= TOL, (k, err)
    for k, v in ft.items():
        assert np.any(ref[k] != 0), k
        err = _rel(v.cpu().numpy(), ref[k])
        assert err <= TOL, (k, err)
    # accumulation: a second call ADDS the field gradients
    fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, t, dd, dc, df, scratch)
    torch.cuda.synchronize()
    assert _rel(ft["w_d"].cpu().numpy(), 2 * ref["w_d"]) <= TOL


@pytest.mark.parametrize("config,n", [("neu3d", 100), ("hypernerf", 45)])
def test_deform_backward_width128_matches_oracle(config, n):
    """phi_d width 128 (the H / N3 / S fields): the deform backward's CTA-tiled path at 32 rows per CTA,
    with a ragged last CTA (100 = 3 x 32 + 4; 45 = 32 + 13), against the autograd oracle."""
    import torch

    from oracle import backward as B
    s = make_scene(config, n=n, width=48, height=40, n_frames=2, seed=4)
    s = dataclasses.replace(s, means=(s.means * 0.6).astype(np.float32))
    s = with_heads(s, 0.5, seed=11, bias_sigma=0.05)
    assert s.mlp.w_d.shape == (128, 64)
    ds = fgs.DeviceScene(s)
    t = float(s.times[1])
    rng = np.random.default_rng(19)
    up = {"means": rng.normal(size=(s.n, 3)), "log_scales": rng.normal(size=(s.n, 3)),
          "quats": rng.normal(size=(s.n, 4))}
    up = {k: v.astype(np.float32) for k, v in up.items()}
    dd, dt = ds.alloc_gaussian_grads()
    for k, v in up.items():
        dt[k].copy_(torch.from_numpy(v))
    dc, ct = ds.alloc_gaussian_grads()
    df, ft = ds.alloc_field_grads()
    scratch = torch.empty(fgs.fgs_deform_backward_scratch_bytes(ds.field, ds.mlp), dtype=torch.uint8, device="cuda")
    fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, t, dd, dc, df, scratch)
    torch.cuda.synchronize()
    ref = B.deform_grads_ref(s, t, up)
    for k in ("means", "log_scales", "quats"):
        err = _rel(ct[k].cpu().numpy(), ref[k])
        assert err <= TOL, (k, err)
    for k, v in ft.items():
        assert np.any(ref[k] != 0), k
        err = _rel(v.cpu().numpy(), ref[k])
        assert err <= TOL, (k, err)


def test_losses_match_oracle():
    """L1 value and gradient (B2), TV value and plane gradients (B1) against the oracle."""
    import torch

    from oracle import backward as B
    s = _scene(n=50)
    ds = fgs.DeviceScene(s)
    rng = np.random.default_rng(3)
    a = rng.uniform(size=(3, 37, 53)).astype(np.float32)
    b = rng.uniform(size=(3, 37, 53)).astype(np.float32)
    b[0, :3, :3] = a[0, :3, :3]                         # exact equality: zero subgradient
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    grad = torch.empty_like(at)
    part = torch.empty(fgs.FGS_LOSS_PARTIALS, dtype=torch.float64, device="cuda")
    loss = torch.empty(1, device="cuda")
    fgs.fgs_l1_loss(at, bt, grad, part, loss)
    A = torch.from_numpy(a.astype(np.float64)).requires_grad_(True)
    L = B.l1_loss(A, b)
    L.backward()
    assert abs(float(loss.item()) - float(L.detach())) <= 1e-6 * float(L.detach())
    assert np.array_equal(grad.cpu().numpy(), A.grad.numpy().astype(np.float32))
    df, ft = ds.alloc_field_grads()
    fgs.fgs_tv_loss(ds.field, 0.25, df, part, loss)
    planes = [torch.from_numpy(np.asarray(P, np.float64)).requires_grad_(True) for ps in s.field.planes for P in ps]
    Lt = 0.25 * B.tv_loss(planes)
    Lt.backward()
    assert abs(float(loss.item()) - float(Lt.detach())) <= 1e-6 * float(Lt.detach())
    q = 0
    for l, ps in enumerate(s.field.planes):
        for p in range(6):
            err = _rel(ft[f"plane{l}_{p}"].cpu().numpy(), planes[q].grad.numpy())
            assert err <= 1e-5, (l, p, err)
            q += 1


def _train_frame(ds, s, frame, target_t, tvw):
    """The whole training-side chain of one frame on the GPU; returns (loss, canonical grads, field grads)."""
    import torch
    d, tens, img, ws = _forward(ds, s, frame)
    dimg = torch.empty_like(img)
    part = torch.empty(fgs.FGS_LOSS_PARTIALS, dtype=torch.float64, device="cuda")
    l1 = torch.empty(1, device="cuda")
    tv = torch.empty(1, device="cuda")
    fgs.fgs_l1_loss(img, target_t, dimg, part, l1)
    dg, gt = ds.alloc_gaussian_grads()
    rs = torch.empty(fgs.fgs_render_backward_scratch_bytes(s.n), dtype=torch.uint8, device="cuda")
    fgs.fgs_render_backward(ds.cams[frame], d, img, dimg, ws, rs, dg)
    df, ft = ds.alloc_field_grads()
    fgs.fgs_tv_loss(ds.field, tvw, df, part, tv)
    dc, ct = ds.alloc_gaussian_grads()
    dsb = torch.empty(fgs.fgs_deform_backward_scratch_bytes(ds.field, ds.mlp), dtype=torch.uint8, device="cuda")
    fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, float(s.times[frame]), dg, dc, df, dsb)
    torch.cuda.synchronize()
    canon = {k: ct[k].cpu().numpy() for k in ("means", "log_scales", "quats")}
    # with a P:1232 decoder the canonical SH / logits gradient comes out of the deformation backward
    canon["opacity_logits"] = (ct if ds.has_a else gt)["opacity_logits"].cpu().numpy()
    canon["sh"] = (ct if ds.has_c else gt)["sh"].cpu().numpy()
    return float(l1.item() + tv.item()), canon, {k: v.cpu().numpy() for k, v in ft.items()}


def test_full_frame_gradients_match_oracle():
    """L = L1 + w L_tv of one frame, every parameter's gradient (canonical Gaussians, planes, MLP) from
    the GPU chain fgs_deform -> fgs_render -> fgs_l1_loss / fgs_tv_loss -> fgs_render_backward ->
    fgs_deform_backward, against the autograd oracle of the same frame."""
    import torch

    from oracle import backward as B
    s = _scene(n=60, W=40, H=32, deg=1, seed=4)
    ds = fgs.DeviceScene(s)
    frame = 1
    cam = s.cameras[frame]
    target = np.random.default_rng(2).uniform(size=(3, cam.height, cam.width)).astype(np.float32)
    L, canon, field = _train_frame(ds, s, frame, torch.from_numpy(target).cuda(), 0.05)
    ref, Lref, _ = B.grads_ref(s, frame, target, 0.05)
    assert abs(L - Lref) <= 1e-4 * abs(Lref)
    for k, v in canon.items():
        err = _rel(v, ref[k])
        assert err <= TOL, (k, err)
    for k, v in field.items():
        err = _rel(v, ref[k])
        assert err <= TOL, (k, err)


def test_backward_deterministic_full_size():
    """The training chain on a full-size D frame (100k Gaussians, 800x800): finite gradients, and two runs
    bit-identical (fixed-point accumulation: SPEC S:173)."""
    import torch
    s = make_scene("dnerf", n_frames=2)
    ds = fgs.DeviceScene(s)
    target = torch.rand((3, 800, 800), generator=torch.Generator().manual_seed(0)).cuda()
    a = _train_frame(ds, s, 1, target, 0.01)
    b = _train_frame(ds, s, 1, target, 0.01)
    assert a[0] == b[0]
    for x, y in ((a[1], b[1]), (a[2], b[2])):
        for k in x:
            assert np.all(np.isfinite(x[k])), k
            assert np.array_equal(x[k], y[k]), k
    assert np.abs(a[1]["means"]).max() > 0 and np.abs(a[2]["w_d"]).max() > 0


def test_backward_edge_cases():
    """Degenerate inputs of the training side: an empty set (calls succeed, nothing written), Gaussians
    behind the camera / culled (zero splat gradients), opaque Gaussians whose alpha clamps at 0.99 (the
    oracle's clamp branch: zero dalpha/de), and t at both ends of [0, 1] for the deformation backward."""
    import torch

    from oracle import backward as B
    # empty set
    s0 = _scene(n=1)
    ds0 = fgs.DeviceScene(dataclasses.replace(s0, means=s0.means[:0], log_scales=s0.log_scales[:0],
                                              quats=s0.quats[:0], opacity_logits=s0.opacity_logits[:0],
                                              sh=s0.sh[:0]))
    d, tens, img, ws = _forward(ds0, ds0.scene, 0)
    dg, _ = ds0.alloc_gaussian_grads()
    rs = torch.empty(fgs.fgs_render_backward_scratch_bytes(0), dtype=torch.uint8, device="cuda")
    fgs.fgs_render_backward(ds0.cams[0], d, img, torch.zeros_like(img), ws, rs, dg)
    # culled + clamped
    s = _scene(n=40, seed=5)
    cam0 = s.cameras[0]
    R0, t0 = cam0.R.astype(np.float64), cam0.t.astype(np.float64)
    campos = -R0.T @ t0
    s.means[:4] = (campos - 1.0 * R0[2]).astype(np.float32)   # 1 unit behind the camera: culled
    s.opacity_logits[4:12] = 12.0                          # opaque: alpha clamps at 0.99 near their centres
    ds = fgs.DeviceScene(s)
    d, tens, img, ws = _forward(ds, s, 0)
    cam = s.cameras[0]
    w = np.random.default_rng(3).normal(size=(3, cam.height, cam.width)).astype(np.float32)
    dg, gt = ds.alloc_gaussian_grads()
    rs = torch.empty(fgs.fgs_render_backward_scratch_bytes(s.n), dtype=torch.uint8, device="cuda")
    fgs.fgs_render_backward(ds.cams[0], d, img, torch.from_numpy(w).cuda(), ws, rs, dg)
    torch.cuda.synchronize()
    G = {k: v.cpu().numpy() for k, v in tens.items()}
    ref, _ = B.render_grads_ref(G, s.opacity_logits, s.sh, s.sh_degree, cam, w)
    for k in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        g = gt[k].cpu().numpy()
        assert np.all(g[:4] == 0), k
        assert _rel(g, ref[k]) <= TOL, (k, _rel(g, ref[k]))
    # deformation backward at t = 0 and t = 1
    rng = np.random.default_rng(4)
    for t in (0.0, 1.0):
        up = {"means": rng.normal(size=(s.n, 3)).astype(np.float32), "log_scales": rng.normal(size=(s.n, 3)).astype(np.float32),
              "quats": rng.normal(size=(s.n, 4)).astype(np.float32)}
        dd, dt = ds.alloc_gaussian_grads()
        for k, v in up.items():
            dt[k].copy_(torch.from_numpy(v))
        dc, ct = ds.alloc_gaussian_grads()
        df, ft = ds.alloc_field_grads()
        sb = torch.empty(fgs.fgs_deform_backward_scratch_bytes(ds.field, ds.mlp), dtype=torch.uint8, device="cuda")
        fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, t, dd, dc, df, sb)
        torch.cuda.synchronize()
        ref = B.deform_grads_ref(s, t, up)
        for k, v in list(ft.items()) + [(k, ct[k]) for k in ("means", "log_scales", "quats")]:
            assert _rel(v.cpu().numpy(), ref[k]) <= TOL, (t, k)


@pytest.mark.parametrize("deg,colour,opacity", [(1, True, True), (3, True, False), (0, False, True),
                                                (3, True, True)])
def test_deform_backward_colour_heads_match_oracle(deg, colour, opacity):
    """The P:1232 decoders phi_C / phi_alpha in the deformation backward: dL/dC', dL/dlogit' in, their
    w_c, b_c, w_a, b_a gradients, the pass-through to the canonical SH / logits, and the decoders' share
    of dL/df_d (hence of every plane and w_d, b_d), against the autograd oracle."""
    import torch

    from oracle import backward as B
    from paper_2310_08528_b200.inputs import with_colour_heads
    s = with_colour_heads(_scene(n=300, deg=deg, seed=6, heads=0.4), 0.2, 0.3, colour=colour, opacity=opacity)
    ds = fgs.DeviceScene(s)
    t = float(s.times[1])
    rng = np.random.default_rng(11)
    up = {"means": rng.normal(size=(s.n, 3)), "log_scales": rng.normal(size=(s.n, 3)),
          "quats": rng.normal(size=(s.n, 4))}
    if colour:
        up["sh"] = rng.normal(size=s.sh.shape)
    if opacity:
        up["opacity_logits"] = rng.normal(size=(s.n,))
    up = {k: v.astype(np.float32) for k, v in up.items()}
    dd, dt = ds.alloc_gaussian_grads()
    for k, v in up.items():
        dt[k].copy_(torch.from_numpy(v))
    dc, ct = ds.alloc_gaussian_grads()
    df, ft = ds.alloc_field_grads()
    assert ("w_c" in ft) == colour and ("w_a" in ft) == opacity
    scratch = torch.empty(fgs.fgs_deform_backward_scratch_bytes(ds.field, ds.mlp), dtype=torch.uint8, device="cuda")
    fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, t, dd, dc, df, scratch)
    torch.cuda.synchronize()
    ref = B.deform_grads_ref(s, t, up)
    keys = ["means", "log_scales", "quats"] + (["sh"] if colour else []) + (["opacity_logits"] if opacity else [])
    for k in keys:
        err = _rel(ct[k].cpu().numpy(), ref[k])
        assert err <= TOL, (k, err)
    if colour:     # the pass-through is exact
        assert np.array_equal(ct["sh"].cpu().numpy(), up["sh"])
    if not opacity:
        assert not ct["opacity_logits"].any()        # untouched
    for k, v in ft.items():
        assert np.any(ref[k] != 0), k
        err = _rel(v.cpu().numpy(), ref[k])
        assert err <= TOL, (k, err)


def test_full_frame_gradients_with_colour_heads():
    """The whole chain of test_full_frame_gradients_match_oracle with both P:1232 decoders: the render
    backward's SH / opacity gradients feed the deformation backward."""
    import torch

    from oracle import backward as B
    from paper_2310_08528_b200.inputs import with_colour_heads
    s = with_colour_heads(_scene(n=60, W=40, H=32, deg=1, seed=4), 0.05, 0.1)
    ds = fgs.DeviceScene(s)
    frame = 1
    cam = s.cameras[frame]
    target = np.random.default_rng(2).uniform(size=(3, cam.height, cam.width)).astype(np.float32)
    L, canon, field = _train_frame(ds, s, frame, torch.from_numpy(target).cuda(), 0.05)
    ref, Lref, _ = B.grads_ref(s, frame, target, 0.05)
    assert abs(L - Lref) <= 1e-4 * abs(Lref)
    assert set(field) >= {"w_c", "b_c", "w_a", "b_a"}
    for k, v in list(canon.items()) + list(field.items()):
        err = _rel(v, ref[k])
        assert err <= TOL, (k, err)


def test_backward_rejects_bad_arguments():
    """Synchronous validation (FGS_E_INVALID) of the training-side calls, incl. the P:1232 decoders'
    gradient pointers."""
    import torch

    from paper_2310_08528_b200.inputs import with_colour_heads
    s = _scene(n=20)
    ds = fgs.DeviceScene(s)
    d, tens, img, ws = _forward(ds, s, 0)
    dg, _ = ds.alloc_gaussian_grads()
    small = torch.empty(8, dtype=torch.uint8, device="cuda")
    with pytest.raises(fgs.FgsError) as e:
        fgs.fgs_render_backward(ds.cams[0], d, img, img, ws, small, dg)
    assert e.value.code == fgs.FGS_E_INVALID
    with pytest.raises(fgs.FgsError) as e:
        fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, 1.5, dg, dg, ds.alloc_field_grads()[0], small)
    assert e.value.code == fgs.FGS_E_INVALID
    sc = with_colour_heads(s, 0.1, 0.1)
    dsc = fgs.DeviceScene(sc)
    big = torch.empty(fgs.fgs_deform_backward_scratch_bytes(dsc.field, dsc.mlp), dtype=torch.uint8, device="cuda")
    df_no_heads = ds.alloc_field_grads()[0]          # no w_c / w_a gradient buffers
    dfc = dsc.alloc_field_grads()[0]
    dgc, _ = dsc.alloc_gaussian_grads()
    fgs.fgs_deform_backward(dsc.g, dsc.field, dsc.mlp, 0.5, dgc, dgc, dfc, big)   # the valid call
    with pytest.raises(fgs.FgsError) as e:
        fgs.fgs_deform_backward(dsc.g, dsc.field, dsc.mlp, 0.5, dgc, dgc, df_no_heads, big)
    assert e.value.code == fgs.FGS_E_INVALID


def test_adam_matches_oracle():
    """fgs_adam_step against the fp64 Adam oracle (oracle/optim.py) over a 40-step random gradient trace."""
    import torch

    from oracle import optim
    rng = np.random.default_rng(12)
    p0 = rng.normal(size=4099).astype(np.float32)
    p, m, v = (torch.from_numpy(p0.copy()).cuda(), torch.zeros(4099, device="cuda"), torch.zeros(4099, device="cuda"))
    pr, mr, vr = p0.astype(np.float64), np.zeros(4099), np.zeros(4099)
    for t in range(1, 41):
        g = (rng.normal(size=4099) * (0.01 + t % 5)).astype(np.float32)
        fgs.fgs_adam_step(p, torch.from_numpy(g).cuda(), m, v, 1.6e-3, t)
        pr, mr, vr = optim.adam_step(pr, g, mr, vr, t, 1.6e-3)
    torch.cuda.synchronize()
    assert np.max(np.abs(p.cpu().numpy() - pr)) <= 3e-6
    assert np.max(np.abs(m.cpu().numpy() - mr)) <= 1e-5 * np.abs(mr).max()


@pytest.mark.parametrize("decoders", [False, True])
def test_training_steps_reduce_the_loss(decoders):
    """The whole training side end to end on the GPU (paper's batch size 1): a scene whose means and
    opacities are perturbed from a ground truth is trained against the ground truth's renders with
    fgs_deform -> fgs_render -> fgs_l1_loss -> fgs_render_backward -> fgs_deform_backward -> fgs_adam_step;
    the L1 over the batch falls, and two runs give bit-identical loss traces (deterministic chain)."""
    import torch

    from paper_2310_08528_b200.train import Trainer
    truth = make_scene("dnerf", n=3000, width=96, height=72, n_frames=4, seed=6)
    truth = with_heads(truth, 0.1, seed=2)
    if decoders:                                   # P:1232 phi_C / phi_alpha trained too
        from paper_2310_08528_b200.inputs import with_colour_heads
        truth = with_colour_heads(truth, 0.05, 0.05)
    dst = fgs.DeviceScene(truth)
    outs, _ = dst.alloc_deformed(4)
    targets = [torch.empty((3, 72, 96), device="cuda") for _ in range(4)]
    fgs.fgs_frames(dst.g, dst.field, dst.mlp, dst.times, dst.cams, outs, targets, dst.alloc_workspace(4))
    rng = np.random.default_rng(3)
    start = dataclasses.replace(truth, means=(truth.means + rng.normal(0, 0.03, truth.means.shape)).astype(np.float32),
                                opacity_logits=(truth.opacity_logits + rng.normal(0, 0.5, truth.n)).astype(np.float32))
    traces = []
    for run in range(2):
        ds = fgs.DeviceScene(start)
        tr = Trainer(ds, lr_gaussians=2e-3, lr_field=1e-3, lr_mlp=1e-4, tv_weight=1e-3)
        losses = []
        for it in range(80):
            l1, _ = tr.step(it % 4, targets[it % 4])
            losses.append(float(l1.item()))
        traces.append(losses)
    first, last = np.mean(traces[0][:4]), np.mean(traces[0][-4:])
    assert last < 0.7 * first, (first, last)
    assert traces[0] == traces[1]
