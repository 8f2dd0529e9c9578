"""Training-side report (GPU): per-tensor gradient errors vs the autograd oracle on small scenes, and
per-stage device times of one training frame at a full-size config.  Usage: python tools/backward_report.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2310_08528_b200 import fgs  # noqa: E402
from paper_2310_08528_b200.inputs import make_scene  # noqa: E402

import test_gpu_backward as T  # noqa: E402


def errors():
    from oracle import backward as B
    out = {}
    s = T._scene(n=60, W=40, H=32, deg=1, seed=4)
    ds = fgs.DeviceScene(s)
    cam = s.cameras[1]
    target = np.random.default_rng(2).uniform(size=(3, cam.height, cam.width)).astype(np.float32)
    L, canon, field = T._train_frame(ds, s, 1, torch.from_numpy(target).cuda(), 0.05)
    ref, Lref, _ = B.grads_ref(s, 1, target, 0.05)
    out["loss_rel_err"] = abs(L - Lref) / abs(Lref)
    out["grad_rel_err"] = {k: T._rel(v, ref[k]) for k, v in {**canon, **field}.items()}
    return out


def timing(name="dnerf", reps=10):
    s = make_scene(name, n_frames=2)
    ds = fgs.DeviceScene(s)
    frame = 1
    cam = s.cameras[frame]
    target = torch.rand((3, cam.height, cam.width), generator=torch.Generator().manual_seed(0)).cuda()
    outs, tens = ds.alloc_deformed(1)
    ws = ds.alloc_workspace(1)
    img = torch.empty((3, cam.height, cam.width), device="cuda")
    dimg = torch.empty_like(img)
    part = torch.empty(fgs.FGS_LOSS_PARTIALS, dtype=torch.float64, device="cuda")
    l1 = torch.empty(1, device="cuda")
    tv = torch.empty(1, device="cuda")
    dg, _ = ds.alloc_gaussian_grads()
    df, _ = ds.alloc_field_grads()
    dc, _ = ds.alloc_gaussian_grads()
    rs = torch.empty(fgs.fgs_render_backward_scratch_bytes(s.n), dtype=torch.uint8, device="cuda")
    dsb = torch.empty(fgs.fgs_deform_backward_scratch_bytes(ds.field, ds.mlp), dtype=torch.uint8, device="cuda")
    t = float(s.times[frame])
    stages = {
        "deform": lambda: fgs.fgs_deform(ds.g, ds.field, ds.mlp, t, outs[0]),
        "render": lambda: fgs.fgs_render(ds.cams[frame], outs[0], img, ws),
        "l1_loss": lambda: fgs.fgs_l1_loss(img, target, dimg, part, l1),
        "tv_loss": lambda: fgs.fgs_tv_loss(ds.field, 0.01, df, part, tv),
        "render_backward": lambda: fgs.fgs_render_backward(ds.cams[frame], outs[0], img, dimg, ws, rs, dg),
        "deform_backward": lambda: fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, t, dg, dc, df, dsb),
    }
    for _ in range(3):
        for f in stages.values():
            f()
    torch.cuda.synchronize()
    ms = {k: 0.0 for k in stages}
    for _ in range(reps):
        for k, f in stages.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            torch.cuda.synchronize()
            ms[k] += a.elapsed_time(b) / reps
    return {"config": name, "n": s.n, "image": f"{cam.width}x{cam.height}", "ms": ms,
            "train_frame_ms": sum(ms.values()), "train_frames_per_s": 1e3 / sum(ms.values())}


if __name__ == "__main__":
    res = {"errors": errors(), "timing": [timing("dnerf"), timing("neu3d")]}
    print(json.dumps(res, indent=1))
