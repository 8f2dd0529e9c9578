"""Bounds of the e2e step at a config: pure device->host copy of the F images, pure host->device copy
of the model, the device-only fgs_frames step, and fgs_frames_host — CUDA events, warm, 5 repeats."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_08528_b200 import build, fgs  # noqa: E402
from paper_2310_08528_b200.inputs import make_scene  # noqa: E402

build.build()
name = sys.argv[1] if len(sys.argv) > 1 else "dnerf"
s = make_scene(name)
F = s.n_frames
W, H = s.cameras[0].width, s.cameras[0].height
dev = torch.device("cuda")
ds = fgs.DeviceScene(s, dev)
outs, _t = ds.alloc_deformed(F)
imgs = [torch.empty((3, H, W), device=dev) for _ in range(F)]
cap = 16 * s.n
ws = ds.alloc_workspace(F, cap)
himgs = [torch.empty((3, H, W)).pin_memory() for _ in range(F)]
hs = fgs.HostScene(s)
nbytes = fgs.fgs_frames_host_workspace_bytes(hs.g, hs.field, hs.mlp, F, W, H, cap)
dws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
big = torch.empty(hs.h2d_bytes(), dtype=torch.uint8).pin_memory()
bigd = torch.empty_like(big, device=dev)


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def d2h():
    for i in range(F):
        himgs[i].copy_(imgs[i], non_blocking=True)


def h2d():
    bigd.copy_(big, non_blocking=True)


def dev_step():
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, imgs, ws)


def host_step():
    fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, himgs, dws)


t_d2h, t_h2d, t_dev, t_host = timeit(d2h), timeit(h2d), timeit(dev_step), timeit(host_step)
img_bytes = F * 3 * W * H * 4
print(f"{name}: F={F} d2h {t_d2h:.3f} ms ({img_bytes / t_d2h / 1e6:.1f} GB/s)  h2d {t_h2d:.3f} ms "
      f"({hs.h2d_bytes() / t_h2d / 1e6:.1f} GB/s)  device step {t_dev:.3f} ms  host step {t_host:.3f} ms "
      f"-> e2e {F / t_host * 1e3:.0f} frames/s, bound max(d2h, h2d + dev) {F / max(t_d2h, t_h2d + t_dev) * 1e3:.0f}")
