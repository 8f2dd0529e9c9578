import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, os.getcwd())
import torch
from paper_2310_08528_b200 import fgs
from paper_2310_08528_b200.inputs import make_scene
n, frames, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
s = make_scene("dnerf", n=n, n_frames=frames)
ds = fgs.DeviceScene(s)
outs, _ = ds.alloc_deformed(frames)
fgs.fgs_deform_batch(ds.g, ds.field, ds.mlp, ds.times, outs)
imgs = [torch.empty((3, 800, 800), device="cuda") for _ in range(frames)]
ws = ds.alloc_workspace(frames)
fgs.fgs_set_tuning(fgs.FGS_TUNE_RADIX, mode)
for _ in range(4):
    fgs.fgs_render_batch(ds.cams, outs, imgs, ws)
torch.cuda.synchronize()
print("ok")
