"""FGS_TUNE_TILE_CULL on vs off: images / final T / contributor counts bit-identical, instance counts, stage times.
    python tools/tile_cull_check.py [config] [frames]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import numpy as np
import torch
from paper_2310_08528_b200 import fgs
from paper_2310_08528_b200.inputs import make_scene

cfg = sys.argv[1] if len(sys.argv) > 1 else "dnerf"
F = int(sys.argv[2]) if len(sys.argv) > 2 else 4
s = make_scene(cfg, n_frames=F)
dev = torch.device("cuda:0")
ds = fgs.DeviceScene(s, dev)
W, H = s.cameras[0].width, s.cameras[0].height
outs, _ = ds.alloc_deformed(F)
ws = ds.alloc_workspace(F, 16 * s.n)
res = {}
for mode in (0, 1):
    fgs.fgs_set_tuning(fgs.FGS_TUNE_TILE_CULL, mode)
    imgs = [torch.empty((3, H, W), device=dev) for _ in range(F)]
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, imgs, ws)
    fgs.fgs_render_status(ws, F)
    torch.cuda.synchronize()
    fgs.fgs_profile_enable(True); fgs.fgs_profile_read()
    for _ in range(5):
        fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, imgs, ws)
    torch.cuda.synchronize()
    st = fgs.fgs_profile_read(); fgs.fgs_profile_enable(False)
    res[mode] = (imgs, st)
same = all(torch.equal(a, b) for a, b in zip(res[0][0], res[1][0]))
print(json.dumps({"config": cfg, "frames": F, "images_identical": same,
                  "stages_off": str(res[0][1]), "stages_on": str(res[1][1])}))
