"""One training frame (forward + L1 + TV + backward) of a config, repeated: the target for ncu captures of
the backward kernels.  Usage: python tools/bwd_one.py [config] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from paper_2310_08528_b200.inputs import make_scene  # noqa: E402
from paper_2310_08528_b200 import fgs  # noqa: E402

import test_gpu_backward as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "dnerf"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
s = make_scene(name, n_frames=2)
ds = fgs.DeviceScene(s)
cam = s.cameras[1]
target = torch.rand((3, cam.height, cam.width), generator=torch.Generator().manual_seed(0)).cuda()
for _ in range(reps):
    T._train_frame(ds, s, 1, target, 0.01)
torch.cuda.synchronize()
print("ok")
