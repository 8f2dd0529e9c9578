import torch, numpy as np
from paper_2310_08528_b200 import fgs
from paper_2310_08528_b200.inputs import make_scene
import sys; sys.path.insert(0,'tests')
from gpu_util import gpu_render_debug, gpu_deform
s = make_scene('dnerf', n_frames=3)
ds = fgs.DeviceScene(s)
for f in range(3):
    d, g, _ = gpu_deform(ds, float(s.times[f]))
    out = gpu_render_debug(ds, s.cameras[f], d)
    print(f, out['M'], int(out['tiles_touched'].sum()), out['status'], (out['ranges'][:,1]-out['ranges'][:,0]).sum())
    ne = torch.zeros((800,800), dtype=torch.int32, device='cuda'); ni = torch.zeros(1, dtype=torch.int32, device='cuda')
    aux = fgs.fgs_render_aux(n_evaluated=ne.data_ptr(), n_instances=ni.data_ptr())
    ws1 = ds.alloc_workspace(1, 16*s.n); im = torch.empty((3,800,800), device='cuda')
    fgs.fgs_render_debug(ds.cams[f], d, im, ws1, aux); torch.cuda.synchronize()
    print('  aux-only', int(ni[0]), int(ne.sum()))
