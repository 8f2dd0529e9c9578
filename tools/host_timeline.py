"""Timeline of one fgs_frames_host call at a config (torch.profiler / CUPTI: kernels and memcpys of
every stream): prints each activity's start and end relative to the first.  Usage:
python tools/host_timeline.py [config]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_08528_b200 import build, fgs  # noqa: E402
from paper_2310_08528_b200.inputs import make_scene  # noqa: E402

build.build()
s = make_scene(sys.argv[1] if len(sys.argv) > 1 else "dnerf")
F = s.n_frames
W, H = s.cameras[0].width, s.cameras[0].height
hs = fgs.HostScene(s)
cap = 16 * s.n
himgs = [torch.empty((3, H, W)).pin_memory() for _ in range(F)]
dws = torch.empty(fgs.fgs_frames_host_workspace_bytes(hs.g, hs.field, hs.mlp, F, W, H, cap),
                  dtype=torch.uint8, device="cuda")
for _ in range(3):
    fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, himgs, dws)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, himgs, dws)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/host_trace.json")
ev = [e for e in json.load(open("/tmp/host_trace.json"))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in ev)
for e in sorted(ev, key=lambda e: e["ts"]):
    name = e["name"][:60]
    print(f"{(e['ts'] - t0) / 1e3:8.3f} -> {(e['ts'] + e['dur'] - t0) / 1e3:8.3f} ms  s{e['args'].get('stream', '?')}  {name}")
