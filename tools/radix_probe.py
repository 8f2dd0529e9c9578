"""Time fgs_render_batch of a few frames with the per-tile sorts vs the radix binning path (eager and
CUDA graph, with and without an L2 flush between reps) — the binning path selection experiment."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2310_08528_b200 import fgs  # noqa: E402
from paper_2310_08528_b200.inputs import make_scene  # noqa: E402


def run(n, frames, mode, flush, graph, reps=10):
    s = make_scene("dnerf", n=n, n_frames=frames)
    ds = fgs.DeviceScene(s)
    outs, _ = ds.alloc_deformed(frames)
    fgs.fgs_deform_batch(ds.g, ds.field, ds.mlp, ds.times, outs)
    imgs = [torch.empty((3, 800, 800), device="cuda") for _ in range(frames)]
    ws = ds.alloc_workspace(frames)
    fl = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    fgs.fgs_set_tuning(fgs.FGS_TUNE_RADIX, mode)

    def step():
        fgs.fgs_render_batch(ds.cams, outs, imgs, ws)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    g = None
    if graph:
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            step()
            st.synchronize()
            with torch.cuda.graph(g, stream=st):
                step()
        torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush:
            fl.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay() if g is not None else step()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    fgs.fgs_render_status(ws, frames)
    fgs.fgs_set_tuning(fgs.FGS_TUNE_RADIX, 1)
    ts.sort()
    return ts[len(ts) // 2] * 1e3 / frames


if __name__ == "__main__":
    res = []
    for n in (int(x) for x in sys.argv[1:] or [1_000_000]):
        for frames in (1, 4):
            for mode in (0, 2):
                for flush in (False, True):
                    for graph in (False, True):
                        us = run(n, frames, mode, flush, graph)
                        res.append(dict(n=n, frames=frames, radix=mode, flush=flush, graph=graph, us_per_frame=us))
                        print(json.dumps(res[-1]), flush=True)
