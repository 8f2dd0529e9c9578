"""Small workload through every kernel of libfgs.so, for compute-sanitizer (racecheck / synccheck /
memcheck / initcheck).  Usage: compute-sanitizer --tool racecheck python tools/sanitize_run.py

Covers: the warp-specialised deform (TMEM / mbarrier pipeline, setmaxnreg re-split) at phi_d widths 32
and 64 and with the colour / opacity decoders; preprocess at SH 0 and 3; tile scan; duplicate with the
CTA-aggregated AND the direct-atomics binning path (FGS_TUNE_AGG_TILES); the warp tile sort and the
persistent long-list CTA sort with its work queue (FGS_TUNE_TILE_SORT_CAP lowered); the blend with and
without the cull; the debug copy; fgs_frames_host's copy streams.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2310_08528_b200 import build, fgs  # noqa: E402
from paper_2310_08528_b200.inputs import make_scene, with_colour_heads  # noqa: E402


def frames(s, ws_frames=None):
    ds = fgs.DeviceScene(s)
    F = s.n_frames
    W, H = s.cameras[0].width, s.cameras[0].height
    outs, _ = ds.alloc_deformed(F)
    imgs = [torch.empty((3, H, W), device="cuda") for _ in range(F)]
    ws = ds.alloc_workspace(F, 16 * s.n)
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, imgs, ws)
    fgs.fgs_render_status(ws, F)
    torch.cuda.synchronize()
    return ds, outs


def main():
    build.build()
    fgs.lib()
    s_tiny = make_scene("tiny", n=2011, n_frames=2)
    frames(s_tiny)
    s_d = make_scene("dnerf", n=6000, width=160, height=128, n_frames=2)
    ds, outs = frames(s_d)
    # long-list CTA sort + direct-atomics binning + unculled blend
    with fgs.tuning(fgs.FGS_TUNE_TILE_SORT_CAP, 32), fgs.tuning(fgs.FGS_TUNE_AGG_TILES, 1):
        frames(s_d)
    with fgs.tuning(fgs.FGS_TUNE_BLEND_CULL, 0):
        frames(s_d)
    # debug render (debug copy kernel, DBG blend)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from gpu_util import gpu_render_debug
    gpu_render_debug(ds, s_d.cameras[0], outs[0])
    # phi_d width 128 + the P:1232 decoders
    frames(with_colour_heads(make_scene("hypernerf", n=3001, width=96, height=64, n_frames=2), 0.1, 0.2))
    # host path
    hs = fgs.HostScene(s_d)
    nbytes = fgs.fgs_frames_host_workspace_bytes(hs.g, hs.field, hs.mlp, 2, 160, 128, 16 * s_d.n)
    dws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    himgs = [torch.empty((3, 128, 160)).pin_memory() for _ in range(2)]
    fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, himgs, dws)
    fgs.fgs_frames_host_status(hs.g, hs.field, hs.mlp, hs.cams, dws)
    torch.cuda.synchronize()
    print("sanitize workload done, launches:", fgs.fgs_launch_count())


if __name__ == "__main__":
    main()
