"""Blend work-layout simulation (analysis aid, not product code): on sampled tiles of one frame, walk
each tile's sorted list with per-pixel early termination (Eq. 4; oracle preprocess / binning)
and count, for a warp layout, the warp-level Gaussian iterations (a Gaussian some live box of the warp
can reach by the exact ellipse-vs-box bound) and the box evaluations (live box x reachable).

layout "2w8x4": 2 warps per tile, each an 8-wide column block split into 4 boxes of 8x4 (round-2 kernel)
layout "1w16x4": 1 warp per tile, 4 boxes of 16x4 (each lane owns a horizontal pixel pair per box)
layout "1w8x4": 1 warp per tile, 8 boxes of 8x4
Usage: python tools/blend_layout_sim.py [config] [n_tiles]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import render as OR  # noqa: E402
from paper_2310_08528_b200.inputs import make_scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "dnerf"
ntile = int(sys.argv[2]) if len(sys.argv) > 2 else 150
s = make_scene(name, n_frames=1)
cam = s.cameras[0]
pre = OR.preprocess_ref(s.means, s.log_scales, s.quats, s.opacity_logits, s.sh, s.sh_degree, cam)
tiles, gids, ranges = OR.bin_ref(pre, cam)
gx, gy = OR.tile_grid(cam.width, cam.height)
A, B, C = pre["conic"].T
o = pre["opacity"]
m = pre["mean2d"]
thr = 2 * np.log(np.maximum(255 * o, 1e-30))


def qmin_box(g, xl, xh, yl, yh):
    a, b, c = A[g], B[g], C[g]
    inx = (xl <= 0) & (xh >= 0)
    iny = (yl <= 0) & (yh >= 0)
    best = np.where(inx & iny, 0.0, np.inf)
    for ex, cond in ((xl, xl > 0), (xh, xh < 0)):
        dy = np.clip(-b * ex / c, yl, yh)
        best = np.where(cond, np.minimum(best, a * ex * ex + 2 * b * ex * dy + c * dy * dy), best)
    for ey, cond in ((yl, yl > 0), (yh, yh < 0)):
        dx = np.clip(-b * ey / a, xl, xh)
        best = np.where(cond, np.minimum(best, a * dx * dx + 2 * b * dx * ey + c * ey * ey), best)
    return best


LAYOUTS = {
    "2w8x4": [[(bx, by, 8, 4) for by in range(0, 16, 4)] for bx in (0, 8)],
    "1w16x4": [[(0, by, 16, 4) for by in range(0, 16, 4)]],
    "1w8x8": [[(0, by, 16, 8) for by in range(0, 16, 8)]],
    "1w8x4": [[(bx, by, 8, 4) for by in range(0, 16, 4) for bx in (0, 8)]],
}
rng = np.random.default_rng(0)
lens = ranges[:, 1] - ranges[:, 0]
nz = np.nonzero(lens)[0]
sample = rng.choice(nz, min(ntile, len(nz)), replace=False)
tot = {k: [0, 0, 0] for k in LAYOUTS}   # iterations, box evaluations (boxes), pixel evaluations
contrib = 0
for t in sample:
    g = gids[ranges[t, 0]:ranges[t, 1]]
    tx, ty = t % gx, t // gx
    px, py = np.meshgrid(np.arange(16) + tx * 16, np.arange(16) + ty * 16)
    px = px.astype(float)
    py = py.astype(float)
    T = np.ones((16, 16))
    done = (px >= cam.width) | (py >= cam.height)
    # reachability of every (Gaussian, box) of every layout, and the walk with termination
    reach = {}
    for k, warps in LAYOUTS.items():
        reach[k] = []
        for boxes in warps:
            rr = []
            for (bx, by, bw, bh) in boxes:
                x0, y0 = tx * 16 + bx, ty * 16 + by
                rr.append(qmin_box(g, x0 - m[g, 0], x0 + bw - 1 - m[g, 0], y0 - m[g, 1], y0 + bh - 1 - m[g, 1])
                          <= thr[g])
            reach[k].append(np.array(rr))
    for j, gg in enumerate(g):
        if done.all():
            break
        for k, warps in LAYOUTS.items():
            for w, boxes in enumerate(warps):
                live = [not done[by:by + bh, bx:bx + bw].all() for (bx, by, bw, bh) in boxes]
                ev = [live[b] and reach[k][w][b, j] for b in range(len(boxes))]
                if any(ev):
                    tot[k][0] += 1
                    tot[k][1] += sum(ev)
                    tot[k][2] += sum(boxes[b][2] * boxes[b][3] for b in range(len(boxes)) if ev[b])
        dx = m[gg, 0] - px
        dy = m[gg, 1] - py
        power = -0.5 * (A[gg] * dx * dx + 2 * B[gg] * dx * dy + C[gg] * dy * dy)
        alpha = np.minimum(0.99, o[gg] * np.exp(power))
        ok = (~done) & (alpha >= 1 / 255.)
        tt = T * (1 - alpha)
        stop = ok & (tt < 1e-4)
        upd = ok & ~stop
        contrib += upd.sum()
        T = np.where(upd, tt, T)
        done = done | stop
scale = gx * gy / len(sample)
print(f"{name}: {len(sample)} tiles, contributing pairs per frame {contrib * scale:.3g}")
for k, (it, bx, pe) in tot.items():
    print(f"  {k:7s} iterations {it * scale:.3g}  box evals {bx * scale:.3g}  pixel evals {pe * scale:.3g}")
