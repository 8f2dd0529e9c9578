"""Blend-cull statistics on the D config (analysis aid, not product code): how many (Gaussian,
warp-box) pairs survive (a) the isotropic lambda_max disc bound, (b) the exact ellipse-vs-box bound,
(c) the ideal test (some pixel of the box reaches alpha >= 1/255).  Uses the oracle's preprocess."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import render as OR
from paper_2310_08528_b200.inputs import make_scene

s = make_scene(sys.argv[1] if len(sys.argv) > 1 else "dnerf", n_frames=1)
cam = s.cameras[0]
pre = OR.preprocess_ref(s.means, s.log_scales, s.quats, s.opacity_logits, s.sh, s.sh_degree, cam)
tiles, gids, ranges = OR.bin_ref(pre, cam)
gx, gy = OR.tile_grid(cam.width, cam.height)
rng = np.random.default_rng(0)
sample = rng.choice(gx * gy, 200, replace=False)
A, B, C = pre["conic"].T
o = pre["opacity"]
m = pre["mean2d"]
cov = pre["cov2d"]
mid = 0.5 * (cov[:, 0] + cov[:, 2]); det = cov[:, 0] * cov[:, 2] - cov[:, 1] ** 2
lmax = mid + np.sqrt(np.maximum(0, mid * mid - det))
thr = 2 * np.log(np.maximum(255 * o, 1e-30))    # q <= thr  <=> alpha >= 1/255
def qmin_box(g, xl, xh, yl, yh):
    # exact min of d^T Q d over d in [xl,xh]x[yl,yh] (Q = [[A,B],[B,C]])
    a, b, c = A[g], B[g], C[g]
    inx = (xl <= 0) & (xh >= 0); iny = (yl <= 0) & (yh >= 0)
    best = np.full(len(g), np.inf)
    best[inx & iny] = 0
    for ex, cond in ((xl, xl > 0), (xh, xh < 0)):
        dy = np.clip(-b * ex / c, yl, yh)
        best = np.where(cond, np.minimum(best, a * ex * ex + 2 * b * ex * dy + c * dy * dy), best)
    for ey, cond in ((yl, yl > 0), (yh, yh < 0)):
        dx = np.clip(-b * ey / a, xl, xh)
        best = np.where(cond, np.minimum(best, a * dx * dx + 2 * b * dx * ey + c * ey * ey), best)
    return best
res = {}
for bw, bh in ((16, 16), (8, 8), (8, 4), (4, 4)):
    tot = {"list": 0, "disc": 0, "ellipse": 0, "ideal": 0}
    for t in sample:
        g = gids[ranges[t, 0]:ranges[t, 1]]
        if len(g) == 0: continue
        tx, ty = t % gx, t // gx
        for by in range(0, 16, bh):
            for bx in range(0, 16, bw):
                x0 = tx * 16 + bx; y0 = ty * 16 + by
                xl, xh = x0 - m[g, 0], x0 + bw - 1 - m[g, 0]
                yl, yh = y0 - m[g, 1], y0 + bh - 1 - m[g, 1]
                ddx = np.maximum(np.maximum(xl, -xh), 0); ddy = np.maximum(np.maximum(yl, -yh), 0)
                disc = ddx ** 2 + ddy ** 2 <= thr[g] * lmax[g]
                ell = qmin_box(g, xl, xh, yl, yh) <= thr[g]
                px, py = np.meshgrid(np.arange(x0, x0 + bw), np.arange(y0, y0 + bh))
                dx = m[g, 0][:, None] - px.ravel()[None]; dy = m[g, 1][:, None] - py.ravel()[None]
                q = A[g][:, None] * dx * dx + 2 * B[g][:, None] * dx * dy + C[g][:, None] * dy * dy
                ideal = (q <= thr[g][:, None]).any(1)
                npx = bw * bh
                tot["list"] += len(g) * npx; tot["disc"] += disc.sum() * npx
                tot["ellipse"] += ell.sum() * npx; tot["ideal"] += ideal.sum() * npx
    scale = gx * gy / len(sample)
    print(f"box {bw}x{bh}: pixel-evals per frame " + ", ".join(f"{k} {v * scale:.3g}" for k, v in tot.items()))
