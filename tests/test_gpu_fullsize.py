"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times.

Every config runs through `fgs_frames` exactly as bench.py does (one call: the whole batch of (t, view)
frames deformed and rendered in shared launches).  The oracle cannot redo whole frames at these sizes
in seconds, so the comparison is on samples it computes one by one:
  * deformation: a contiguous window of Gaussians plus the ragged tail of the array, for the first and
    last frame of the batch — max |err| <= 1e-4 (north_star);
  * integer work: radii, rects, tiles_touched and depth keys of ALL Gaussians of a frame (the oracle's
    preprocess is vectorised), and the ordered per-tile lists of sampled tiles, via fgs_render_debug on
    the batch's own G' (bit-exact outside boundary Gaussians);
  * pixels: sampled tiles of the batch images vs the oracle fed the GPU's fp32 G' (PSNR >= 60 dB, max
    |err| <= 2e-3 on unflagged pixels), and the batch image equals the single-frame render bit for bit.
"""
import numpy as np
import pytest

import oracle
from oracle import render as OR
from paper_2310_08528_b200 import fgs
from paper_2310_08528_b200.inputs import make_scene

from gpu_util import compare_pixels, ensure_lib, gpu_render_debug

pytestmark = pytest.mark.gpu

DEFORM_TOL = 1e-4
PIX_TOL = 2e-3
PSNR_MIN = 60.0

# (config, frames in the batch): the bench batches of D (20) and N3 (8); H and S with fewer frames of
# the same per-frame size (their full batches only repeat the same kernels with other t / cameras).
CASES = [("dnerf", None, None), ("neu3d", None, None), ("hypernerf", 6, None), ("scaling", 3, None),
         ("dnerf", 4, 1_000_000), ("dnerf", 4, 10_000)]     # ends of the N sweep


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    ensure_lib()


def _run_frames(s):
    import torch
    ds = fgs.DeviceScene(s)
    F = s.n_frames
    W, H = s.cameras[0].width, s.cameras[0].height
    outs, tens = ds.alloc_deformed(F)
    imgs = [torch.empty((3, H, W), dtype=torch.float32, device="cuda") for _ in range(F)]
    ws = ds.alloc_workspace(F, 16 * s.n)
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, imgs, ws)
    fgs.fgs_render_status(ws, F)
    torch.cuda.synchronize()
    return ds, outs, tens, imgs


@pytest.mark.parametrize("name,frames,n", CASES)
def test_fullsize_batch_parity(name, frames, n):
    s = make_scene(name, n_frames=frames, n=n)
    ds, outs, tens, imgs = _run_frames(s)
    F = s.n_frames
    n = s.n
    rng = np.random.default_rng(123)
    W, H = s.cameras[0].width, s.cameras[0].height
    gx, gy = OR.tile_grid(W, H)
    for f in sorted({0, F - 1}):
        t = float(s.times[f])
        # ---- deformation: a window + the ragged tail ----
        b = int(rng.integers(0, n - 4096))
        # frames sharing a time render from the first such frame's G' (fgs_frames deforms each t once)
        f0 = next(i for i in range(F) if np.float32(s.times[i]).tobytes() == np.float32(t).tobytes())
        g = {k: v.cpu().numpy() for k, v in tens[f0].items()}
        for (lo, hi) in ((b, b + 4096), (n - 77, n)):
            ref = oracle.deform_ref(s, t, begin=lo, end=hi)
            err = max(float(np.abs(g[k][lo:hi].astype(np.float64) - ref[k]).max()) for k in ref)
            assert err <= DEFORM_TOL, (name, f, lo, err)
        # ---- integer work on the batch's own G' (all Gaussians) ----
        cam = s.cameras[f]
        pre = OR.preprocess_ref(g["means"], g["log_scales"], g["quats"], s.opacity_logits, s.sh, s.sh_degree, cam)
        dbg = gpu_render_debug(ds, cam, outs[f0])
        assert dbg["status"] == fgs.FGS_OK
        keep = ~pre["boundary"]
        assert np.sum((dbg["radii"][:n] != pre["radius"]) & keep) == 0
        assert np.sum(np.any(dbg["rect"][:n] != pre["rect"], axis=1) & keep) == 0
        assert np.sum((dbg["tiles_touched"][:n] != pre["tiles_touched"]) & keep) == 0
        assert np.sum((dbg["depth_key"][:n] != pre["depth_key"]) & keep) == 0
        # the batch image is the single-frame render, bit for bit
        assert np.array_equal(imgs[f].cpu().numpy(), dbg["image"])
        # ---- sampled tiles: lists and pixels ----
        lens = np.diff(dbg["ranges"], axis=1)[:, 0]
        busiest = np.argsort(lens)[-3:].tolist()
        tiles = sorted(set(rng.choice(gx * gy, 12, replace=False).tolist()) | set(busiest) | {gx * gy - 1})
        for tile in tiles:
            want = OR.tile_list_ref(pre, cam, tile)
            st, en = dbg["ranges"][tile]
            got = dbg["sorted_gid"][st:en]
            assert np.array_equal(got[keep[got]], want[keep[want]]), (name, f, tile)
        ref = OR.render_ref(g, s.opacity_logits, s.sh, s.sh_degree, cam, tiles_subset=tiles, pre=pre,
                            full_bins=False)
        pix = compare_pixels(imgs[f].cpu().numpy(), ref["image"], ref["flagged"])
        assert pix["psnr"] >= PSNR_MIN and pix["max_unflagged"] <= PIX_TOL, (name, f, pix)


@pytest.mark.parametrize("name", ["dnerf", "scaling"])
def test_blend_cull_exact_on_whole_fullsize_frames(name):
    """The blend's per-warp ellipse cull (Eq. 4 evaluations skipped when alpha < 1/255 on a whole 8x4
    sub-box) must not change any pixel: two full-size frames (D: all 2,500 tiles; S: all 8,160 tiles of
    1920x1080 with 2M Gaussians), image / final T / contributor counts bit-identical with the cull on
    and off (FGS_TUNE_BLEND_CULL)."""
    s = make_scene(name, n_frames=2)
    ds, outs, tens, imgs = _run_frames(s)
    for f in range(2):
        # frames sharing a time render from the first such frame's G' (fgs_frames deforms each t once)
        f0 = next(i for i in range(2) if np.float32(s.times[i]).tobytes() == np.float32(s.times[f]).tobytes())
        on = gpu_render_debug(ds, s.cameras[f], outs[f0])
        with fgs.tuning(fgs.FGS_TUNE_BLEND_CULL, 0):
            off = gpu_render_debug(ds, s.cameras[f], outs[f0])
        assert on["status"] == off["status"] == fgs.FGS_OK
        for k in ("image", "final_T", "n_contrib"):
            assert np.array_equal(on[k], off[k]), (name, f, k, int(np.sum(on[k] != off[k])))
        assert np.array_equal(imgs[f].cpu().numpy(), on["image"])
        # the cull really skipped work: fewer (warp, Gaussian) evaluations than the unculled loop
        assert on["blend_work"][0] < off["blend_work"][0]


@pytest.mark.parametrize("name", ["dnerf", "scaling", "neu3d"])
def test_tile_cull_exact_on_whole_fullsize_frames(name):
    """FGS_TUNE_TILE_CULL = 1 (non-contributing (tile, Gaussian) pairs left out of the lists) must not
    change any pixel: two full-size frames per config, image / final T / contributor counts bit-identical
    with the knob on and off, the lists shorter, and no tile's list longer than before."""
    s = make_scene(name, n_frames=2)
    ds, outs, tens, imgs = _run_frames(s)
    for f in range(2):
        f0 = next(i for i in range(2) if np.float32(s.times[i]).tobytes() == np.float32(s.times[f]).tobytes())
        off = gpu_render_debug(ds, s.cameras[f], outs[f0])
        with fgs.tuning(fgs.FGS_TUNE_TILE_CULL, 1):
            on = gpu_render_debug(ds, s.cameras[f], outs[f0])
        assert on["status"] == off["status"] == fgs.FGS_OK
        for k in ("image", "final_T", "n_contrib"):
            assert np.array_equal(on[k], off[k]), (name, f, k, int(np.sum(on[k] != off[k])))
        assert on["M"] < off["M"]
        assert np.all(np.diff(on["ranges"], axis=1) <= np.diff(off["ranges"], axis=1))
    # and through fgs_frames (the batch path) with the knob on
    with fgs.tuning(fgs.FGS_TUNE_TILE_CULL, 1):
        ds2, outs2, tens2, imgs2 = _run_frames(s)
    for f in range(2):
        assert np.array_equal(imgs[f].cpu().numpy(), imgs2[f].cpu().numpy()), (name, f)

