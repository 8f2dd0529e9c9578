"""GPU parity: the sm_100a path (through the C ABI) against the fp64 oracle.

Tolerances (BASELINE.json north_star):
  * deformed means / log-scales / raw quats: max |err| <= 1e-4 (also on the stress heads N(0,1));
  * integer work (radii, rects, tiles_touched, depth keys, per-tile ordered lists) bit-exact except
    boundary Gaussians (within 1e-5 px of a tile-rule boundary, see oracle.render.BAND_PX);
  * pixels: PSNR >= 60 dB over all pixels, max |err| <= 2e-3 over pixels whose blend decisions are
    not within relative 1e-4 of a threshold (reading P1).
Integer and pixel checks feed BOTH sides the GPU's fp32 G' (so the deform tolerance cannot move
rects).
"""
import numpy as np
import pytest

import oracle
from oracle import render as OR
from paper_2310_08528_b200 import fgs
from paper_2310_08528_b200.inputs import make_scene, with_heads, with_max_opacity

from gpu_util import compare_integer_work, compare_pixels, ensure_lib, gpu_deform, gpu_render_debug

pytestmark = pytest.mark.gpu

DEFORM_TOL = 1e-4
PIX_TOL = 2e-3
PSNR_MIN = 60.0


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    ensure_lib()


def _ds(scene):
    return fgs.DeviceScene(scene)


def _deform_err(scene, g, t):
    ref = oracle.deform_ref(scene, t)
    return max(float(np.max(np.abs(g[k].astype(np.float64) - ref[k]))) for k in ref)


@pytest.mark.parametrize("variant", ["tiny", "tiny_stress", "dnerf_sub", "dnerf_sub_stress", "hyper_sub"])
def test_deform_matches_oracle(variant):
    if variant.startswith("tiny"):
        s = make_scene("tiny", n=2011)                       # ragged last tile of 64
    elif variant.startswith("dnerf"):
        s = make_scene("dnerf", n=20_003, n_frames=3)
    else:
        s = make_scene("hypernerf", n=5_000, n_frames=2)
    if variant.endswith("stress"):
        s = with_heads(s, 1.0, seed=7, bias_sigma=0.5)
    ds = _ds(s)
    for t in list(s.times[:2]) + [0.0, 1.0]:
        _, g, _ = gpu_deform(ds, float(t))
        err = _deform_err(s, g, float(t))
        assert err <= DEFORM_TOL, (variant, float(t), err)


def test_deform_range_and_batch_bit_identical():
    s = with_heads(make_scene("dnerf", n=9_001, n_frames=5), 0.3, seed=3)
    ds = _ds(s)
    t = float(s.times[2])
    _, full, _ = gpu_deform(ds, t)
    for (b, e) in ((0, 9001), (100, 4567), (4567, 9001), (63, 64)):
        _, part, _ = gpu_deform(ds, t, b, e)
        for k in full:
            assert np.array_equal(part[k][b:e], full[k][b:e]), (k, b, e)
            assert np.all(np.isnan(part[k][:b])) and np.all(np.isnan(part[k][e:]))
    outs, tens = ds.alloc_deformed(len(s.times))
    fgs.fgs_deform_batch(ds.g, ds.field, ds.mlp, [float(x) for x in s.times], outs)
    for f, tf in enumerate(s.times):
        _, single, _ = gpu_deform(ds, float(tf))
        for k in single:
            assert np.array_equal(tens[f][k].cpu().numpy(), single[k]), (f, k)


def test_zero_heads_identity_on_gpu():
    s = with_heads(make_scene("tiny"), 0.0)
    ds = _ds(s)
    _, g, _ = gpu_deform(ds, 0.37)
    assert np.array_equal(g["means"], s.means) and np.array_equal(g["quats"], s.quats)
    assert np.array_equal(g["log_scales"], s.log_scales)


def _render_parity(scene, frame=0, tiles_subset=None, check_tiles=True, max_instances=None):
    ds = _ds(scene)
    cam = scene.cameras[frame]
    dstruct, g, _ = gpu_deform(ds, float(scene.times[frame]))
    out = gpu_render_debug(ds, cam, dstruct, max_instances)
    assert out["status"] == fgs.FGS_OK
    ref = OR.render_ref(g, scene.opacity_logits, scene.sh, scene.sh_degree, cam, tiles_subset=tiles_subset)
    ints = compare_integer_work(out, ref["pre"], (ref["tiles"], ref["gids"], ref["ranges"]))
    assert out["M"] == len(ref["tiles"]) or ints["n_boundary"] > 0
    for k in ("radii", "rect", "tiles_touched", "depth_key"):
        assert ints[k] == 0, ints
    if check_tiles:
        assert ints["tile_lists"] == 0, ints
    pix = compare_pixels(out["image"], ref["image"], ref["flagged"])
    assert pix["psnr"] >= PSNR_MIN and pix["max_unflagged"] <= PIX_TOL, pix
    m = np.isfinite(ref["final_T"])
    assert np.max(np.abs(out["final_T"][m] - ref["final_T"][m])) <= PIX_TOL
    return out, ref, ints, pix


@pytest.mark.parametrize("W,H", [(64, 64), (70, 50), (33, 100)])
def test_render_tiny_matches_oracle(W, H):
    s = make_scene("tiny", width=W, height=H)
    _render_parity(s)


def test_render_tiny_stress_heads():
    _render_parity(with_heads(make_scene("tiny", width=72, height=56), 0.2, seed=11))


def test_render_low_opacity_bruteforce():
    """north_star: tiled == brute force over all Gaussians at opacity <= 0.017 (oracle side), GPU == both."""
    s = with_max_opacity(make_scene("tiny", n=800, width=48, height=40), 0.017)
    out, ref, _, _ = _render_parity(s)
    bf = OR.render_ref_bruteforce(oracle.deform_ref(s, float(s.times[0])), s.opacity_logits, s.sh, 0,
                                  s.cameras[0], rect_predicate=False)
    assert np.max(np.abs(out["image"] - bf["image"])) <= PIX_TOL


def test_render_dnerf_full_size_sampled():
    """D config at full size (100k, 800x800, SH 3): all integer work bit-exact (outside boundary
    Gaussians); pixels on 60 sampled tiles + the busiest tiles."""
    s = make_scene("dnerf", n_frames=2)
    rng = np.random.default_rng(0)
    tiles = sorted(set(rng.choice(2500, 50, replace=False).tolist()) | {1224, 1225, 1275})
    _render_parity(s, frame=1, tiles_subset=tiles)


def test_static_render_bit_identical_on_gpu():
    """north_star: zero heads -> fgs_render(fgs_deform(G, t)) == fgs_render(G) bit-exact."""
    s = with_heads(make_scene("tiny", width=80, height=72), 0.0)
    ds = _ds(s)
    dstruct, _, _ = gpu_deform(ds, 0.37)
    a = gpu_render_debug(ds, s.cameras[0], dstruct)
    b = gpu_render_debug(ds, s.cameras[0], ds.canonical_struct())
    assert np.array_equal(a["image"], b["image"])


def test_determinism_and_batch_equals_single():
    import torch
    s = make_scene("dnerf", n=30_000, width=256, height=200, n_frames=4)
    ds = _ds(s)
    outs, tens = ds.alloc_deformed(4)
    fgs.fgs_deform_batch(ds.g, ds.field, ds.mlp, ds.times, outs)
    ws = ds.alloc_workspace(4)
    imgs = [torch.empty((3, 200, 256), device="cuda") for _ in range(4)]
    fgs.fgs_render_batch(ds.cams, outs, imgs, ws)
    fgs.fgs_render_status(ws, 4)
    first = [im.cpu().numpy() for im in imgs]
    fgs.fgs_render_batch(ds.cams, outs, imgs, ws)
    for a, im in zip(first, imgs):
        assert np.array_equal(a, im.cpu().numpy())
    for f in range(4):
        ws1 = ds.alloc_workspace(1)
        im = torch.empty((3, 200, 256), device="cuda")
        fgs.fgs_render(ds.cams[f], outs[f], im, ws1)
        assert np.array_equal(im.cpu().numpy(), first[f])
    # fgs_frames (deform + render in one call) gives the same images
    scratch, _ = ds.alloc_deformed(4)
    imgs2 = [torch.empty((3, 200, 256), device="cuda") for _ in range(4)]
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, scratch, imgs2, ws)
    for a, im in zip(first, imgs2):
        assert np.array_equal(a, im.cpu().numpy())


def test_empty_and_single_gaussian():
    import torch
    s = make_scene("tiny", n=0, width=40, height=24)
    ds = _ds(s)
    img = torch.full((3, 24, 40), float("nan"), device="cuda")
    ws = ds.alloc_workspace(1)
    fgs.fgs_render(ds.cams[0], ds.canonical_struct(), img, ws)
    fgs.fgs_render_status(ws)
    assert torch.all(img == 0)
    s1 = make_scene("tiny", n=1, width=40, height=24)
    _render_parity(s1)


def test_capacity_overflow_reported():
    import torch
    s = make_scene("tiny")
    ds = _ds(s)
    ws = ds.alloc_workspace(1, max_instances=100)
    img = torch.empty((3, 64, 64), device="cuda")
    fgs.fgs_render(ds.cams[0], ds.canonical_struct(), img, ws)
    with pytest.raises(fgs.FgsError) as e:
        fgs.fgs_render_status(ws)
    assert e.value.code == fgs.FGS_E_CAPACITY


def test_nan_and_degenerate_gaussians_are_culled():
    s = with_heads(make_scene("tiny", n=300), 0.0)   # zero heads: the zero quaternions survive deform
    s.quats[:10] = 0.0            # zero quaternion -> NaN covariance -> culled
    s.means[10:20] = np.nan
    out, ref, _, _ = _render_parity(s, check_tiles=True)
    assert np.all(out["radii"][:20] == 0) and np.all(out["tiles_touched"][:20] == 0)


@pytest.mark.parametrize("cap", [1, 16, 100, 300, 700])
def test_long_list_sort_path_matches(cap):
    with fgs.tuning(fgs.FGS_TUNE_RADIX, 0):       # the per-tile sorts (the radix path is tested below)
        _long_list_sort_path_matches(cap)


def _long_list_sort_path_matches(cap):
    """Tile lists longer than the shared-memory sort cap go through long_sort_kernel (global-memory
    runs + merge-path merges): same lists, same image, bit for bit, as the in-smem bitonic path."""
    s = make_scene("tiny", width=70, height=50)
    ds = _ds(s)
    dstruct, _, _ = gpu_deform(ds, float(s.times[0]))
    base = gpu_render_debug(ds, s.cameras[0], dstruct)
    old = fgs.fgs_get_tuning(fgs.FGS_TUNE_TILE_SORT_CAP)
    fgs.fgs_set_tuning(fgs.FGS_TUNE_TILE_SORT_CAP, cap)
    try:
        out = gpu_render_debug(ds, s.cameras[0], dstruct)
        _render_parity(s)
    finally:
        fgs.fgs_set_tuning(fgs.FGS_TUNE_TILE_SORT_CAP, old)
    lengths = np.diff(base["ranges"], axis=1)
    assert lengths.max() > cap
    for k in ("image", "sorted_gid", "sorted_tile", "ranges", "final_T", "n_contrib"):
        assert np.array_equal(out[k], base[k]), k


@pytest.mark.parametrize("cap,radix", [(None, 0), (100, 0), (None, 2)])
def test_sort_exact_and_near_depth_ties(cap, radix):
    """The tile sort's 32-bit prefix words (depth key relative to the list minimum, shifted right when
    the list's depth range does not fit beside the slot index): groups of Gaussians at bit-identical
    depths (exact ties, ordered by index) and Gaussians along view rays from depth 0.5 to 500 (wide
    ranges: shifted prefixes, near ties resolved on the full key) give the oracle's (tile, depth,
    index) lists bit for bit, through the warp sorts, (cap 100) the long-list sort and (radix 2) the radix
    binning path (stable depth sort: exact ties keep index order)."""
    s = with_heads(make_scene("tiny", n=3000, width=64, height=64), 0.0)   # zero heads: means as given
    rng = np.random.default_rng(7)
    i = 0
    for k in range(40):                       # 40 groups of 2..41 copies of one mean
        m = 2 + k
        s.means[i:i + m] = s.means[rng.integers(i + m, s.n)]
        i += m
    cam = s.cameras[0]
    idx = np.arange(2000, 2400)
    z = np.geomspace(0.5, 500.0, idx.size)
    u = rng.uniform(-0.4, 0.4, (idx.size, 2))
    pc = np.stack([u[:, 0] * z, u[:, 1] * z, z], 1)
    s.means[idx] = ((pc - cam.t.astype(np.float64)) @ cam.R.astype(np.float64)).astype(np.float32)
    old = fgs.fgs_get_tuning(fgs.FGS_TUNE_TILE_SORT_CAP)
    if cap is not None:
        fgs.fgs_set_tuning(fgs.FGS_TUNE_TILE_SORT_CAP, cap)
    try:
        with fgs.tuning(fgs.FGS_TUNE_RADIX, radix):
            out, ref, _, _ = _render_parity(s, check_tiles=True)
    finally:
        fgs.fgs_set_tuning(fgs.FGS_TUNE_TILE_SORT_CAP, old)
    tiles, gids = np.asarray(ref["tiles"]), np.asarray(ref["gids"])
    dk = np.asarray(ref["pre"]["depth_key"]).astype(np.int64)[gids]
    same = tiles[1:] == tiles[:-1]
    assert np.any(same & (dk[1:] == dk[:-1])), "no exact depth ties in the lists"
    starts = np.flatnonzero(np.r_[True, ~same])
    spans = np.maximum.reduceat(dk, starts) - np.minimum.reduceat(dk, starts)
    assert spans.max() >= 1 << 25, "no list with a depth range wider than the prefix bits"


@pytest.mark.parametrize("ties,radix", [(False, 0), (True, 0), (False, 2), (True, 2)])
def test_long_lists_multi_run_merge(ties, radix):
    """A list longer than several 2048-entry runs (merge passes) sorted in global memory: many
    Gaussians piled on one tile (segments of 4096 on the 32-bit prefix-word CTA sort); with ties,
    groups of bit-identical depths inside those segments (the word sort's tie fixup).  radix 2: the
    same lists through the radix binning path."""
    s = make_scene("tiny", n=9000, width=32, height=32)
    if ties:
        s = with_heads(s, 0.0)
        rng = np.random.default_rng(5)
        for k in range(60):
            s.means[100 * k:100 * k + 2 + k] = s.means[rng.integers(6100, s.n)]
    ds = _ds(s)
    dstruct, g, _ = gpu_deform(ds, float(s.times[0]))
    with fgs.tuning(fgs.FGS_TUNE_RADIX, radix):
        out = gpu_render_debug(ds, s.cameras[0], dstruct)
    assert np.diff(out["ranges"], axis=1).max() > 4096
    ref = OR.render_ref(g, s.opacity_logits, s.sh, s.sh_degree, s.cameras[0])
    ints = compare_integer_work(out, ref["pre"], (ref["tiles"], ref["gids"], ref["ranges"]))
    assert ints["tile_lists"] == 0 and ints["rect"] == 0, ints
    pix = compare_pixels(out["image"], ref["image"], ref["flagged"])
    assert pix["psnr"] >= PSNR_MIN and pix["max_unflagged"] <= PIX_TOL, pix


@pytest.mark.parametrize("case", ["smem", "global", "skewed"])
def test_long_sort_bucket_pass_paths(case):
    """The long-list sort's bucket pass (FGS_TUNE_LONG_SORT = 1, the default) against the networks +
    merges (0) and the oracle's (tile, depth, index) lists, on each of its paths, asserted through
    fgs_render_aux.long_sort_paths: scratch in shared memory (lists of 1025..8192), in the inst2 scratch
    (lists over 8192), and the fallback to the networks when a bucket holds more than 64 instances
    (hundreds of Gaussians at one bit-identical depth: exact ties, ordered by index)."""
    W = 16 if case == "global" else 32                          # one 16x16 tile: every kept Gaussian in one list
    s = make_scene("tiny", n={"smem": 3000, "global": 9500, "skewed": 3000}[case], width=W, height=W)
    if case == "skewed":
        s = with_heads(s, 0.0)                                  # zero heads: means as given
        s.means[:400] = s.means[1000]
    ds = _ds(s)
    dstruct, g, _ = gpu_deform(ds, float(s.times[0]))
    res = {}
    for mode in (1, 0):
        with fgs.tuning(fgs.FGS_TUNE_LONG_SORT, mode):
            res[mode] = gpu_render_debug(ds, s.cameras[0], dstruct)
    lengths = np.diff(res[1]["ranges"], axis=1)
    paths = res[1]["long_sort_paths"].tolist()
    assert lengths.max() > 1024
    if case == "smem":
        assert lengths.max() <= 8192 and paths[0] > 0 and paths[2] == 0, paths
    elif case == "global":
        assert lengths.max() > 8192 and paths[1] > 0 and paths[2] == 0, paths
    else:
        assert paths[2] > 0, paths
    assert res[0]["long_sort_paths"].tolist()[:2] == [0, 0]
    for k in ("sorted_gid", "sorted_tile", "ranges", "image", "final_T", "n_contrib"):
        assert np.array_equal(res[0][k], res[1][k]), k
    ref = OR.render_ref(g, s.opacity_logits, s.sh, s.sh_degree, s.cameras[0])
    ints = compare_integer_work(res[1], ref["pre"], (ref["tiles"], ref["gids"], ref["ranges"]))
    assert ints["tile_lists"] == 0 and ints["rect"] == 0, ints


@pytest.mark.parametrize("case", ["n200", "n600", "n1000", "ties"])
def test_warp_bucket_sort_matches_networks(case):
    """Warp-sorted lists of 129..1024 instances take one bucket pass (512 depth buckets, rank within the
    bucket) when FGS_TUNE_LONG_SORT = 1 (the default) and the register networks + merge when it is 0; a
    list with a bucket of more than 32 instances (here 300 Gaussians at one bit-identical depth: exact
    ties, ordered by index) falls back to the networks.  One 16x16 tile holds every kept Gaussian; both
    modes give the oracle's (tile, depth, index) list and identical images."""
    n = {"n200": 200, "n600": 600, "n1000": 1000, "ties": 800}[case]
    s = make_scene("tiny", n=n, width=16, height=16)
    if case == "ties":
        s = with_heads(s, 0.0)                                  # zero heads: means as given
        s.means[:300] = s.means[500]
    ds = _ds(s)
    dstruct, g, _ = gpu_deform(ds, float(s.times[0]))
    res = {}
    for mode in (1, 0):
        with fgs.tuning(fgs.FGS_TUNE_LONG_SORT, mode):
            res[mode] = gpu_render_debug(ds, s.cameras[0], dstruct)
    L = int(np.diff(res[1]["ranges"], axis=1).max())
    assert 128 < L <= 1024, L
    for k in ("sorted_gid", "sorted_tile", "ranges", "image", "final_T", "n_contrib"):
        assert np.array_equal(res[0][k], res[1][k]), k
    ref = OR.render_ref(g, s.opacity_logits, s.sh, s.sh_degree, s.cameras[0])
    ints = compare_integer_work(res[1], ref["pre"], (ref["tiles"], ref["gids"], ref["ranges"]))
    assert ints["tile_lists"] == 0 and ints["rect"] == 0, ints


def test_sharded_frames_single_rank_equals_fgs_frames():
    """(e2) pipeline (sharding.sharded_frames) at world size 1: deform via fgs_deform_range into the
    gather buffers + render per time gives the same images as fgs_frames."""
    import torch
    from paper_2310_08528_b200.sharding import ShardedDeform, sharded_frames
    s = make_scene("dnerf", n=20_000, width=128, height=96, n_frames=3)
    ds = _ds(s)
    sd = ShardedDeform(s.n, 1, 0, "cuda", n_slots=2)
    imgs = [torch.empty((3, 96, 128), device="cuda") for _ in range(3)]
    ws = ds.alloc_workspace(1)
    views = [[(ds.cams[k], k)] for k in range(3)]
    sharded_frames(ds, sd, ds.times, views, imgs, ws)
    scratch, _ = ds.alloc_deformed(3)
    ref = [torch.empty((3, 96, 128), device="cuda") for _ in range(3)]
    ws3 = ds.alloc_workspace(3)
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, scratch, ref, ws3)
    torch.cuda.synchronize()
    for a, b in zip(imgs, ref):
        assert torch.equal(a, b)


def _flat_deformed(ds, rows):
    """One flat [rows x 10] fp32 buffer holding quats | means | log_scales back to back (the layout of
    ShardedDeform's symmetric buffers): returns (flat, struct, views)."""
    import torch
    flat = torch.full((rows * 10,), float("nan"), dtype=torch.float32, device="cuda")
    q, m, ls = flat[:rows * 4].view(rows, 4), flat[rows * 4:rows * 7].view(rows, 3), flat[rows * 7:].view(rows, 3)
    return flat, ds.deformed_struct(m, ls, q), {"means": m, "log_scales": ls, "quats": q}


@pytest.mark.parametrize("n_peers", [1, 2, 3])
def test_deform_range_peers_writes_every_replica(n_peers):
    """§8(e2) fused deform + gather on one GPU: fgs_deform_range_peers stores rows [begin, end) into
    every replica (here other local buffers at the given byte offsets) — each replica equals
    fgs_deform_range's rows bit for bit and the rows outside the range stay untouched."""
    import torch
    s = make_scene("dnerf", n=20_011, width=64, height=64, n_frames=1)
    ds = _ds(s)
    t = float(s.times[0])
    n, lo, hi = s.n, 3_001, 17_777
    bufs = [_flat_deformed(ds, n) for _ in range(n_peers)]
    offs = [bufs[q][0].data_ptr() - bufs[0][0].data_ptr() for q in range(n_peers)]
    fgs.fgs_deform_range_peers(ds.g, ds.field, ds.mlp, t, lo, hi, bufs[0][1], offs)
    ref_flat, ref_struct, ref = _flat_deformed(ds, n)
    fgs.fgs_deform_range(ds.g, ds.field, ds.mlp, t, lo, hi, ref_struct)
    torch.cuda.synchronize()
    for flat, _, views in bufs:
        for k in ("means", "log_scales", "quats"):
            assert torch.equal(views[k][lo:hi], ref[k][lo:hi]), k
            assert torch.isnan(views[k][:lo]).all() and torch.isnan(views[k][hi:]).all(), k


def test_deform_range_peers_rejects_bad_arguments():
    s = make_scene("tiny")
    ds = _ds(s)
    _, st, _ = _flat_deformed(ds, s.n)
    for offs in ([], [0] * 9, [0, 2]):
        with pytest.raises(fgs.FgsError):
            fgs.fgs_deform_range_peers(ds.g, ds.field, ds.mlp, 0.5, 0, s.n, st, offs)


def test_sharded_frames_fused_world1_equals_fgs_frames():
    """(e2) fused mode: symmetric-memory gather buffers, the deform epilogue writes every rank's copy
    (fgs_deform_range_peers), a stream-ordered barrier replaces the all-gather — at world size 1 (a
    one-rank NCCL group) the images equal fgs_frames bit for bit."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2310_08528_b200.sharding import ShardedDeform, sharded_frames
    assert not dist.is_initialized()
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        s = make_scene("dnerf", n=20_000, width=128, height=96, n_frames=3)
        ds = _ds(s)
        sd = ShardedDeform(s.n, 1, 0, "cuda", n_slots=2, fused=True)
        assert sd.offsets[0] == [0]
        imgs = [torch.empty((3, 96, 128), device="cuda") for _ in range(3)]
        ws = ds.alloc_workspace(1)
        views = [[(ds.cams[k], k)] for k in range(3)]
        sharded_frames(ds, sd, ds.times, views, imgs, ws)
        scratch, _ = ds.alloc_deformed(3)
        ref = [torch.empty((3, 96, 128), device="cuda") for _ in range(3)]
        ws3 = ds.alloc_workspace(3)
        fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, scratch, ref, ws3)
        torch.cuda.synchronize()
        for a, b in zip(imgs, ref):
            assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


def test_frames_sharing_a_time_share_the_deformation():
    """fgs_frames deforms each distinct t once; frames at the same t (views of one instant) render
    from it — images equal the per-frame deform + render path bit for bit."""
    import torch
    s = make_scene("dnerf", n=20_000, width=160, height=120, n_frames=3)
    ds = _ds(s)
    ts = [float(s.times[1]), float(s.times[1]), float(s.times[2])]
    scratch, _ = ds.alloc_deformed(3)
    imgs = [torch.empty((3, 120, 160), device="cuda") for _ in range(3)]
    ws = ds.alloc_workspace(3)
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ts, ds.cams, scratch, imgs, ws)
    for f in range(3):
        d, _, _ = gpu_deform(ds, ts[f])
        ws1 = ds.alloc_workspace(1)
        im = torch.empty((3, 120, 160), device="cuda")
        fgs.fgs_render(ds.cams[f], d, im, ws1)
        assert torch.equal(im, imgs[f]), f


def test_composition_of_two_models():
    """two 4D-GS models with their own fields and MLPs are deformed into
    row ranges of ONE G' (fgs_deformed row views) and rendered together; equals the oracle render of
    the merged set (deform per model by the oracle, then one render)."""
    import torch
    a = make_scene("tiny", n=1203, seed=10, width=72, height=56)
    b = make_scene("tiny", n=801, seed=11, width=72, height=56)
    b.means[:] = (b.means * 0.5 + np.float32(0.3)).astype(np.float32)   # a second object, inside A's box
    dA, dB = _ds(a), _ds(b)
    N = a.n + b.n
    X = torch.empty((N, 3), device="cuda"); S = torch.empty((N, 3), device="cuda")
    Q = torch.empty((N, 4), device="cuda")
    op = torch.cat([dA.opacity_logits, dB.opacity_logits]).contiguous()
    sh = torch.cat([dA.sh, dB.sh]).contiguous()
    whole = fgs.fgs_deformed(N, 0, X.data_ptr(), S.data_ptr(), Q.data_ptr(), op.data_ptr(), sh.data_ptr())
    t = 0.61
    fgs.fgs_deform(dA.g, dA.field, dA.mlp, t, fgs.deformed_rows(whole, 0, a.n, op.data_ptr(), sh.data_ptr()))
    fgs.fgs_deform(dB.g, dB.field, dB.mlp, t, fgs.deformed_rows(whole, a.n, b.n, op.data_ptr(), sh.data_ptr()))
    torch.cuda.synchronize()
    g = {"means": X.cpu().numpy(), "log_scales": S.cpu().numpy(), "quats": Q.cpu().numpy()}
    ra, rb = oracle.deform_ref(a, t), oracle.deform_ref(b, t)
    for k in g:
        ref = np.concatenate([ra[k], rb[k]])
        assert np.abs(g[k].astype(np.float64) - ref).max() <= DEFORM_TOL, k
    cam = a.cameras[0]
    ws = dA.alloc_workspace(1, 16 * N)
    img = torch.empty((3, 56, 72), device="cuda")
    fgs.fgs_render(fgs.make_camera(cam), whole, img, ws)
    fgs.fgs_render_status(ws)
    opn = np.concatenate([a.opacity_logits, b.opacity_logits]); shn = np.concatenate([a.sh, b.sh])
    ref = OR.render_ref(g, opn, shn, 0, cam)
    pix = compare_pixels(img.cpu().numpy(), ref["image"], ref["flagged"])
    assert pix["psnr"] >= PSNR_MIN and pix["max_unflagged"] <= PIX_TOL, pix


@pytest.mark.parametrize("heads", ["both", "colour", "opacity"])
def test_colour_opacity_decoders(heads):
    """P:1232 variant: phi_C / phi_alpha deform the SH coefficients and the opacity logit per frame;
    deformed SH / opacity match the oracle (<= 1e-4), and the render of the deformed set matches the
    oracle render of the GPU's fp32 G' (pixels, integer work); fgs_frames gives the same images."""
    import torch
    from paper_2310_08528_b200.inputs import with_colour_heads
    s = make_scene("dnerf", n=12_007, width=120, height=96, n_frames=3)
    s = with_heads(s, 0.5, seed=2, bias_sigma=0.1)
    s = with_colour_heads(s, 0.2, 0.3, seed=3, colour=heads in ("both", "colour"),
                          opacity=heads in ("both", "opacity"))
    ds = _ds(s)
    t = float(s.times[1])
    dstruct, g, _ = gpu_deform(ds, t)
    ref = oracle.deform_ref(s, t)
    assert set(ref) == set(g)
    for k in ref:
        assert np.abs(g[k].astype(np.float64) - ref[k]).max() <= DEFORM_TOL, k
    cam = s.cameras[1]
    out = gpu_render_debug(ds, cam, dstruct)
    opac = g.get("opacity_logits", s.opacity_logits)
    sh = g.get("sh", s.sh)
    oref = OR.render_ref(g, opac, sh, s.sh_degree, cam)
    ints = compare_integer_work(out, oref["pre"], (oref["tiles"], oref["gids"], oref["ranges"]))
    assert ints["rect"] == 0 and ints["tile_lists"] == 0, ints
    pix = compare_pixels(out["image"], oref["image"], oref["flagged"])
    assert pix["psnr"] >= PSNR_MIN and pix["max_unflagged"] <= PIX_TOL, pix
    # whole frames through fgs_frames == per-frame deform + render
    scratch, _ = ds.alloc_deformed(3)
    imgs = [torch.empty((3, 96, 120), device="cuda") for _ in range(3)]
    ws = ds.alloc_workspace(3)
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, scratch, imgs, ws)
    assert np.array_equal(imgs[1].cpu().numpy(), out["image"])


def test_colour_decoder_rejects_canonical_alias():
    from paper_2310_08528_b200.inputs import with_colour_heads
    s = with_colour_heads(make_scene("tiny", n=500), 0.1, 0.1)
    ds = _ds(s)
    outs, tens = ds.alloc_deformed(1)
    bad = ds.deformed_struct(tens[0]["means"], tens[0]["log_scales"], tens[0]["quats"])   # canonical SH
    with pytest.raises(fgs.FgsError) as e:
        fgs.fgs_deform(ds.g, ds.field, ds.mlp, 0.5, bad)
    assert e.value.code == fgs.FGS_E_INVALID


@pytest.mark.parametrize("deg", [1, 2])
def test_sh_degrees_1_and_2(deg):
    """preprocess_kernel<1>/<2> (the configs use degrees 0 and 3): SH truncated to degree `deg`."""
    from dataclasses import replace
    s = make_scene("dnerf", n=6_000, width=96, height=80, n_frames=1)
    K = (deg + 1) ** 2
    s = replace(s, sh=np.ascontiguousarray(s.sh[:, :K, :]), sh_degree=deg)
    _render_parity(s)


def test_screen_covering_and_near_plane_gaussians():
    """Edge geometry: a few huge Gaussians whose rects cover every tile (long lists; the 13x10-tile image
    keeps the CTA aggregation box far below its 4096-tile limit — the direct-atomics path is forced in
    test_binning_direct_atomics_path), Gaussians straddling and behind the near plane, t at 0 and 1."""
    from dataclasses import replace
    s = make_scene("tiny", n=1500, width=200, height=150)
    ls = s.log_scales.copy()
    ls[:6] = np.float32(0.5)                          # ~1.6 world units: covers the whole image
    means = s.means.copy()
    eye_z = 4.0                                       # tiny camera at (0,0,4) looking at the origin
    means[6:12, 2] = np.float32(eye_z - 0.2)          # at the near plane (z_cam ~ 0.2)
    means[12:18, 2] = np.float32(eye_z + 0.5)         # behind the camera
    s = replace(s, log_scales=ls, means=means)
    s = with_heads(s, 0.0)
    for t in (0.0, 1.0):
        s.times[0] = np.float32(t)
        _render_parity(s)


@pytest.mark.parametrize("variant", ["tiny", "dnerf_stress", "hyper"])
def test_deform_widths_and_times_match_oracle(variant):
    """The deformation kernel against the oracle at phi_d widths 32/64/128, incl. the 3xTF32 stress
    heads, ragged tails and t at both ends of [0, 1]."""
    if variant == "tiny":
        s = make_scene("tiny", n=2011)
    elif variant == "dnerf_stress":
        s = with_heads(make_scene("dnerf", n=7_777, n_frames=2), 1.0, seed=7, bias_sigma=0.5)
    else:
        s = make_scene("hypernerf", n=3_001, n_frames=2)
    ds = _ds(s)
    for t in (0.0, float(s.times[0]), 1.0):
        _, g, _ = gpu_deform(ds, t)
        assert _deform_err(s, g, t) <= DEFORM_TOL, (variant, t)


def test_deform_l2_fallback_bit_identical_to_staged_lines():
    """tc3 stages the time lines of a group's knot windows in shared memory; a group whose windows do not
    fit (a model in draw order, not spatially sorted) reads the temporal planes from L2 instead.  Both
    paths compute the same operations in the same order: the same Gaussians give bit-identical G'."""
    from paper_2310_08528_b200.inputs import morton_order
    sd = make_scene("dnerf", n=20_000, n_frames=2, order="draw")       # L2 path (windows span the axes)
    sm = make_scene("dnerf", n=20_000, n_frames=2)                     # staged path (Morton order)
    perm = morton_order(sd.means, sd.field.bmin, sd.field.bmax)
    t = float(sd.times[1])
    _, gd, _ = gpu_deform(_ds(sd), t)
    _, gm, _ = gpu_deform(_ds(sm), t)
    assert _deform_err(sd, gd, t) <= DEFORM_TOL
    for k in gd:
        assert np.array_equal(gd[k][perm], gm[k]), k


@pytest.mark.parametrize("heads", [False, True])
def test_frames_host_equals_device_path(heads, F=9, n=15_000):
    """fgs_frames_host (host model in, host images out; copies overlapped with rendering on a side
    stream) gives the device path's images bit for bit, with and without the P:1232 decoders."""
    import torch
    from paper_2310_08528_b200.inputs import with_colour_heads
    s = make_scene("dnerf", n=n, width=144, height=112, n_frames=F)
    if heads:
        s = with_colour_heads(s, 0.1, 0.2)
    ds = _ds(s)
    scratch, _ = ds.alloc_deformed(F)
    imgs = [torch.empty((3, 112, 144), device="cuda") for _ in range(F)]
    ws = ds.alloc_workspace(F)
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, scratch, imgs, ws)
    hs = fgs.HostScene(s)
    himgs = [torch.full((3, 112, 144), float("nan")).pin_memory() for _ in range(F)]
    nbytes = fgs.fgs_frames_host_workspace_bytes(hs.g, hs.field, hs.mlp, F, 144, 112, 16 * s.n)
    dws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, himgs, dws)
    torch.cuda.synchronize()
    for a, b in zip(imgs, himgs):
        assert torch.equal(a.cpu(), b)


def test_frames_host_ragged_model():
    """The host path on a model spanning more than two Gaussian tiles per SM with a ragged last tile
    (n = 60,001): same images as the device path bit for bit."""
    test_frames_host_equals_device_path(False, F=5, n=60_001)


def test_frames_host_long_batch():
    """The host path over a batch longer than one render launch (37 frames: chunks 1, 2, 4, 4, ...
    across the 32-frame launch limit) equals the device path bit for bit."""
    test_frames_host_equals_device_path(False, F=37)


def test_frames_cuda_graph_capture_and_replay():
    """fgs_frames is capturable into a CUDA graph (no host synchronisation, no allocation on the path);
    replaying the graph reproduces the eager images bit for bit."""
    import torch
    s = make_scene("dnerf", n=20_000, width=128, height=96, n_frames=4)
    ds = _ds(s)
    scratch, _ = ds.alloc_deformed(4)
    ws = ds.alloc_workspace(4)
    eager = [torch.empty((3, 96, 128), device="cuda") for _ in range(4)]
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, scratch, eager, ws)
    torch.cuda.synchronize()
    imgs = [torch.full((3, 96, 128), float("nan"), device="cuda") for _ in range(4)]
    stream = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, scratch, imgs, ws)   # warm-up on stream
        stream.synchronize()
        for im in imgs:
            im.fill_(float("nan"))
        with torch.cuda.graph(graph, stream=stream):
            fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, scratch, imgs, ws,
                           stream=torch.cuda.current_stream())
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, imgs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("W,H", [(1, 1), (17, 1), (1, 33), (16, 16), (31, 47)])
def test_degenerate_image_sizes(W, H):
    """Images smaller than a tile or one pixel wide/high: partial tiles everywhere."""
    s = make_scene("tiny", n=700, width=W, height=H)
    _render_parity(s)


def test_gpu_image_invariant_to_array_order():
    """S:147 on the GPU: permuting the Gaussian array (all depths distinct) leaves the image unchanged —
    the per-tile (depth, index) sort, not the storage order, decides the compositing order."""
    from dataclasses import replace
    import torch
    s = with_heads(make_scene("dnerf", n=8_000, width=96, height=80, n_frames=1), 0.0)
    perm = np.random.default_rng(5).permutation(s.n)
    sp = replace(s, means=s.means[perm], log_scales=s.log_scales[perm], quats=s.quats[perm],
                 opacity_logits=s.opacity_logits[perm], sh=s.sh[perm])
    ds = _ds(s)
    a = gpu_render_debug(ds, s.cameras[0], ds.canonical_struct())
    dsp = _ds(sp)
    b = gpu_render_debug(dsp, sp.cameras[0], dsp.canonical_struct())
    # Gaussians sharing an fp32 depth key are ordered by index, which the permutation changes: tiles they
    # touch are compared within the pixel tolerance, every other pixel bit for bit
    kept = a["tiles_touched"] > 0
    keys, counts = np.unique(a["depth_key"][kept], return_counts=True)
    tied = np.isin(a["depth_key"], keys[counts > 1]) & kept
    mask = np.zeros(a["image"].shape[1:], bool)
    for x0, y0, x1, y1 in a["rect"][tied]:
        mask[16 * y0:16 * y1, 16 * x0:16 * x1] = True
    assert np.array_equal(a["image"][:, ~mask], b["image"][:, ~mask])
    assert np.abs(a["image"] - b["image"]).max() <= PIX_TOL


def test_batches_longer_than_one_launch():
    """More frames than one launch's frame table (kMaxFrames = 32): fgs_frames / fgs_deform_batch split
    the batch; every frame equals its single-frame deform + render."""
    import torch
    s = make_scene("dnerf", n=6_000, width=64, height=48, n_frames=35)
    ds = _ds(s)
    scratch, _ = ds.alloc_deformed(35)
    imgs = [torch.empty((3, 48, 64), device="cuda") for _ in range(35)]
    ws = ds.alloc_workspace(35)
    fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, scratch, imgs, ws)
    fgs.fgs_render_status(ws, 35)
    for f in (0, 31, 32, 34):
        d, _, _ = gpu_deform(ds, float(s.times[f]))
        ws1 = ds.alloc_workspace(1)
        im = torch.empty((3, 48, 64), device="cuda")
        fgs.fgs_render(ds.cams[f], d, im, ws1)
        assert torch.equal(im, imgs[f]), f


@pytest.mark.parametrize("limit", [1, 64])
def test_binning_direct_atomics_path(limit):
    """The direct-global-atomics fallback of the per-tile counting and the key duplication (taken when a
    CTA's rect union exceeds the shared aggregation box): forced by lowering FGS_TUNE_AGG_TILES, the
    debug counter proves every preprocess / duplicate CTA with kept Gaussians took it (limit 1) or some
    did (limit 64), and the integer work and image stay at parity (bit-identical to the aggregated run)."""
    s = make_scene("tiny", n=1500, width=200, height=150)
    ls = s.log_scales.copy()
    ls[:6] = np.float32(0.5)                          # screen-covering rects: unions of the whole grid
    from dataclasses import replace
    s = replace(s, log_scales=ls)
    ds = _ds(s)
    dstruct, _, _ = gpu_deform(ds, float(s.times[0]))
    base = gpu_render_debug(ds, s.cameras[0], dstruct)
    assert base["binning_direct"].tolist() == [0, 0]
    with fgs.tuning(fgs.FGS_TUNE_AGG_TILES, limit):
        out, ref, ints, pix = _render_parity(s)
        forced = gpu_render_debug(ds, s.cameras[0], dstruct)
    n_cta = (s.n + 255) // 256
    if limit == 1:
        assert forced["binning_direct"].tolist() == [n_cta, n_cta]
    else:
        assert 0 < forced["binning_direct"][0] and 0 < forced["binning_direct"][1]
    for k in ("image", "final_T", "n_contrib", "sorted_gid", "ranges", "radii", "rect"):
        assert np.array_equal(forced[k], base[k]), k


def test_blend_cull_knob_is_result_neutral_tiny():
    """FGS_TUNE_BLEND_CULL = 0 evaluates every list entry on every live pixel (the unculled Eq. 4 loop);
    image, final T and contributor counts are bit-identical to the culled blend (ragged tiny frames,
    stress heads)."""
    for s in (make_scene("tiny", width=70, height=50), with_heads(make_scene("tiny", width=72, height=56), 0.2, seed=11)):
        ds = _ds(s)
        dstruct, _, _ = gpu_deform(ds, float(s.times[0]))
        on = gpu_render_debug(ds, s.cameras[0], dstruct)
        with fgs.tuning(fgs.FGS_TUNE_BLEND_CULL, 0):
            off = gpu_render_debug(ds, s.cameras[0], dstruct)
        for k in ("image", "final_T", "n_contrib"):
            assert np.array_equal(on[k], off[k]), k
        assert off["blend_work"][0] >= on["blend_work"][0]


def test_frames_host_status_reports_overflow():
    """fgs_frames_host's renders live inside its device workspace: fgs_frames_host_status finds an
    instance-capacity overflow there (FGS_E_CAPACITY) and reports FGS_OK for a workspace that fits."""
    import torch
    s = make_scene("dnerf", n=15_000, width=144, height=112, n_frames=3)
    hs = fgs.HostScene(s)
    himgs = [torch.empty((3, 112, 144)).pin_memory() for _ in range(3)]
    for cap, ok in ((16 * s.n, True), (1000, False)):
        nbytes = fgs.fgs_frames_host_workspace_bytes(hs.g, hs.field, hs.mlp, 3, 144, 112, cap)
        dws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, himgs, dws)
        if ok:
            fgs.fgs_frames_host_status(hs.g, hs.field, hs.mlp, hs.cams, dws)
        else:
            with pytest.raises(fgs.FgsError) as e:
                fgs.fgs_frames_host_status(hs.g, hs.field, hs.mlp, hs.cams, dws)
            assert e.value.code == fgs.FGS_E_CAPACITY


def test_frames_host_concurrent_threads():
    """fgs_frames_host is reentrant: four host threads, each with its own stream, workspace and host
    images, enqueue concurrently (each call holds its own copy stream / events); every result equals
    the serial one bit for bit."""
    import threading
    import torch
    s = make_scene("dnerf", n=15_000, width=144, height=112, n_frames=5)
    hs = fgs.HostScene(s)
    nbytes = fgs.fgs_frames_host_workspace_bytes(hs.g, hs.field, hs.mlp, 5, 144, 112, 16 * s.n)
    ref = [torch.empty((3, 112, 144)).pin_memory() for _ in range(5)]
    dws0 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, ref, dws0)
    torch.cuda.synchronize()
    K = 4
    outs = [[torch.full((3, 112, 144), float("nan")).pin_memory() for _ in range(5)] for _ in range(K)]
    wss = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(K)]
    streams = [torch.cuda.Stream() for _ in range(K)]
    errs = []

    def work(k):
        try:
            torch.cuda.set_device(0)
            for _ in range(3):
                fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, outs[k], wss[k], stream=streams[k])
            streams[k].synchronize()
        except Exception as e:   # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k in range(K):
        for a, b in zip(ref, outs[k]):
            assert torch.equal(a, b), k


@pytest.mark.parametrize("case", ["tiny", "dnerf", "elongated"])
def test_tile_cull_keeps_every_contributor(case):
    """FGS_TUNE_TILE_CULL = 1 leaves a Gaussian out of a tile's list only where it cannot contribute: the
    image, final T and contributor counts equal the unculled render bit for bit; every tile's list is an
    order-preserving subsequence of the [3dgs] list (which the oracle's lists pin with the knob off); and
    each (tile, Gaussian) pair left out has, by the fp64 oracle's conic, mean and opacity (Eq. 1 / Eq. 4,
    P:694), alpha < 1/255 at every pixel of the tile.  tiles_touched and n_instances count what
    remains, and something is in fact removed."""
    if case == "tiny":
        s = make_scene("tiny", n=3000, width=150, height=106)
    elif case == "dnerf":
        s = make_scene("dnerf", n=25_000, width=208, height=160)
    else:                                # long thin Gaussians: big rects, few tiles reached
        s = with_heads(make_scene("tiny", n=1500, width=160, height=128), 0.0)
        s.log_scales[:, 0] += 1.6
        s.log_scales[:, 1:] -= 1.2
    ds = _ds(s)
    cam = s.cameras[0]
    dstruct, g, _ = gpu_deform(ds, float(s.times[0]))
    cap = 80 * s.n if case == "elongated" else None      # 80 tiles: every Gaussian on every tile fits
    off = gpu_render_debug(ds, cam, dstruct, cap)
    with fgs.tuning(fgs.FGS_TUNE_TILE_CULL, 1):
        on = gpu_render_debug(ds, cam, dstruct, cap)
    assert off["status"] == fgs.FGS_OK and on["status"] == fgs.FGS_OK
    for k in ("image", "final_T", "n_contrib", "radii", "rect", "depth_key"):
        assert np.array_equal(off[k], on[k]), k
    assert on["M"] < off["M"] and on["M"] == int(on["tiles_touched"].sum())
    assert np.all(on["tiles_touched"] <= off["tiles_touched"])
    pre = OR.preprocess_ref(g["means"], g["log_scales"], g["quats"], s.opacity_logits, s.sh, s.sh_degree, cam)
    gx = (cam.width + 15) // 16
    n_dropped = 0
    worst = 0.0
    for tile in range(off["ranges"].shape[0]):
        a = off["sorted_gid"][off["ranges"][tile, 0]:off["ranges"][tile, 1]]
        b = on["sorted_gid"][on["ranges"][tile, 0]:on["ranges"][tile, 1]]
        pos = {int(gid): k for k, gid in enumerate(a)}
        idx = [pos.get(int(gid), -1) for gid in b]
        assert all(i >= 0 for i in idx) and all(x < y for x, y in zip(idx, idx[1:])), tile
        dropped = np.setdiff1d(a, b)
        if len(dropped) == 0:
            continue
        n_dropped += len(dropped)
        tx, ty = tile % gx, tile // gx
        px, py = np.meshgrid(np.arange(16 * tx, min(16 * tx + 16, cam.width), dtype=np.float64),
                             np.arange(16 * ty, min(16 * ty + 16, cam.height), dtype=np.float64))
        for gid in dropped:
            dx, dy = pre["mean2d"][gid, 0] - px, pre["mean2d"][gid, 1] - py
            A, B, C = pre["conic"][gid]
            alpha = pre["opacity"][gid] * np.exp(-0.5 * (A * dx * dx + C * dy * dy) - B * dx * dy)
            worst = max(worst, float(alpha.max()))
    assert n_dropped == off["M"] - on["M"]
    assert worst < 1.0 / 255.0, worst


def test_frames_host_two_calls_in_flight():
    """bench.py's pipelined e2e: one host thread keeps two fgs_frames_host calls in flight on two
    streams (each lane its own workspace and pinned images; the SH upload and the image downloads ride
    separate side streams), eight steps alternating two different batches of times.  Every lane ends
    with the images of its last batch, bit-equal to the one-call-at-a-time result."""
    import dataclasses
    import numpy as np
    import torch
    F = 6
    s0 = make_scene("dnerf", n=40_000, width=208, height=160, n_frames=F)
    s1 = dataclasses.replace(s0, times=np.asarray(s0.times[::-1], np.float32).copy())
    hs = [fgs.HostScene(s0), fgs.HostScene(s1)]
    nbytes = fgs.fgs_frames_host_workspace_bytes(hs[0].g, hs[0].field, hs[0].mlp, F, 208, 160, 16 * s0.n)
    ref = []
    for h in hs:
        out = [torch.empty((3, 160, 208)).pin_memory() for _ in range(F)]
        dws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        fgs.fgs_frames_host(h.g, h.field, h.mlp, h.times, h.cams, out, dws)
        torch.cuda.synchronize()
        ref.append(out)
    assert not all(torch.equal(a, b) for a, b in zip(ref[0], ref[1]))   # the two batches differ
    lanes = [torch.cuda.Stream() for _ in range(2)]
    wss = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    outs = [[torch.full((3, 160, 208), float("nan")).pin_memory() for _ in range(F)] for _ in range(2)]
    last = [None, None]
    for k in range(8):
        j = k % 2
        which = (k // 2) % 2          # lane j renders batch 0, 1, 0, 1
        h = hs[which]
        fgs.fgs_frames_host(h.g, h.field, h.mlp, h.times, h.cams, outs[j], wss[j], stream=lanes[j])
        last[j] = which
    for j in range(2):
        fgs.fgs_frames_host_status(hs[last[j]].g, hs[last[j]].field, hs[last[j]].mlp, hs[last[j]].cams, wss[j],
                                   stream=lanes[j])
        for a, b in zip(ref[last[j]], outs[j]):
            assert torch.equal(a, b), j


@pytest.mark.parametrize("mode", ["default", "long_sort_direct_atomics_unculled", "radix"])
def test_repeated_runs_bit_identical(mode):
    """Race stand-in (compute-sanitizer is closed on the GPU pool): 12 back-to-back fgs_frames calls of
    the full metric batch (D: 100k Gaussians, 20 frames of 800x800) must give bit-identical images.  The
    warp-specialised deform (TMEM / mbarrier pipeline), the atomics-based binning (slot claims in
    arbitrary order), the persistent long-list sort's work queue and the blend all run every time; a
    missing barrier or fence shows up as a differing image.  The second mode sends most tiles through
    the long-list CTA sort (sort cap 32), forces the direct-atomics binning and disables the blend cull."""
    import contextlib
    import torch
    s = make_scene("dnerf")
    ds = _ds(s)
    F = s.n_frames
    outs, _ = ds.alloc_deformed(F)
    imgs = [torch.empty((3, 800, 800), device="cuda") for _ in range(F)]
    ws = ds.alloc_workspace(F)
    ctx = contextlib.ExitStack()
    if mode == "long_sort_direct_atomics_unculled":
        ctx.enter_context(fgs.tuning(fgs.FGS_TUNE_RADIX, 0))
        ctx.enter_context(fgs.tuning(fgs.FGS_TUNE_TILE_SORT_CAP, 32))
        ctx.enter_context(fgs.tuning(fgs.FGS_TUNE_AGG_TILES, 1))
        ctx.enter_context(fgs.tuning(fgs.FGS_TUNE_BLEND_CULL, 0))
    elif mode == "radix":
        ctx.enter_context(fgs.tuning(fgs.FGS_TUNE_RADIX, 2))
    with ctx:
        ref = None
        for it in range(12):
            fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, imgs, ws)
            fgs.fgs_render_status(ws, F)
            cur = torch.stack(imgs).clone()
            if ref is None:
                ref = cur
            else:
                assert torch.equal(cur, ref), (mode, it, int((cur != ref).sum()))
    # and the default configuration gives the same images as the stressed one
    if mode != "default":
        fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, imgs, ws)
        assert torch.equal(torch.stack(imgs), ref)


@pytest.mark.parametrize("name,n,W,H,frames", [("tiny", 2011, 70, 50, 1), ("dnerf", 30_000, 200, 136, 3),
                                                ("hypernerf", 40_000, 240, 136, 2), ("neu3d", 20_000, 338, 254, 2)])
def test_radix_path_bit_identical_to_tile_sorts(name, n, W, H, frames):
    """The radix binning path (FGS_TUNE_RADIX = 2: stable LSD depth sort of the Gaussians, emission in
    depth order, stable tile passes) gives exactly the per-tile sorts' lists, ranges and images, through
    fgs_frames batches (several frames per launch, ragged tile grids), and the oracle's lists."""
    import torch
    s = make_scene(name, n=n, width=W, height=H, n_frames=frames)
    ds = _ds(s)
    outs, _ = ds.alloc_deformed(frames)
    res = {}
    for mode in (0, 2):
        imgs = [torch.empty((3, H, W), device="cuda") for _ in range(frames)]
        ws = ds.alloc_workspace(frames)
        with fgs.tuning(fgs.FGS_TUNE_RADIX, mode):
            fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, imgs, ws)
            fgs.fgs_render_status(ws, frames)
            dbg = gpu_render_debug(ds, s.cameras[0], outs[0])
        res[mode] = ([im.cpu().numpy() for im in imgs], dbg)
    for a, b in zip(res[0][0], res[2][0]):
        assert np.array_equal(a, b)
    for k in ("sorted_gid", "sorted_tile", "ranges", "image", "n_contrib"):
        assert np.array_equal(res[0][1][k], res[2][1][k]), k
    if n <= 2011:
        _render_parity(s)


def test_radix_auto_selection_and_threshold():
    """Auto mode (FGS_TUNE_RADIX = 1) takes the radix path on long-list frames only (n >= 64 x tiles and
    mean list >= the threshold); the result is identical for every threshold and to the default path."""
    import torch
    s = make_scene("dnerf", n=40_000, width=160, height=128, n_frames=2)      # 80 tiles: lists ~3000
    ds = _ds(s)
    dstruct, _, _ = gpu_deform(ds, float(s.times[0]))
    outs = [gpu_render_debug(ds, s.cameras[0], dstruct)]
    for thr in (1, 768, 1 << 20):
        with fgs.tuning(fgs.FGS_TUNE_RADIX, 1), fgs.tuning(fgs.FGS_TUNE_RADIX_MIN_LIST, thr):
            outs.append(gpu_render_debug(ds, s.cameras[0], dstruct))
    for o in outs[1:]:
        for k in ("sorted_gid", "ranges", "image"):
            assert np.array_equal(o[k], outs[0][k]), k


@pytest.mark.parametrize("W,H", [(16384, 24), (20, 16384)])
def test_maximum_image_extent(W, H):
    """The largest image side the ABI accepts (16384 px: 1024 tiles along it, the 16-bit packed rect's
    range): strips through the tiny scene, integer work and pixels against the oracle, tile lists
    bit-exact (every tile)."""
    s = make_scene("tiny", n=1500, width=W, height=H)
    _render_parity(s, max_instances=400 * s.n)        # fx ~ 17.6k px at 16384 wide: big rects
    with pytest.raises(fgs.FgsError):
        bad = make_scene("tiny", n=10, width=16385, height=8)
        ds = _ds(bad)
        gpu_render_debug(ds, bad.cameras[0], ds.canonical_struct())
