"""Helpers shared by the -m gpu tests: run the CUDA path through the C ABI and
compare with the fp64 oracle by the parity protocol of SURVEY §8(c.5)."""
import math

import numpy as np

from paper_2310_08528_b200 import build, fgs


def ensure_lib():
    build.build()
    return fgs.lib()


def gpu_deform(ds, t, begin=None, end=None):
    import torch
    outs, tens = ds.alloc_deformed(1)
    for v in tens[0].values():
        v.fill_(float("nan"))
    if begin is None:
        fgs.fgs_deform(ds.g, ds.field, ds.mlp, t, outs[0])
    else:
        fgs.fgs_deform_range(ds.g, ds.field, ds.mlp, t, begin, end, outs[0])
    torch.cuda.synchronize()
    return outs[0], {k: v.cpu().numpy() for k, v in tens[0].items()}, tens[0]


def gpu_render_debug(ds, cam, dstruct, max_instances=None):
    """Render one frame with every debug output; returns numpy dict."""
    import torch
    n = ds.n
    W, H = cam.width, cam.height
    cap = max(16 * n, 1024) if max_instances is None else max_instances
    ws = ds.alloc_workspace(1, cap, W, H)
    dev = ds.device
    gx, gy = (W + 15) // 16, (H + 15) // 16
    t = {
        "radii": torch.zeros(max(n, 1), dtype=torch.int32, device=dev),
        "rect": torch.zeros((max(n, 1), 4), dtype=torch.int32, device=dev),
        "mean2d": torch.zeros((max(n, 1), 2), dtype=torch.float32, device=dev),
        "depth_key": torch.zeros(max(n, 1), dtype=torch.int32, device=dev),
        "tiles_touched": torch.zeros(max(n, 1), dtype=torch.int32, device=dev),
        "n_instances": torch.zeros(1, dtype=torch.int32, device=dev),
        "sorted_tile": torch.zeros(cap, dtype=torch.int32, device=dev),
        "sorted_gid": torch.zeros(cap, dtype=torch.int32, device=dev),
        "ranges": torch.zeros((gx * gy, 2), dtype=torch.int32, device=dev),
        "final_T": torch.zeros((H, W), dtype=torch.float32, device=dev),
        "n_contrib": torch.zeros((H, W), dtype=torch.int32, device=dev),
        "n_evaluated": torch.zeros((H, W), dtype=torch.int32, device=dev),
        "blend_work": torch.zeros(2, dtype=torch.int64, device=dev),
        "binning_direct": torch.zeros(2, dtype=torch.int32, device=dev),
        "long_sort_paths": torch.zeros(3, dtype=torch.int32, device=dev),
    }
    aux = fgs.fgs_render_aux(**{k: v.data_ptr() for k, v in t.items()})
    image = torch.full((3, H, W), float("nan"), dtype=torch.float32, device=dev)
    fgs.fgs_render_debug(fgs.make_camera(cam), dstruct, image, ws, aux)
    status = fgs.lib().fgs_render_status(fgs._ptr(ws), ws.numel(), 1, fgs._stream())
    out = {k: v.cpu().numpy() for k, v in t.items()}
    out["image"] = image.cpu().numpy()
    out["status"] = status
    out["depth_key"] = out["depth_key"].view(np.uint32)
    M = int(out["n_instances"][0])
    out["M"] = M
    out["sorted_tile"] = out["sorted_tile"][:min(M, cap)].astype(np.int64)
    out["sorted_gid"] = out["sorted_gid"][:min(M, cap)].astype(np.int64)
    return out


def compare_integer_work(g, o_pre, o_bins, boundary=None):
    """Bit-exact comparison of radii, rects, tiles_touched, depth keys and per-tile lists,
    excluding boundary Gaussians (§8(c.5)).  Returns a dict of mismatch counts."""
    bnd = o_pre["boundary"] if boundary is None else boundary
    keep = ~bnd
    n = len(keep)
    res = {}
    res["radii"] = int(np.sum((g["radii"][:n] != o_pre["radius"]) & keep))
    res["rect"] = int(np.sum(np.any(g["rect"][:n] != o_pre["rect"], axis=1) & keep))
    res["tiles_touched"] = int(np.sum((g["tiles_touched"][:n] != o_pre["tiles_touched"]) & keep))
    res["depth_key"] = int(np.sum((g["depth_key"][:n] != o_pre["depth_key"]) & keep))
    o_tiles, o_gids, o_ranges = o_bins
    bad_tiles = 0
    g_ranges = g["ranges"]
    for tile in range(o_ranges.shape[0]):
        a = o_gids[o_ranges[tile, 0]:o_ranges[tile, 1]]
        b = g["sorted_gid"][g_ranges[tile, 0]:g_ranges[tile, 1]]
        a = a[keep[a]]
        b = b[keep[b]] if b.size else b
        if a.shape != b.shape or not np.array_equal(a, b):
            bad_tiles += 1
    res["tile_lists"] = bad_tiles
    res["n_boundary"] = int(bnd.sum())
    return res


def psnr(a, b):
    mse = float(np.mean((a - b) ** 2))
    return float("inf") if mse == 0 else 10 * math.log10(1.0 / mse)


def compare_pixels(g_img, o_img, o_flag, tiles_mask=None):
    """PSNR over all compared pixels and max |delta| over unflagged ones."""
    m = np.isfinite(o_img[0]) if tiles_mask is None else tiles_mask
    d = np.abs(g_img - o_img)
    un = m & ~o_flag
    return {"psnr": psnr(g_img[:, m], o_img[:, m]), "max_unflagged": float(d[:, un].max()) if un.any() else 0.0,
            "max_all": float(d[:, m].max()), "flagged": int((o_flag & m).sum()), "pixels": int(m.sum())}
