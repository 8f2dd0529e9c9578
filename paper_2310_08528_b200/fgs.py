"""Thin ctypes binding of libfgs.so (include/fgs.h) — argument marshalling only.

Every step of the path runs in the sm_100a kernels of libfgs.so; this module only
builds the C structs from torch CUDA tensors (device memory) and passes
`torch.cuda.current_stream()`.  There is no CPU fallback: if the library cannot
be loaded the calls raise.  Function names are the C ABI's.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_int64, c_size_t, c_void_p
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# FGS_LIB=checked loads the checked build (device-side assertions, build.py --checked) — same ABI
LIB_PATH = os.path.join(HERE, "libfgs_checked.so" if os.environ.get("FGS_LIB", "") == "checked" else "libfgs.so")

FGS_OK, FGS_E_INVALID, FGS_E_CUDA, FGS_E_CAPACITY, FGS_E_NOTIMPL = 0, -1, -2, -3, -4
MAX_SCALES, PLANES, TILE = 4, 6, 16


class FgsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"fgs error {code}: {msg}")
        self.code = code


class fgs_gaussians(ctypes.Structure):
    _fields_ = [("n", c_int64), ("sh_degree", c_int32), ("means", c_void_p), ("log_scales", c_void_p),
                ("quats", c_void_p), ("opacity_logits", c_void_p), ("sh", c_void_p)]


class fgs_hexplanes(ctypes.Structure):
    _fields_ = [("n_scales", c_int32), ("feat", c_int32), ("t_res", c_int32),
                ("res", c_int32 * MAX_SCALES), ("bmin", c_float * 3), ("bmax", c_float * 3),
                ("planes", (c_void_p * PLANES) * MAX_SCALES)]


MLP_ARRAYS = ("w_d", "b_d", "w_x", "b_x", "w_r", "b_r", "w_s", "b_s", "w_c", "b_c", "w_a", "b_a")


class fgs_mlp(ctypes.Structure):
    _fields_ = [("in_dim", c_int32), ("width", c_int32)] + [(k, c_void_p) for k in MLP_ARRAYS]


class fgs_deformed(ctypes.Structure):
    _fields_ = [("n", c_int64), ("sh_degree", c_int32), ("means", c_void_p), ("log_scales", c_void_p),
                ("quats", c_void_p), ("opacity_logits", c_void_p), ("sh", c_void_p)]


class fgs_camera(ctypes.Structure):
    _fields_ = [("R", c_float * 9), ("t", c_float * 3), ("fx", c_float), ("fy", c_float),
                ("cx", c_float), ("cy", c_float), ("width", c_int32), ("height", c_int32),
                ("bg", c_float * 3)]


class fgs_render_aux(ctypes.Structure):
    _fields_ = [(k, c_void_p) for k in ("radii", "rect", "mean2d", "depth_key", "tiles_touched",
                                        "n_instances", "sorted_tile", "sorted_gid", "ranges",
                                        "final_T", "n_contrib", "n_evaluated", "blend_work",
                                        "binning_direct", "long_sort_paths")]


class fgs_gaussian_grads(ctypes.Structure):
    _fields_ = [(k, c_void_p) for k in ("means", "log_scales", "quats", "opacity_logits", "sh")]


class fgs_field_grads(ctypes.Structure):
    _fields_ = [("planes", (c_void_p * PLANES) * MAX_SCALES)] + [(k, c_void_p) for k in MLP_ARRAYS]


FGS_LOSS_PARTIALS = 1024

_LIB = None
EXPORTS = ("fgs_deform", "fgs_deform_range", "fgs_deform_range_peers", "fgs_deform_batch", "fgs_render_workspace_bytes",
           "fgs_render", "fgs_render_batch", "fgs_render_debug", "fgs_render_status", "fgs_frames",
           "fgs_frames_host_workspace_bytes", "fgs_frames_host", "fgs_frames_host_status", "fgs_profile_enable", "fgs_profile_read",
           "fgs_launch_count", "fgs_set_tuning", "fgs_get_tuning", "fgs_last_error", "fgs_version",
           "fgs_l1_loss", "fgs_tv_loss", "fgs_render_backward_scratch_bytes", "fgs_render_backward",
           "fgs_deform_backward_scratch_bytes", "fgs_deform_backward", "fgs_adam_step")
SIZE_EXPORTS = ("fgs_render_workspace_bytes", "fgs_frames_host_workspace_bytes", "fgs_render_backward_scratch_bytes",
                "fgs_deform_backward_scratch_bytes")
STAGES = ("deform", "preprocess", "tile_scan", "duplicate", "tile_sort", "blend")
FGS_TUNE_TILE_SORT_CAP = 0
FGS_TUNE_BLEND_CULL = 2
FGS_TUNE_AGG_TILES = 3
FGS_TUNE_RADIX = 4
FGS_TUNE_RADIX_MIN_LIST = 5
FGS_TUNE_LONG_SORT = 6
FGS_TUNE_TILE_CULL = 7


def lib():
    """Load libfgs.so (raises if it is missing: there is no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise FgsError(FGS_E_CUDA, f"{LIB_PATH} not built: run `python -m paper_2310_08528_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        P = POINTER
        L.fgs_deform.argtypes = [P(fgs_gaussians), P(fgs_hexplanes), P(fgs_mlp), c_float, P(fgs_deformed), c_void_p]
        L.fgs_deform_range.argtypes = [P(fgs_gaussians), P(fgs_hexplanes), P(fgs_mlp), c_float, c_int64, c_int64,
                                       P(fgs_deformed), c_void_p]
        L.fgs_deform_range_peers.argtypes = [P(fgs_gaussians), P(fgs_hexplanes), P(fgs_mlp), c_float, c_int64,
                                             c_int64, P(fgs_deformed), P(c_int64), c_int32, c_void_p]
        L.fgs_deform_batch.argtypes = [P(fgs_gaussians), P(fgs_hexplanes), P(fgs_mlp), P(c_float), c_int32,
                                       P(fgs_deformed), c_void_p]
        L.fgs_render_workspace_bytes.argtypes = [c_int64, c_int32, c_int32, c_int64]
        L.fgs_render_workspace_bytes.restype = c_size_t
        L.fgs_render.argtypes = [P(fgs_camera), P(fgs_deformed), c_void_p, c_void_p, c_size_t, c_void_p]
        L.fgs_render_batch.argtypes = [P(fgs_camera), P(fgs_deformed), P(c_void_p), c_int32, c_void_p, c_size_t,
                                       c_void_p]
        L.fgs_render_debug.argtypes = [P(fgs_camera), P(fgs_deformed), c_void_p, c_void_p, c_size_t,
                                       P(fgs_render_aux), c_void_p]
        L.fgs_render_status.argtypes = [c_void_p, c_size_t, c_int32, c_void_p]
        L.fgs_frames.argtypes = [P(fgs_gaussians), P(fgs_hexplanes), P(fgs_mlp), P(c_float), P(fgs_camera),
                                 c_int32, P(fgs_deformed), P(c_void_p), c_void_p, c_size_t, c_void_p]
        L.fgs_frames_host_workspace_bytes.argtypes = [P(fgs_gaussians), P(fgs_hexplanes), P(fgs_mlp), c_int32,
                                                      c_int32, c_int32, c_int64]
        L.fgs_frames_host_workspace_bytes.restype = c_size_t
        L.fgs_frames_host.argtypes = [P(fgs_gaussians), P(fgs_hexplanes), P(fgs_mlp), P(c_float), P(fgs_camera),
                                      c_int32, P(c_void_p), c_void_p, c_size_t, c_void_p]
        L.fgs_frames_host_status.argtypes = [P(fgs_gaussians), P(fgs_hexplanes), P(fgs_mlp), P(fgs_camera),
                                             c_int32, c_void_p, c_size_t, c_void_p]
        L.fgs_l1_loss.argtypes = [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]
        L.fgs_tv_loss.argtypes = [P(fgs_hexplanes), c_float, P(fgs_field_grads), c_void_p, c_void_p, c_void_p]
        L.fgs_render_backward_scratch_bytes.argtypes = [c_int64]
        L.fgs_render_backward_scratch_bytes.restype = c_size_t
        L.fgs_render_backward.argtypes = [P(fgs_camera), P(fgs_deformed), c_void_p, c_void_p, c_void_p, c_size_t,
                                          c_void_p, c_size_t, P(fgs_gaussian_grads), c_void_p]
        L.fgs_deform_backward_scratch_bytes.argtypes = [P(fgs_hexplanes), P(fgs_mlp)]
        L.fgs_deform_backward_scratch_bytes.restype = c_size_t
        L.fgs_deform_backward.argtypes = [P(fgs_gaussians), P(fgs_hexplanes), P(fgs_mlp), c_float,
                                          P(fgs_gaussian_grads), P(fgs_gaussian_grads), P(fgs_field_grads), c_void_p,
                                          c_size_t, c_void_p]
        L.fgs_adam_step.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_float, c_float, c_float,
                                    c_float, c_int32, c_void_p]
        L.fgs_profile_enable.argtypes = [c_int]
        L.fgs_profile_read.argtypes = [P(ctypes.c_double), P(c_int64)]
        L.fgs_launch_count.restype = c_int64
        L.fgs_set_tuning.argtypes = [c_int32, c_int64]
        L.fgs_get_tuning.argtypes = [c_int32]
        L.fgs_get_tuning.restype = c_int64
        L.fgs_last_error.restype = c_char_p
        L.fgs_version.restype = c_char_p
        for name in EXPORTS:
            if name not in SIZE_EXPORTS + ("fgs_launch_count", "fgs_get_tuning", "fgs_last_error", "fgs_version"):
                getattr(L, name).restype = c_int
        _LIB = L
    return _LIB


def _check(rc):
    if rc != FGS_OK:
        raise FgsError(rc, lib().fgs_last_error().decode())
    return rc


def _stream(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return c_void_p(s.cuda_stream)


def _ptr(t):
    return c_void_p(0 if t is None else t.data_ptr())


# ---------------------------------------------------------------- the C calls
def fgs_deform(g, field, mlp, t, out, stream=None):
    return _check(lib().fgs_deform(ctypes.byref(g), ctypes.byref(field), ctypes.byref(mlp), c_float(t),
                                   ctypes.byref(out), _stream(stream)))


def fgs_deform_range(g, field, mlp, t, begin, end, out, stream=None):
    return _check(lib().fgs_deform_range(ctypes.byref(g), ctypes.byref(field), ctypes.byref(mlp), c_float(t),
                                         c_int64(begin), c_int64(end), ctypes.byref(out), _stream(stream)))


def fgs_deform_range_peers(g, field, mlp, t, begin, end, out, peer_offsets: Sequence[int], stream=None):
    """fgs_deform_range whose outputs are also stored at byte offsets peer_offsets[q] from `out`'s
    arrays (the §8(e2) fused deform + gather; include/fgs.h)."""
    n = len(peer_offsets)
    arr = (c_int64 * max(n, 1))(*[int(x) for x in peer_offsets])
    return _check(lib().fgs_deform_range_peers(ctypes.byref(g), ctypes.byref(field), ctypes.byref(mlp), c_float(t),
                                               c_int64(begin), c_int64(end), ctypes.byref(out), arr, n,
                                               _stream(stream)))


def fgs_deform_batch(g, field, mlp, ts: Sequence[float], outs: Sequence[fgs_deformed], stream=None):
    n = len(ts)
    tarr = (c_float * max(n, 1))(*[float(x) for x in ts])
    oarr = (fgs_deformed * max(n, 1))(*outs)
    return _check(lib().fgs_deform_batch(ctypes.byref(g), ctypes.byref(field), ctypes.byref(mlp), tarr, n, oarr,
                                         _stream(stream)))


def fgs_render_workspace_bytes(n, width, height, max_instances):
    return int(lib().fgs_render_workspace_bytes(n, width, height, max_instances))


def fgs_render(cam, g, image, ws, stream=None):
    return _check(lib().fgs_render(ctypes.byref(cam), ctypes.byref(g), _ptr(image), _ptr(ws), ws.numel(),
                                   _stream(stream)))


def fgs_render_batch(cams, defs, images, ws, stream=None):
    F = len(cams)
    carr = (fgs_camera * max(F, 1))(*cams)
    darr = (fgs_deformed * max(F, 1))(*defs)
    iarr = (c_void_p * max(F, 1))(*[im.data_ptr() for im in images])
    return _check(lib().fgs_render_batch(carr, darr, iarr, F, _ptr(ws), ws.numel(), _stream(stream)))


def fgs_render_debug(cam, g, image, ws, aux, stream=None):
    return _check(lib().fgs_render_debug(ctypes.byref(cam), ctypes.byref(g), _ptr(image), _ptr(ws), ws.numel(),
                                         ctypes.byref(aux), _stream(stream)))


def fgs_render_status(ws, n_frames=1, stream=None):
    return _check(lib().fgs_render_status(_ptr(ws), ws.numel(), n_frames, _stream(stream)))


def fgs_frames(g, field, mlp, ts, cams, defs_scratch, images, ws, stream=None):
    F = len(ts)
    tarr = (c_float * max(F, 1))(*[float(x) for x in ts])
    carr = (fgs_camera * max(F, 1))(*cams)
    darr = (fgs_deformed * max(F, 1))(*defs_scratch)
    iarr = (c_void_p * max(F, 1))(*[im.data_ptr() for im in images])
    return _check(lib().fgs_frames(ctypes.byref(g), ctypes.byref(field), ctypes.byref(mlp), tarr, carr, F, darr,
                                   iarr, _ptr(ws), ws.numel(), _stream(stream)))


def fgs_frames_host_workspace_bytes(g_host, field_host, mlp_host, n_frames, width, height, max_instances):
    return int(lib().fgs_frames_host_workspace_bytes(ctypes.byref(g_host), ctypes.byref(field_host),
                                                     ctypes.byref(mlp_host), n_frames, width, height,
                                                     max_instances))


def fgs_frames_host(g_host, field_host, mlp_host, ts, cams, images_host, dev_ws, stream=None):
    """images_host: list of pinned CPU float32 tensors [3,H,W]; dev_ws: device uint8 tensor."""
    F = len(ts)
    tarr = (c_float * max(F, 1))(*[float(x) for x in ts])
    carr = (fgs_camera * max(F, 1))(*cams)
    iarr = (c_void_p * max(F, 1))(*[im.data_ptr() for im in images_host])
    return _check(lib().fgs_frames_host(ctypes.byref(g_host), ctypes.byref(field_host), ctypes.byref(mlp_host),
                                        tarr, carr, F, iarr, _ptr(dev_ws), dev_ws.numel(), _stream(stream)))


def fgs_frames_host_status(g_host, field_host, mlp_host, cams, dev_ws, stream=None):
    """FGS_E_CAPACITY (raised) if a frame of the last fgs_frames_host call into dev_ws overflowed."""
    F = len(cams)
    carr = (fgs_camera * max(F, 1))(*cams)
    return _check(lib().fgs_frames_host_status(ctypes.byref(g_host), ctypes.byref(field_host),
                                               ctypes.byref(mlp_host), carr, F, _ptr(dev_ws), dev_ws.numel(),
                                               _stream(stream)))


class tuning:
    """Context manager: set a tuning knob for the block, restore it after (tests, tools)."""

    def __init__(self, key, value):
        self.key, self.value = key, value

    def __enter__(self):
        self.old = fgs_get_tuning(self.key)
        fgs_set_tuning(self.key, self.value)
        return self

    def __exit__(self, *exc):
        fgs_set_tuning(self.key, self.old)
        return False


def fgs_l1_loss(image, target, dL_dimage, partials, loss, stream=None):
    """loss[0] = mean |image - target|; dL_dimage = sign / (3HW) (device tensors; partials float64[1024])."""
    H, W = image.shape[-2], image.shape[-1]
    return _check(lib().fgs_l1_loss(_ptr(image), _ptr(target), W, H, _ptr(dL_dimage), _ptr(partials), _ptr(loss),
                                    _stream(stream)))


def fgs_tv_loss(field, weight, grads, partials, loss, stream=None):
    return _check(lib().fgs_tv_loss(ctypes.byref(field), c_float(weight), None if grads is None else ctypes.byref(grads),
                                    _ptr(partials), _ptr(loss), _stream(stream)))


def fgs_render_backward_scratch_bytes(n):
    return int(lib().fgs_render_backward_scratch_bytes(n))


def fgs_render_backward(cam, g, image, dL_dimage, ws, scratch, dg, stream=None):
    return _check(lib().fgs_render_backward(ctypes.byref(cam), ctypes.byref(g), _ptr(image), _ptr(dL_dimage),
                                            _ptr(ws), ws.numel(), _ptr(scratch), scratch.numel(), ctypes.byref(dg),
                                            _stream(stream)))


def fgs_deform_backward_scratch_bytes(field, mlp):
    return int(lib().fgs_deform_backward_scratch_bytes(ctypes.byref(field), ctypes.byref(mlp)))


def fgs_deform_backward(g, field, mlp, t, d_deformed, d_canonical, d_field, scratch, stream=None):
    return _check(lib().fgs_deform_backward(ctypes.byref(g), ctypes.byref(field), ctypes.byref(mlp), c_float(t),
                                            ctypes.byref(d_deformed), ctypes.byref(d_canonical), ctypes.byref(d_field),
                                            _ptr(scratch), scratch.numel(), _stream(stream)))


def fgs_adam_step(param, grad, m, v, lr, step, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
    """One Adam step on device tensors of equal numel (param, m, v updated in place)."""
    return _check(lib().fgs_adam_step(_ptr(param), _ptr(grad), _ptr(m), _ptr(v), param.numel(), c_float(lr),
                                      c_float(beta1), c_float(beta2), c_float(eps), int(step), _stream(stream)))


def fgs_profile_enable(enable=True):
    return _check(lib().fgs_profile_enable(1 if enable else 0))


def fgs_profile_read():
    """Returns {stage: (ms, launches)} accumulated since the last read (synchronises)."""
    ms = (ctypes.c_double * len(STAGES))()
    cnt = (c_int64 * len(STAGES))()
    _check(lib().fgs_profile_read(ms, cnt))
    return {name: (ms[i], cnt[i]) for i, name in enumerate(STAGES)}


def fgs_launch_count():
    return int(lib().fgs_launch_count())


def fgs_set_tuning(key, value):
    return _check(lib().fgs_set_tuning(key, value))


def fgs_get_tuning(key):
    return int(lib().fgs_get_tuning(key))


def fgs_last_error():
    return lib().fgs_last_error().decode()


def fgs_version():
    return lib().fgs_version().decode()


# ---------------------------------------------------------------- marshalling helpers
def make_camera(cam) -> fgs_camera:
    """inputs.Camera -> fgs_camera (host struct)."""
    c = fgs_camera()
    c.R[:] = [float(v) for v in np.asarray(cam.R, np.float32).ravel()]
    c.t[:] = [float(v) for v in np.asarray(cam.t, np.float32).ravel()]
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.width, c.height = int(cam.width), int(cam.height)
    c.bg[:] = [float(v) for v in np.asarray(cam.bg, np.float32).ravel()]
    return c


def deformed_rows(d: fgs_deformed, row0: int, n: int, opacity_logits=None, sh=None) -> fgs_deformed:
    """View of rows [row0, row0 + n) of a deformed set's means / log_scales / quats as an fgs_deformed
    of n Gaussians (composition: deform model k into its own row range of one G', then render the
    union).  opacity/sh default to the same row range of d's arrays."""
    K3 = (d.sh_degree + 1) ** 2 * 3
    return fgs_deformed(n, d.sh_degree, d.means + 12 * row0, d.log_scales + 12 * row0, d.quats + 16 * row0,
                        (d.opacity_logits + 4 * row0) if opacity_logits is None else opacity_logits,
                        (d.sh + 4 * K3 * row0) if sh is None else sh)


class HostScene:
    """A Scene's arrays in pinned host memory + C structs whose pointers are HOST pointers
    (the inputs of fgs_frames_host, i.e. the end-to-end path)."""

    def __init__(self, scene):
        import torch

        def T(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).pin_memory()

        self.scene = scene
        self.n = scene.n
        self.arrays = {k: T(getattr(scene, k)) for k in ("means", "log_scales", "quats", "opacity_logits", "sh")}
        a = self.arrays
        self.g = fgs_gaussians(self.n, scene.sh_degree, a["means"].data_ptr(), a["log_scales"].data_ptr(),
                               a["quats"].data_ptr(), a["opacity_logits"].data_ptr(), a["sh"].data_ptr())
        f = scene.field
        self.planes = [[T(P) for P in ps] for ps in f.planes]
        hp = fgs_hexplanes()
        hp.n_scales, hp.feat, hp.t_res = len(f.res), f.feat, f.t_res
        for l, R in enumerate(f.res):
            hp.res[l] = R
            for p in range(PLANES):
                hp.planes[l][p] = self.planes[l][p].data_ptr()
        hp.bmin[:] = [float(v) for v in f.bmin]
        hp.bmax[:] = [float(v) for v in f.bmax]
        self.field = hp
        m = scene.mlp
        self.mlp_t = {k: T(getattr(m, k)) for k in MLP_ARRAYS if getattr(m, k, None) is not None}
        mm = fgs_mlp()
        mm.in_dim, mm.width = m.in_dim, m.width
        for k, v in self.mlp_t.items():
            setattr(mm, k, v.data_ptr())
        self.mlp = mm
        self.cams = [make_camera(c) for c in scene.cameras]
        self.times = [float(t) for t in scene.times]

    def h2d_bytes(self):
        tot = sum(v.numel() * 4 for v in self.arrays.values())
        tot += sum(P.numel() * 4 for ps in self.planes for P in ps)
        tot += sum(v.numel() * 4 for v in self.mlp_t.values())
        return tot


class DeviceScene:
    """A Scene's arrays resident in device memory (torch tensors) + the C structs over them."""

    def __init__(self, scene, device="cuda"):
        import torch

        def T(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device)

        self.scene = scene
        self.device = device
        self.n = scene.n
        self.sh_degree = scene.sh_degree
        self.means, self.log_scales, self.quats = T(scene.means), T(scene.log_scales), T(scene.quats)
        self.opacity_logits, self.sh = T(scene.opacity_logits), T(scene.sh)
        f = scene.field
        self.planes = [[T(P) for P in ps] for ps in f.planes]
        m = scene.mlp
        self.mlp_t = {k: T(getattr(m, k)) for k in MLP_ARRAYS if getattr(m, k, None) is not None}
        self.has_c = "w_c" in self.mlp_t
        self.has_a = "w_a" in self.mlp_t
        self.g = fgs_gaussians(self.n, self.sh_degree, self.means.data_ptr(), self.log_scales.data_ptr(),
                               self.quats.data_ptr(), self.opacity_logits.data_ptr(), self.sh.data_ptr())
        hp = fgs_hexplanes()
        hp.n_scales, hp.feat, hp.t_res = len(f.res), f.feat, f.t_res
        for l, R in enumerate(f.res):
            hp.res[l] = R
            for p in range(PLANES):
                hp.planes[l][p] = self.planes[l][p].data_ptr()
        hp.bmin[:] = [float(v) for v in f.bmin]
        hp.bmax[:] = [float(v) for v in f.bmax]
        self.field = hp
        mm = fgs_mlp()
        mm.in_dim, mm.width = m.in_dim, m.width
        for k, v in self.mlp_t.items():
            setattr(mm, k, v.data_ptr())
        self.mlp = mm
        self.cams = [make_camera(c) for c in scene.cameras]
        self.times = [float(t) for t in scene.times]

    def alloc_deformed(self, n_frames=1):
        """Device output buffers for n_frames deformations; returns (structs, tensors)."""
        import torch
        outs, tens = [], []
        for _ in range(n_frames):
            X = torch.empty((self.n, 3), dtype=torch.float32, device=self.device)
            S = torch.empty((self.n, 3), dtype=torch.float32, device=self.device)
            Q = torch.empty((self.n, 4), dtype=torch.float32, device=self.device)
            tens.append({"means": X, "log_scales": S, "quats": Q})
            # with the P:1232 decoders the deformed opacity / SH are per-frame outputs too
            O = torch.empty_like(self.opacity_logits) if self.has_a else None
            C = torch.empty_like(self.sh) if self.has_c else None
            if O is not None:
                tens[-1]["opacity_logits"] = O
            if C is not None:
                tens[-1]["sh"] = C
            d = self.deformed_struct(X, S, Q, O, C)
            d._keep = (X, S, Q, O, C)  # the struct owns its device buffers (raw pointers inside)
            outs.append(d)
        return outs, tens

    def deformed_struct(self, means, log_scales, quats, opacity=None, sh=None) -> fgs_deformed:
        return fgs_deformed(self.n, self.sh_degree, means.data_ptr(), log_scales.data_ptr(), quats.data_ptr(),
                            (self.opacity_logits if opacity is None else opacity).data_ptr(),
                            (self.sh if sh is None else sh).data_ptr())

    def canonical_struct(self) -> fgs_deformed:
        """G itself as an fgs_deformed (render the undeformed scene, e.g. the warm-up / static case)."""
        return self.deformed_struct(self.means, self.log_scales, self.quats)

    def alloc_gaussian_grads(self):
        """Zeroed device gradient buffers shaped like the Gaussian arrays; returns (struct, tensors)."""
        import torch
        t = {k: torch.zeros_like(getattr(self, k)) for k in ("means", "log_scales", "quats", "opacity_logits", "sh")}
        st = fgs_gaussian_grads(*[t[k].data_ptr() for k in ("means", "log_scales", "quats", "opacity_logits", "sh")])
        st._keep = t
        return st, t

    def alloc_field_grads(self):
        """Zeroed device gradient buffers shaped like the planes and the MLP; returns (struct, tensors)."""
        import torch
        t = {}
        st = fgs_field_grads()
        for l, ps in enumerate(self.planes):
            for p, P in enumerate(ps):
                t[f"plane{l}_{p}"] = torch.zeros_like(P)
                st.planes[l][p] = t[f"plane{l}_{p}"].data_ptr()
        for k in MLP_ARRAYS:
            if k in self.mlp_t:
                t[k] = torch.zeros_like(self.mlp_t[k])
                setattr(st, k, t[k].data_ptr())
        st._keep = t
        return st, t

    def alloc_workspace(self, n_frames=1, max_instances=None, width=None, height=None):
        import torch
        W = self.scene.cameras[0].width if width is None else width
        H = self.scene.cameras[0].height if height is None else height
        cap = max(16 * self.n, 1024) if max_instances is None else max_instances
        per = fgs_render_workspace_bytes(self.n, W, H, cap)
        return torch.empty(per * n_frames, dtype=torch.uint8, device=self.device)
