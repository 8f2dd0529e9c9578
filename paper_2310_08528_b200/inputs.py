"""Seeded synthetic inputs for the 4D-GS per-frame deform + render path.

This module is shared by the CUDA path (bench, tests) and the fp64 oracle.  It
holds NONE of the method's arithmetic: it only draws random numbers, builds
look-at cameras and lays the arrays out the way the C ABI (include/fgs.h)
expects.  Everything returned is float32 (or int) numpy; the oracle promotes
the same fp32 arrays to fp64, the GPU path copies them to device memory.

Recipe: SURVEY.md §8(d) "Synthetic inputs" (BASELINE.json configs[0..4]).
  * np.random.default_rng(seed), draws in fp64, cast to fp32 (round-to-nearest).
  * Draw order: means, log-scales, quats (normalised after the draw), opacity
    logits, SH DC, SH rest, planes (scale-major; plane order xy,xz,yz,xt,yt,zt),
    W_d, b_d, W_x, W_r, W_s (head biases are 0 and not drawn), cameras, times.
  * Seeds: T=0, D=1, H=2, N3=3, S=4.
The inputs stand in for D-NeRF / HyperNeRF / Neu3D (not in the container); no
item of those datasets is reproduced — only their image sizes, camera layouts
and the paper's field hyper-parameters.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

# Plane order of PAPER.md P:781/P:787: (x,y),(x,z),(y,z),(x,t),(y,t),(z,t).
# Axis ids: 0=x, 1=y, 2=z, 3=t.  Plane (a,b) is stored [n_b][n_a][feat].
PLANE_AXES = ((0, 1), (0, 2), (1, 2), (0, 3), (1, 3), (2, 3))


@dataclass
class Camera:
    """World->camera pinhole camera, OpenCV axes (x right, y down, z forward).

    p_cam = R @ X + t ; pixel = (fx*x/z + cx, fy*y/z + cy).  Mirrors fgs_camera.
    """
    R: np.ndarray          # [3,3] fp32, row-major
    t: np.ndarray          # [3] fp32
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    bg: np.ndarray         # [3] fp32


@dataclass
class Field:
    """Multi-resolution HexPlane R_l(i,j) + AABB (reading D1)."""
    feat: int
    res: List[int]         # spatial resolution per scale
    t_res: int             # temporal resolution (reading D3: fixed over scales)
    bmin: np.ndarray       # [3] fp32
    bmax: np.ndarray       # [3] fp32
    planes: List[List[np.ndarray]]  # [scale][6] -> [n_b][n_a][feat] fp32

    @property
    def n_scales(self) -> int:
        return len(self.res)


@dataclass
class MLP:
    """phi_d (one Linear + ReLU, reading D5) and heads phi_x, phi_r, phi_s (D6).

    Weights row-major [out][in] fp32 (PyTorch Linear layout).
    """
    w_d: np.ndarray
    b_d: np.ndarray
    w_x: np.ndarray
    b_x: np.ndarray
    w_r: np.ndarray
    b_r: np.ndarray
    w_s: np.ndarray
    b_s: np.ndarray
    # optional colour / opacity decoders phi_C, phi_alpha: [3K][W], [3K]; [1][W], [1]
    w_c: Optional[np.ndarray] = None
    b_c: Optional[np.ndarray] = None
    w_a: Optional[np.ndarray] = None
    b_a: Optional[np.ndarray] = None

    @property
    def width(self) -> int:
        return self.w_d.shape[0]

    @property
    def in_dim(self) -> int:
        return self.w_d.shape[1]


@dataclass
class Scene:
    name: str
    seed: int
    means: np.ndarray            # [N,3]
    log_scales: np.ndarray       # [N,3]
    quats: np.ndarray            # [N,4] (w,x,y,z), raw
    opacity_logits: np.ndarray   # [N]
    sh: np.ndarray               # [N,K,3]
    sh_degree: int
    field: Field
    mlp: MLP
    cameras: List[Camera]        # one per frame
    times: np.ndarray            # [F] fp32, one per frame
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.means.shape[0]

    @property
    def n_frames(self) -> int:
        return len(self.cameras)


# --------------------------------------------------------------------------
# Config table (BASELINE.json configs)
# --------------------------------------------------------------------------
CONFIGS = {
    "tiny": dict(seed=0, n=2000, width=64, height=64, feat=16, res=[32], t_res=8,
                 width_mlp=32, sh_degree=0, log_scale=(-3.0, 0.3), bg=(0, 0, 0)),
    "dnerf": dict(seed=1, n=100_000, width=800, height=800, feat=32, res=[64, 128],
                  t_res=25, width_mlp=64, sh_degree=3, log_scale=(-4.5, 0.5), bg=(1, 1, 1)),
    "hypernerf": dict(seed=2, n=250_000, width=960, height=540, feat=32, res=[64, 128],
                      t_res=75, width_mlp=128, sh_degree=3, log_scale=(-5.0, 0.6),
                      bg=(0, 0, 0)),
    "neu3d": dict(seed=3, n=300_000, width=1352, height=1014, feat=32, res=[64, 128],
                  t_res=150, width_mlp=128, sh_degree=3, log_scale=(-5.0, 0.7),
                  bg=(0, 0, 0)),
    "scaling": dict(seed=4, n=2_000_000, width=1920, height=1080, feat=32, res=[128, 256],
                    t_res=150, width_mlp=128, sh_degree=3, log_scale=(-5.5, 0.6),
                    bg=(0, 0, 0)),
}
ALIASES = {"T": "tiny", "D": "dnerf", "H": "hypernerf", "N3": "neu3d", "S": "scaling"}


def fx_for_width(width: int, fovx_deg: float = 50.0) -> float:
    """fx = fy = W / (2 tan(fovx/2)) (reading R15: horizontal fov 50 deg)."""
    return width / (2.0 * math.tan(math.radians(fovx_deg) / 2.0))


def look_at(eye, target, width, height, bg, up=(0.0, 1.0, 0.0)) -> Camera:
    """OpenCV look-at camera (SURVEY §8(d) cameras row; reading R12 for cx, cy)."""
    eye = np.asarray(eye, np.float64)
    target = np.asarray(target, np.float64)
    fwd = target - eye
    fwd /= np.linalg.norm(fwd)
    up = np.asarray(up, np.float64)
    if abs(float(fwd @ up)) > 0.99:
        up = np.array([0.0, 0.0, 1.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    t = -R @ eye
    f = fx_for_width(width)
    return Camera(R=R.astype(np.float32), t=t.astype(np.float32), fx=float(np.float32(f)),
                  fy=float(np.float32(f)), cx=float(np.float32((width - 1) / 2.0)),
                  cy=float(np.float32((height - 1) / 2.0)), width=int(width),
                  height=int(height), bg=np.asarray(bg, np.float32))


def _f32(a):
    return np.asarray(a, np.float64).astype(np.float32)


def _draw_means(rng, name, n):
    if name == "tiny":
        return rng.uniform(-1.0, 1.0, (n, 3))
    if name == "dnerf":
        return rng.uniform(-1.3, 1.3, (n, 3))
    if name == "hypernerf":
        # N(0, diag(1.5,0.8,1.5)) read as a covariance (reading R18).
        return rng.normal(0.0, 1.0, (n, 3)) * np.sqrt([1.5, 0.8, 1.5])
    if name == "neu3d":
        xy = rng.uniform(-3.0, 3.0, (n, 2))
        z = rng.uniform(2.0, 8.0, (n, 1))
        return np.concatenate([xy, z], axis=1)
    if name == "scaling":
        return rng.uniform(-4.0, 4.0, (n, 3))
    raise KeyError(name)


def _aabb(name):
    if name == "tiny":
        return (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)
    if name == "dnerf":
        return (-1.3, -1.3, -1.3), (1.3, 1.3, 1.3)
    if name == "hypernerf":
        a, b = 3 * math.sqrt(1.5), 3 * math.sqrt(0.8)
        return (-a, -b, -a), (a, b, a)
    if name == "neu3d":
        return (-3.0, -3.0, 2.0), (3.0, 3.0, 8.0)
    if name == "scaling":
        return (-4.0, -4.0, -4.0), (4.0, 4.0, 4.0)
    raise KeyError(name)


def _cameras_times(rng, name, width, height, bg, n_frames=None):
    cams, times = [], []
    if name == "tiny":
        cams.append(look_at((0, 0, 4), (0, 0, 0), width, height, bg))
        times.append(0.37)
    elif name == "dnerf":
        F = 20 if n_frames is None else n_frames
        for k in range(F):
            u = rng.normal(size=3)
            u /= np.linalg.norm(u)
            cams.append(look_at(4.0 * u, (0, 0, 0), width, height, bg))
            times.append(k / max(F - 1, 1))
    elif name == "hypernerf":
        F = 50 if n_frames is None else n_frames
        for k in range(F):
            psi, th = rng.uniform(-0.1, 0.1, 2)
            eye = 4.0 * np.array([math.sin(psi) * math.cos(th), math.sin(th),
                                  -math.cos(psi) * math.cos(th)])
            cams.append(look_at(eye, (0, 0, 0), width, height, bg))
            times.append(k / max(F - 1, 1))
    elif name == "neu3d":
        F = 8 if n_frames is None else n_frames
        for j in range(F):
            phi = (j / 7.0 - 0.5) * 0.2
            eye = (5 * math.sin(phi), 0.0, 5 - 5 * math.cos(phi))
            cams.append(look_at(eye, (0, 0, 5), width, height, bg))
        for j in range(F):
            times.append(math.floor(rng.uniform() * 300) / 299.0)
    elif name == "scaling":
        nt, nv = 8, 8
        for i in range(nt):
            for v in range(nv):
                a = 2 * math.pi * v / nv
                eye = 12.0 * np.array([math.cos(0.3) * math.sin(a), math.sin(0.3),
                                       math.cos(0.3) * math.cos(a)])
                cams.append(look_at(eye, (0, 0, 0), width, height, bg))
                times.append(i / 7.0)
        if n_frames is not None:
            cams, times = cams[:n_frames], times[:n_frames]
    else:
        raise KeyError(name)
    return cams, _f32(times)


def morton_order(means, bmin, bmax, bits: int = 10) -> np.ndarray:
    """Permutation that sorts points by the Z-order (Morton) code of their position quantised to
    2^bits cells per axis of the AABB (ties by original index).  A data-layout step of model load
    (SURVEY §8(d) "Model order"), not arithmetic of the method: every Gaussian keeps its values."""
    m = np.asarray(means, np.float64)
    lo, hi = np.asarray(bmin, np.float64), np.asarray(bmax, np.float64)
    u = np.clip((m - lo) / (hi - lo), 0.0, 1.0)
    q = np.minimum((u * (1 << bits)).astype(np.int64), (1 << bits) - 1)
    q = np.where(np.isfinite(m), q, 0)
    code = np.zeros(m.shape[0], np.int64)
    for bit in range(bits):
        for a in range(3):
            code |= ((q[:, a] >> bit) & 1) << (3 * bit + (2 - a))
    return np.lexsort((np.arange(m.shape[0]), code))


def make_scene(name: str, *, n: Optional[int] = None, width: Optional[int] = None,
               height: Optional[int] = None, n_frames: Optional[int] = None,
               seed: Optional[int] = None, order: str = "morton") -> Scene:
    """Build a BASELINE.json config (name in CONFIGS or ALIASES).

    Overrides (n, width, height, n_frames, seed) produce reduced variants of the
    same distributions for parity tests; the draw order is unchanged.
    order: "morton" (default) stores the Gaussians in Z-order of their canonical means over the
    field AABB, the layout a renderer gives a model at load time; "draw" keeps the
    draw order.  The stored order defines the Gaussian index (the sort tie-break, reading R14).
    """
    name = ALIASES.get(name, name)
    cfg = dict(CONFIGS[name])
    seed = cfg["seed"] if seed is None else seed
    n = cfg["n"] if n is None else n
    W = cfg["width"] if width is None else width
    H = cfg["height"] if height is None else height
    rng = np.random.default_rng(seed)
    deg = cfg["sh_degree"]
    K = (deg + 1) ** 2

    means = _draw_means(rng, name, n)
    log_scales = rng.normal(cfg["log_scale"][0], cfg["log_scale"][1], (n, 3))
    q = rng.normal(0.0, 1.0, (n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    opac = rng.normal(0.0, 1.5, n)
    sh = np.zeros((n, K, 3))
    sh[:, 0, :] = rng.normal(0.0, 0.5, (n, 3))
    if K > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.05, (n, K - 1, 3))

    feat, res, t_res = cfg["feat"], cfg["res"], cfg["t_res"]
    planes = []
    for R in res:
        ps = []
        for (a, b) in PLANE_AXES:
            na = R
            nb = t_res if b == 3 else R
            if b == 3:
                ps.append(_f32(1.0 + rng.normal(0.0, 0.1, (nb, na, feat))))
            else:
                ps.append(_f32(rng.uniform(0.1, 0.5, (nb, na, feat))))
        planes.append(ps)
    bmin, bmax = _aabb(name)
    fld = Field(feat=feat, res=list(res), t_res=t_res, bmin=_f32(bmin), bmax=_f32(bmax),
                planes=planes)

    Wm = cfg["width_mlp"]
    in_dim = feat * len(res)
    lim = 1.0 / math.sqrt(in_dim)
    w_d = rng.uniform(-lim, lim, (Wm, in_dim))
    b_d = rng.uniform(-lim, lim, Wm)
    w_x = rng.normal(0.0, 0.01, (3, Wm))
    w_r = rng.normal(0.0, 0.01, (4, Wm))
    w_s = rng.normal(0.0, 0.01, (3, Wm))
    mlp = MLP(w_d=_f32(w_d), b_d=_f32(b_d), w_x=_f32(w_x), b_x=np.zeros(3, np.float32),
              w_r=_f32(w_r), b_r=np.zeros(4, np.float32), w_s=_f32(w_s),
              b_s=np.zeros(3, np.float32))

    cams, times = _cameras_times(rng, name, W, H, cfg["bg"], n_frames)
    if order == "morton":
        perm = morton_order(means, bmin, bmax)
        means, log_scales, q, opac, sh = means[perm], log_scales[perm], q[perm], opac[perm], sh[perm]
    elif order != "draw":
        raise ValueError(f"unknown order {order!r}")
    return Scene(name=name, seed=seed, means=_f32(means), log_scales=_f32(log_scales),
                 quats=_f32(q), opacity_logits=_f32(opac), sh=_f32(sh), sh_degree=deg,
                 field=fld, mlp=mlp, cameras=cams, times=times)


# --------------------------------------------------------------------------
# Variants used by the parity protocol
# --------------------------------------------------------------------------
def with_heads(scene: Scene, sigma: float, seed: int = 1234, bias_sigma: float = 0.0) -> Scene:
    """Replace head weights by N(0, sigma) (sigma=0 -> exact zero heads).

    sigma=1 is the "stress set" of §8(c.5): |Delta| ~ O(0.1-1).
    """
    rng = np.random.default_rng(seed)
    m = scene.mlp
    W = m.width

    def draw(shape):
        return _f32(rng.normal(0.0, sigma, shape)) if sigma > 0 else np.zeros(shape, np.float32)

    def drawb(k):
        return _f32(rng.normal(0.0, bias_sigma, k)) if bias_sigma > 0 else np.zeros(k, np.float32)

    mlp = replace(m, w_x=draw((3, W)), w_r=draw((4, W)), w_s=draw((3, W)),
                  b_x=drawb(3), b_r=drawb(4), b_s=drawb(3))
    return replace(scene, mlp=mlp)


def with_colour_heads(scene: Scene, sigma_c: float, sigma_a: float, seed: int = 4321, colour: bool = True,
                      opacity: bool = True) -> Scene:
    """Add the colour / opacity decoders phi_C, phi_alpha of P:1232 (Table 5 variant): weights
    N(0, sigma), biases N(0, sigma / 2) (sigma = 0 -> exact zero heads)."""
    rng = np.random.default_rng(seed)
    m = scene.mlp
    W = m.width
    K3 = (scene.sh_degree + 1) ** 2 * 3

    def draw(shape, sg):
        return _f32(rng.normal(0.0, sg, shape)) if sg > 0 else np.zeros(shape, np.float32)

    kw = {}
    if colour:
        kw.update(w_c=draw((K3, W), sigma_c), b_c=draw(K3, sigma_c / 2))
    if opacity:
        kw.update(w_a=draw((1, W), sigma_a), b_a=draw(1, sigma_a / 2))
    return replace(scene, mlp=replace(m, **kw))


def with_max_opacity(scene: Scene, max_opacity: float) -> Scene:
    """Clip opacity logits at logit(max_opacity) (low-opacity variant, §8(c.2) step 15)."""
    lim = math.log(max_opacity / (1.0 - max_opacity))
    return replace(scene, opacity_logits=np.minimum(scene.opacity_logits, np.float32(lim)))

