#!/usr/bin/env python
"""bench.py — frames/s of the 4D-GS per-frame deform + render path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config dnerf] [--impl fgs|reference]

A STEP is one pass of the whole hot path over one batch of synthetic
input: for each of the config's F (time, view) frames, fgs_deform at its t and fgs_render at its
camera into its own image (one fgs_frames call through the C ABI).  Default workload: the D-NeRF-like
config (BASELINE.json configs[1]: 100k Gaussians, 800x800, SH 3, 20 frames per step).

Timing (rank-local, then max over ranks): W untimed warm-up steps; K timed steps, each bracketed by
CUDA events on the launching stream, with a 512 MiB buffer written between steps (outside the
events) to flush the 126 MB L2; barrier + torch.cuda.synchronize() on both sides of the region.
Under torchrun (N > 1) the config's F-frame batch is split across the ranks (frame_split: contiguous
chunks, no collective on the data path): value = F frames / max-over-ranks time ("scaling": "strong");
the ranks' images are gathered to rank 0 afterwards (untimed) and checked against a one-GPU render of the
whole batch.  --weak replicates the batch on every rank instead ("scaling": "weak").

Also reported: per-stage device times (library CUDA events), the roofline of the dominant kernel,
e2e through fgs_frames_host (pinned host buffers, copies inside the timed region), the launch
count, SM clocks sampled during the region, and the fp64 oracle timed on the host cores.
`--impl reference` times the oracle arm alone (rank 0; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "frames/s (deform+render) at 800x800, 100k Gaussians; Gaussians deformed/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}   # B200_PROFILING.md fallback


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["_source"] = "fallback (B200_PROFILING.md)"
    return d


def workload_desc(scene):
    f = scene.field
    heads = " + phi_C/phi_alpha decoders (P:1232)" if getattr(scene.mlp, "w_c", None) is not None else ""
    return (f"{scene.name}: {scene.n} Gaussians, {scene.cameras[0].width}x{scene.cameras[0].height}, "
            f"SH{scene.sh_degree}, HexPlane {'/'.join(map(str, f.res))} x t{f.t_res} h{f.feat}, "
            f"phi_d {scene.mlp.width}{heads}, {scene.n_frames} (t, view) frames per step")


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.idx)],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "samples": len(sm),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------------------ oracle (CPU) arm
# state shared with the oracle worker processes (fork start method: inherited, not pickled); every stage
# forks its pool after the state it needs is in place
_ORACLE = {}


def _oracle_task(task):
    """One unit of oracle work in a worker process (single-threaded BLAS):
    ("deform", t, lo, hi) -> G' rows; ("pre", lo, hi) -> preprocess dict of rows; ("blend", tiles) ->
    (flat pixel indices, image [3,P], final_T, n_contrib, flagged) of those tiles."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    import oracle
    from oracle import render as OR
    st = _ORACLE
    sc, cam = st["scene"], st["cam"]
    with threadpool_limits(1):
        if task[0] == "deform":
            return oracle.deform_ref(sc, task[1], begin=task[2], end=task[3])
        if task[0] == "pre":
            lo, hi = task[1], task[2]
            g = st["g"]
            return OR.preprocess_ref(g["means"][lo:hi], g["log_scales"][lo:hi], g["quats"][lo:hi],
                                     sc.opacity_logits[lo:hi], sc.sh[lo:hi], sc.sh_degree, cam)
        out = OR.render_ref(st["g"], sc.opacity_logits, sc.sh, sc.sh_degree, cam, tiles_subset=task[1],
                            pre=st["pre"], bins=st["bins"])
        m = np.isfinite(out["final_T"])
        return (np.flatnonzero(m), out["image"][:, m], out["final_T"][m], out["n_contrib"][m], out["flagged"][m])


def oracle_procs():
    try:
        return max(1, min(32, len(os.sched_getaffinity(0))))
    except Exception:
        return max(1, min(32, os.cpu_count() or 1))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_full_frame(scene, frame, procs, g_render=None):
    """The fp64 oracle on ONE FULL frame of `scene` (SURVEY 8(d) oracle timing (ii)): deform of all N
    Gaussians (a fork pool of `procs` single-BLAS-thread workers over contiguous chunks), preprocess of all
    N (chunks), binning (bin_ref, serial: one sort of all instances), blend of EVERY tile (the pool over
    tile chunks, longest lists spread round-robin).  Nothing is sampled or extrapolated; each stage's wall
    time includes forking its pool.  g_render: the G' to render (the GPU's fp32 G' for the parity summary,
    protocol P3); default the oracle's own deform output.  Returns a dict with the per-stage seconds and
    the oracle's outputs (deformed, pre, bins, image, final_T, n_contrib, flagged)."""
    import multiprocessing as mp

    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import render as OR
    P = procs
    N = scene.n
    cam = scene.cameras[frame]
    t = float(scene.times[frame])
    W, H = cam.width, cam.height
    ctx = mp.get_context("fork")
    _ORACLE.clear()
    _ORACLE.update(scene=scene, cam=cam)
    sec = {}
    # (1) deformation of all N
    t0 = time.perf_counter()
    edges = np.linspace(0, N, 4 * P + 1).astype(int)
    with ctx.Pool(P) as pool:
        parts = pool.map(_oracle_task, [("deform", t, int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a],
                         chunksize=1)
    deformed = {k: np.concatenate([q[k] for q in parts], axis=0) for k in parts[0]}
    sec["deform"] = time.perf_counter() - t0
    g = deformed if g_render is None else g_render
    _ORACLE["g"] = g
    # (2) preprocess of all N
    t0 = time.perf_counter()
    with ctx.Pool(P) as pool:
        parts = pool.map(_oracle_task, [("pre", int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a],
                         chunksize=1)
    pre = {k: np.concatenate([q[k] for q in parts], axis=0) for k in parts[0]}
    sec["preprocess"] = time.perf_counter() - t0
    # (3) binning: instances sorted by (tile, depth key, index), tile ranges
    t0 = time.perf_counter()
    with threadpool_limits(1):
        bins = OR.bin_ref(pre, cam)
    sec["binning"] = time.perf_counter() - t0
    _ORACLE.update(pre=pre, bins=bins)
    # (4) blend of every tile
    t0 = time.perf_counter()
    gx, gy = OR.tile_grid(W, H)
    lens = np.diff(bins[2], axis=1)[:, 0]
    order = np.argsort(-lens, kind="stable")
    n_chunks = min(gx * gy, 8 * P)
    chunks = [sorted(order[i::n_chunks].tolist()) for i in range(n_chunks)]
    img = np.full((3, H * W), np.nan)
    fT = np.full(H * W, np.nan)
    nc = np.full(H * W, -1, np.int64)
    fl = np.zeros(H * W, bool)
    with ctx.Pool(P) as pool:
        for idx, im, T, c, f in pool.imap_unordered(_oracle_task, [("blend", ch) for ch in chunks if ch]):
            img[:, idx] = im
            fT[idx] = T
            nc[idx] = c
            fl[idx] = f
    sec["blend"] = time.perf_counter() - t0
    _ORACLE.clear()
    return {"seconds": sum(sec.values()), "stages_s": sec, "deformed": deformed, "pre": pre, "bins": bins,
            "image": img.reshape(3, H, W), "final_T": fT.reshape(H, W), "n_contrib": nc.reshape(H, W),
            "flagged": fl.reshape(H, W), "procs": P}


def oracle_single_process(scene, frame, g, pre, bins, t_bin, n_def=2000, n_pre=20000, n_tiles=24, seed=0):
    """SURVEY 8(d) oracle timing (i): one process, one BLAS thread, on a bounded sample of the frame,
    scaled to the whole frame (marked extrapolated): deform of n_def Gaussians, preprocess of n_pre, the
    binning time of the full frame (it is serial anyway), blend of n_tiles random tiles."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    import oracle
    from oracle import render as OR
    N = scene.n
    cam = scene.cameras[frame]
    t = float(scene.times[frame])
    gx, gy = OR.tile_grid(cam.width, cam.height)
    rng = np.random.default_rng(seed)
    tiles = sorted(rng.choice(gx * gy, min(n_tiles, gx * gy), replace=False).tolist())
    nd, npre = min(n_def, N), min(n_pre, N)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        oracle.deform_ref(scene, t, begin=0, end=nd)
        t_def = (time.perf_counter() - t0) * N / max(nd, 1)
        t0 = time.perf_counter()
        OR.preprocess_ref(g["means"][:npre], g["log_scales"][:npre], g["quats"][:npre], scene.opacity_logits[:npre],
                          scene.sh[:npre], scene.sh_degree, cam)
        t_pre = (time.perf_counter() - t0) * N / max(npre, 1)
        t0 = time.perf_counter()
        OR.render_ref(g, scene.opacity_logits, scene.sh, scene.sh_degree, cam, tiles_subset=tiles, pre=pre, bins=bins)
        t_blend = (time.perf_counter() - t0) * (gx * gy) / len(tiles)
    frame_s = t_def + t_pre + t_bin + t_blend
    return {"frames_per_s": 1.0 / frame_s, "gaussians_deformed_per_s": N / t_def, "cores": 1,
            "extrapolated": True,
            "sample": f"1 process, 1 BLAS thread: deform of {nd}/{N} Gaussians, preprocess of {npre}/{N}, "
                      f"binning of the full frame, blend of {len(tiles)}/{gx * gy} random tiles, each scaled "
                      f"to the full frame"}


def run_reference(args, scene, rank):
    """The reference arm for this tier: the fp64 oracle, as it stands, on the host cores.  A step is ONE
    FULL frame of the workload (frames cycled through the batch), not a sample: value = frames / s."""
    if rank != 0:
        return
    P = oracle_procs()
    F = scene.n_frames
    for w in range(args.warmup):
        oracle_full_frame(scene, w % F, P)
    secs, t_defs = [], []
    for k in range(args.steps):
        r = oracle_full_frame(scene, k % F, P)
        secs.append(r["seconds"])
        t_defs.append(r["stages_s"]["deform"])
    total = sum(secs)
    value = args.steps / total
    sample = (f"1 full frame of {scene.name} per step (frames cycled through the {F}-frame batch): oracle deform "
              f"of all {scene.n} Gaussians, preprocess of all, binning, blend of every tile; fp64 numpy on {P} "
              f"host processes (1 BLAS thread each); not extrapolated")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_desc(scene), "frames_per_step": 1,
                   "parallelism": f"{P} host processes (oracle over Gaussian chunks and tiles)"},
        "gaussians_deformed_per_s": scene.n * len(t_defs) / sum(t_defs),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": P, "kind": "oracle", "sample": sample,
                         "extrapolated": False, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
STAGE_KERNELS = {"deform": ["deform_tc3_kernel"],
                 "preprocess": ["preprocess_kernel"], "blend": ["blend_kernel"],
                 "binning": ["tile_scan_kernel", "duplicate_kernel", "tile_sort_kernel",
                             "long_sort_kernel"]}


def ncu_traffic(scene, stage):
    """DRAM bytes per launch of a stage's kernel(s) from the committed ncu capture
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), if it was taken on this workload."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    if d.get("config") != scene.name or d.get("frames_per_launch") != scene.n_frames:
        return None
    ks = [d["kernels"][k]["dram_bytes_per_launch"] for k in STAGE_KERNELS.get(stage, []) if k in d["kernels"]]
    if not ks:
        return None
    return sum(ks) if stage == "binning" else ks[0]


def roofline_objects(scene, stage_ms, stage_launches, peaks, counts, sm_mhz, steps):
    """Algorithmic work per launch / measured launch time for each stage.  A stage may
    take several launches per step (render batches of > FGS_MAX_BATCH frames): the work of one launch
    is the step's work / launches per step, so achieved = step work / step time of the stage."""
    F = scene.n_frames
    N = scene.n
    K = (scene.sh_degree + 1) ** 2
    hbm = peaks["hbm_gbs"]
    clk = (sm_mhz or peaks.get("sm_max_mhz", 1965.0)) * 1e6
    sms = counts.get("sms", 148)
    fp32_peak = sms * 128 * clk / 1e12            # T inst/s (FFMA-class lanes)
    f = scene.field
    W = scene.mlp.width
    L = len(f.res)
    out = {}

    def avg_launch_s(stage):
        # per-step stage time; the F frames below are the step's (= launches per step x one launch's)
        return stage_ms.get(stage, 0.0) / 1e3 / max(steps, 1)

    # deform: bound by the on-chip gathers of the time lines: per Gaussian-frame
    # 3 temporal planes x L scales x 2 knots x h fp32 read from shared memory (the spatial product is
    # sampled once per batch and the MLP runs on the tensor core); peak = 128 B/clk/SM shared memory
    t = avg_launch_s("deform")
    if t > 0:
        by_def = 3 * L * 2 * f.feat * 4
        work = by_def * N * F / 1e9
        smem_peak = sms * 128 * clk / 1e9
        out["deform"] = {"bound": "smem", "achieved": work / t, "peak": smem_peak, "unit": "GB/s",
                         "frac": work / t / smem_peak, "traffic": None,
                         "algorithmic": f"{by_def} B of time-line reads per Gaussian-frame x {N}x{F}"}
    # preprocess: HBM bytes per Gaussian (read G' 40 + opacity 4 + SH 12K; write 72 B)
    by_pre = N * (44 + 12 * K + 72) * F
    t = avg_launch_s("preprocess")
    if t > 0:
        out["preprocess"] = {"bound": "hbm", "achieved": by_pre / t / 1e9, "peak": hbm, "unit": "GB/s",
                             "frac": by_pre / t / 1e9 / hbm, "traffic": None,
                             "algorithmic": f"{44 + 12 * K + 72} B per Gaussian-frame",
                             "limiter": "not HBM: the frame-minor grid serves the frame-invariant SH of all "
                                        "but the first frame from L2 (ncu DRAM bytes ~0.3x the algorithmic "
                                        "bytes); the kernel is issue-bound on L1 (l1tex ~75%), XU (~31%) and "
                                        "FP64 (~27%) work (profiles/r02_ncu_summary.md)"}
    # blend: 9 FP32 inst per evaluated pair + 4 per contributing pair
    E, C = counts.get("evaluated_per_frame"), counts.get("contrib_per_frame")
    t = avg_launch_s("blend")
    if t > 0 and E:
        work = (9 * E + 4 * C) * F / 1e12
        # C basis: the algorithmic minimum, as if only the contributing pairs were evaluated
        work_c = 13 * C * F / 1e12
        out["blend"] = {"bound": "alu", "achieved": work / t, "peak": fp32_peak, "unit": "Tinst/s",
                        "frac": work / t / fp32_peak, "traffic": None,
                        "algorithmic": f"9 inst x {E:.3g} evaluated + 4 x {C:.3g} contributing pairs per frame",
                        "achieved_C": work_c / t, "frac_C": work_c / t / fp32_peak,
                        "algorithmic_C": f"13 inst x {C:.3g} contributing pairs per frame (C basis)"}
    M = counts.get("instances_per_frame")
    t_sort = stage_ms.get("tile_scan", 0) + stage_ms.get("duplicate", 0) + stage_ms.get("tile_sort", 0)
    if t_sort > 0 and M:
        by = (16 * M + 16 * N) * F
        out["binning"] = {"bound": "hbm", "achieved": by / (t_sort / 1e3 / steps) / 1e9, "peak": hbm,
                          "unit": "GB/s", "frac": by / (t_sort / 1e3 / steps) / 1e9 / hbm, "traffic": None,
                          "algorithmic": "16 B per instance + 16 B per Gaussian (lower bound)"}
    for k, v in out.items():
        tr = ncu_traffic(scene, k)
        if tr is not None:
            v["traffic"] = tr
            v["traffic_unit"] = "DRAM bytes per launch (ncu --set full, profiles/ncu_traffic.json)"
    return out


def _debug_render(fgs, ds, cam, dstruct, cap, dev, W, H):
    """One untimed fgs_render_debug of a frame with every debug output (work counts, parity summary)."""
    import torch
    n = ds.n
    gx, gy = (W + 15) // 16, (H + 15) // 16
    t = {"radii": torch.zeros(n, dtype=torch.int32, device=dev), "rect": torch.zeros((n, 4), dtype=torch.int32, device=dev),
         "depth_key": torch.zeros(n, dtype=torch.int32, device=dev),
         "tiles_touched": torch.zeros(n, dtype=torch.int32, device=dev),
         "n_instances": torch.zeros(1, dtype=torch.int32, device=dev),
         "sorted_gid": torch.zeros(cap, dtype=torch.int32, device=dev),
         "ranges": torch.zeros((gx * gy, 2), dtype=torch.int32, device=dev),
         "final_T": torch.zeros((H, W), dtype=torch.float32, device=dev),
         "n_contrib": torch.zeros((H, W), dtype=torch.int32, device=dev),
         "n_evaluated": torch.zeros((H, W), dtype=torch.int32, device=dev),
         "blend_work": torch.zeros(2, dtype=torch.int64, device=dev)}
    aux = fgs.fgs_render_aux(**{k: v.data_ptr() for k, v in t.items()})
    ws1 = ds.alloc_workspace(1, cap)
    im = torch.empty((3, H, W), device=dev)
    fgs.fgs_render_debug(cam, dstruct, im, ws1, aux)
    fgs.fgs_render_status(ws1, 1)
    out = {k: v.cpu().numpy() for k, v in t.items()}
    out["image"] = im.cpu().numpy()
    return out


def parity_summary(scene, frame, g_gpu, dbg, orc):
    """SURVEY 8(c.5) protocol on one whole frame, GPU vs the fp64 oracle (untimed; reported in the line):
    deform max |err| over all N (oracle's own deform vs the GPU's G'); integer work bit-exact outside
    boundary Gaussians — radii, rects, tiles_touched, depth keys of all N, the ordered list of every tile —
    with the oracle fed the GPU's fp32 G' (P3); pixels over every pixel: PSNR, max |err| on pixels the
    oracle does not flag, and the flagged count."""
    import numpy as np
    pre = orc["pre"]
    n = scene.n
    derr = max(float(np.max(np.abs(g_gpu[k].astype(np.float64) - orc["deformed"][k]))) for k in orc["deformed"])
    keep = ~pre["boundary"]
    mism = {
        "radii": int(np.sum((dbg["radii"][:n] != pre["radius"]) & keep)),
        "rect": int(np.sum(np.any(dbg["rect"][:n] != pre["rect"], axis=1) & keep)),
        "tiles_touched": int(np.sum((dbg["tiles_touched"][:n] != pre["tiles_touched"]) & keep)),
        "depth_key": int(np.sum((dbg["depth_key"][:n].view(np.uint32) != pre["depth_key"]) & keep)),
    }
    _, o_gids, o_ranges = orc["bins"]
    bad = 0
    for tile in range(o_ranges.shape[0]):
        a = o_gids[o_ranges[tile, 0]:o_ranges[tile, 1]]
        b = dbg["sorted_gid"][dbg["ranges"][tile, 0]:dbg["ranges"][tile, 1]].astype(np.int64)
        if not np.array_equal(a[keep[a]], b[keep[b]]):
            bad += 1
    mism["tile_lists"] = bad
    img, ref, flag = dbg["image"].astype(np.float64), orc["image"], orc["flagged"]
    d = np.abs(img - ref)
    mse = float(np.mean(d ** 2))
    psnr = float("inf") if mse == 0 else 10 * math.log10(1.0 / mse)
    return {"frame": frame, "deform_max_abs_err": derr, "deform_tol": 1e-4, "integer_mismatches": mism,
            "boundary_gaussians": int(pre["boundary"].sum()), "pixels": int(flag.size), "psnr_db": psnr,
            "psnr_min_db": 60.0, "max_abs_err_unflagged": float(d[:, ~flag].max()), "pixel_tol": 2e-3,
            "max_abs_err_all": float(d.max()), "flagged_pixels": int(flag.sum()),
            "final_T_max_abs_err": float(np.nanmax(np.abs(dbg["final_T"] - orc["final_T"]))),
            "n_contrib_mismatch_unflagged": int(np.sum((dbg["n_contrib"] != orc["n_contrib"]) & ~flag)),
            "pass": bool(derr <= 1e-4 and all(v == 0 for v in mism.values()) and psnr >= 60.0
                         and float(d[:, ~flag].max()) <= 2e-3)}


def run_fgs(args, scene, rank, world, local_rank):
    import dataclasses

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2310_08528_b200 import build, fgs
    from paper_2310_08528_b200.sharding import frame_split, gather_frames

    build.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if args.radix is not None:
        fgs.fgs_set_tuning(fgs.FGS_TUNE_RADIX, args.radix)
    if args.radix_min_list is not None:
        fgs.fgs_set_tuning(fgs.FGS_TUNE_RADIX_MIN_LIST, args.radix_min_list)
    F_all = scene.n_frames
    # (e1) frame-batch split: the config's batch is cut across ranks (strong scaling); --weak gives every
    # rank its own copy of the whole batch instead
    split = not args.weak
    mine = frame_split(F_all, rank, world) if split else list(range(F_all))
    full_scene = scene
    scene = dataclasses.replace(scene, cameras=[scene.cameras[f] for f in mine],
                                times=np.asarray([scene.times[f] for f in mine], np.float32))
    ds = fgs.DeviceScene(scene, dev)
    F = scene.n_frames
    W, H = full_scene.cameras[0].width, full_scene.cameras[0].height
    outs, outs_t = ds.alloc_deformed(max(F, 1))     # keep the tensors alive (structs hold raw pointers)
    images = [torch.empty((3, H, W), dtype=torch.float32, device=dev) for _ in range(F)]
    cap = 16 * scene.n
    ws = ds.alloc_workspace(max(F, 1), cap)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)   # 512 MiB > 126 MB L2
    stream = torch.cuda.current_stream()

    def step_eager():
        if F:
            fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs[:F], images, ws)

    for _ in range(args.warmup):
        step_eager()
    if F:
        fgs.fgs_render_status(ws, F)
    graph = None
    launches_per_step = None
    if not args.no_graph and F:
        # one step captured in a CUDA graph: the timed steps replay it (same kernels, no launch gaps)
        graph = torch.cuda.CUDAGraph()
        l0 = fgs.fgs_launch_count()
        with torch.cuda.graph(graph):
            fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs[:F], images, ws,
                           stream=torch.cuda.current_stream())
        launches_per_step = fgs.fgs_launch_count() - l0
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()

    # work counts of this rank's frames (deterministic; one debug render per frame, untimed)
    counts = {"sms": torch.cuda.get_device_properties(dev).multi_processor_count}
    dbg0 = None
    if rank == 0 and F:
        Ev, Cv, Mv, Wv, Tv = [], [], [], [], []
        for fi in range(F):
            dbg = _debug_render(fgs, ds, ds.cams[fi], outs[fi] if _first_of_time(scene, fi) == fi
                                else outs[_first_of_time(scene, fi)], cap, dev, W, H)
            if fi == 0:
                dbg0 = dbg
            Ev.append(int(dbg["n_evaluated"].sum()))
            Cv.append(int(dbg["n_contrib"].sum()))
            Mv.append(int(dbg["n_instances"][0]))
            Wv.append(int(dbg["blend_work"][0]) * 32)
            Tv.append(int(dbg["blend_work"][1]))
        counts.update(evaluated_per_frame=float(np.mean(Ev)), contrib_per_frame=float(np.mean(Cv)),
                      instances_per_frame=float(np.mean(Mv)), blend_pixel_evals_per_frame=float(np.mean(Wv)),
                      blend_warp_tests_per_frame=float(np.mean(Tv)))

    def timed(run_step, profile):
        """K steps between CUDA events on the launching stream, L2 flushed between steps (outside the
        events); barrier + synchronize on both sides; returns (max-over-ranks ms, launches, stages)."""
        if profile:
            fgs.fgs_profile_enable(True)
            fgs.fgs_profile_read()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = fgs.fgs_launch_count()
        evs = []
        for _ in range(args.steps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run_step()
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        nl = fgs.fgs_launch_count() - l0
        if world > 1:
            dist.barrier()
        st = None
        if profile:
            st = fgs.fgs_profile_read()
            fgs.fgs_profile_enable(False)
        if F:
            fgs.fgs_render_status(ws, F)
        per = [a.elapsed_time(b) for a, b in evs]
        timed.per_step = per
        t_ms = sum(per)
        if world > 1:
            tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_ms = float(tt.item())
        return t_ms, nl, st

    # (1) eager steps with the library's per-stage CUDA events: the stage breakdown and the roofline
    #     launch durations; (2) the headline: the same step replayed from the CUDA graph.
    t_eager, launches_eager, stages = timed(step_eager, True)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if graph is not None:
        t_max, _, _ = timed(graph.replay, False)
        launches = launches_per_step * args.steps
    else:
        t_max, launches = timed(step_eager, False)[:2]
    per_step = sorted(timed.per_step)
    step_stats = {"median": statistics.median(per_step), "p10": per_step[int(0.1 * (len(per_step) - 1))],
                  "p90": per_step[int(round(0.9 * (len(per_step) - 1)))], "unit": "ms (this rank)"}
    clk = clocks.stop()
    # --tile-cull: the same step with FGS_TUNE_TILE_CULL = 1 (non-contributing (tile, Gaussian) pairs left
    # out of the lists; an opt-in knob, default off) timed the same way, its images compared bit for bit
    tile_cull = None
    if args.tile_cull and F and graph is not None:
        ref_imgs = [im.clone() for im in images]
        with fgs.tuning(fgs.FGS_TUNE_TILE_CULL, 1):
            for _ in range(args.warmup):
                step_eager()
            fgs.fgs_render_status(ws, F)
            t_e2, _, st2 = timed(step_eager, True)
            graph2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph2):
                fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs[:F], images, ws,
                               stream=torch.cuda.current_stream())
            torch.cuda.synchronize()
            for _ in range(args.warmup):
                graph2.replay()
            t2, _, _ = timed(graph2.replay, False)
        fps = F_all if split else F_all * world
        tile_cull = {"value": fps * args.steps / (t2 / 1e3), "unit": "frames/s", "ms_per_step": t2 / args.steps,
                     "value_eager": fps * args.steps / (t_e2 / 1e3),
                     "stages_ms_per_step": {k: v[0] / args.steps for k, v in st2.items()},
                     "images_identical": all(torch.equal(a, b) for a, b in zip(ref_imgs, images)),
                     "note": "FGS_TUNE_TILE_CULL = 1 (opt-in; the headline value above is with the default, 0)"}
        del graph2, ref_imgs
    frames_per_step = F_all if split else F_all * world
    value = frames_per_step * args.steps / (t_max / 1e3)
    value_eager = frames_per_step * args.steps / (t_eager / 1e3)
    deform_ms = stages["deform"][0]

    # ---- e2e through the C ABI with host (pinned) buffers ----
    e2e = None
    if not args.no_e2e:
        hs = fgs.HostScene(scene)
        himgs = [torch.empty((3, H, W), dtype=torch.float32).pin_memory() for _ in range(F)]
        nbytes = fgs.fgs_frames_host_workspace_bytes(hs.g, hs.field, hs.mlp, max(F, 1), W, H, cap)
        dws = torch.empty(nbytes, dtype=torch.uint8, device=dev)

        def step_host():
            if F:
                fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, himgs, dws)

        for _ in range(max(1, args.warmup)):
            step_host()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        eev = []
        for _ in range(args.steps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step_host()
            b.record(stream)
            eev.append((a, b))
        torch.cuda.synchronize()
        e_ms = sum(a.elapsed_time(b) for a, b in eev)
        if F:
            fgs.fgs_frames_host_status(hs.g, hs.field, hs.mlp, hs.cams, dws)   # no capacity overflow
        if world > 1:
            tt = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        # parity of the host path against the device path (same inputs -> same images)
        same = all(torch.equal(himgs[i], images[i].cpu()) for i in range(F))
        serial = frames_per_step * args.steps / (e_ms / 1e3)
        # Pipelined: the way a caller renders a stream of batches — two calls in flight on two streams,
        # each with its own device workspace and pinned image set (fgs.h: reentrant for distinct
        # workspaces), so step k+1's upload + deform + render overlap step k's image download.  Every
        # step still uploads the whole model from pinned host memory and downloads all its images; the
        # timed region is one event pair around all K steps (start before the first upload, end after
        # the last download).  No L2 flush: each step's inputs arrive from the host and the two
        # alternating workspaces (>= 2 x the batch's images) exceed the 126 MB L2.
        pipe = None
        if F and not args.no_e2e_pipeline:
            depth = max(2, args.e2e_depth)
            dws2 = [dws] + [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(depth - 1)]
            himgs2 = [himgs] + [[torch.empty((3, H, W), dtype=torch.float32).pin_memory() for _ in range(F)]
                                for _ in range(depth - 1)]
            lanes = [torch.cuda.Stream(device=dev) for _ in range(depth)]

            def run_pipe(k_steps):
                for ln in lanes:
                    ln.wait_stream(stream)
                for k in range(k_steps):
                    j = k % depth
                    fgs.fgs_frames_host(hs.g, hs.field, hs.mlp, hs.times, hs.cams, himgs2[j], dws2[j],
                                        stream=lanes[j])
                for ln in lanes:
                    stream.wait_stream(ln)

            run_pipe(max(depth, args.warmup))
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            pa = torch.cuda.Event(enable_timing=True)
            pb = torch.cuda.Event(enable_timing=True)
            pa.record(stream)
            run_pipe(args.steps)
            pb.record(stream)
            torch.cuda.synchronize()
            p_ms = pa.elapsed_time(pb)
            for j in range(depth):
                fgs.fgs_frames_host_status(hs.g, hs.field, hs.mlp, hs.cams, dws2[j], stream=lanes[j])
            if world > 1:
                tt = torch.tensor([p_ms], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                p_ms = float(tt.item())
            same = same and all(torch.equal(himgs2[j][i], himgs[i]) for j in range(1, depth) for i in range(F))
            pipe = {"value": frames_per_step * args.steps / (p_ms / 1e3), "depth": depth, "ms_per_step": p_ms / args.steps}
            del dws2, himgs2
        e2e = {"value": pipe["value"] if pipe else serial, "unit": "frames/s",
               "h2d_bytes_per_step": hs.h2d_bytes() + F * 4, "d2h_bytes_per_step": F * 3 * H * W * 4,
               "api": "fgs_frames_host (pinned host model in, host images out)", "matches_device_path": same,
               "serial_value": serial,
               "mode": ("%d fgs_frames_host calls in flight (one stream and one workspace each): one event pair around "
                        "all K steps, every step's copies inside it" % pipe["depth"]) if pipe else
                       "one call at a time, per-step events, L2 flushed between steps",
               "serial_note": "serial_value: one call at a time (the next upload starts after the last download)"}
        if pipe:
            e2e["pipeline_ms_per_step"] = pipe["ms_per_step"]
            e2e["l2"] = ("pipelined: no flush (every step's inputs arrive from pinned host memory and the alternating "
                         "device workspaces, %.0f MB each, exceed the 126 MB L2); serial_value: flushed between steps"
                         % (nbytes / 1e6))
        del dws

    # ---- (e1) untimed: the ranks' images gathered to rank 0 == a single-GPU render of the whole batch ----
    split_check = None
    if world > 1 and split:
        got = gather_frames(images, F_all, rank, world)
        if rank == 0:
            fds = fgs.DeviceScene(full_scene, dev)
            fo, _ = fds.alloc_deformed(F_all)
            fimgs = [torch.empty((3, H, W), dtype=torch.float32, device=dev) for _ in range(F_all)]
            fws = fds.alloc_workspace(F_all, cap)
            fgs.fgs_frames(fds.g, fds.field, fds.mlp, fds.times, fds.cams, fo, fimgs, fws)
            fgs.fgs_render_status(fws, F_all)
            split_check = {"frames_gathered": len(got),
                           "bit_identical_to_one_gpu_batch": all(torch.equal(a, b) for a, b in zip(got, fimgs))}
            del fws

    if rank != 0:
        return
    peaks = load_peaks()
    steps = args.steps
    stage_ms = {k: v[0] for k, v in stages.items()}
    stage_launches = {k: v[1] for k, v in stages.items()}
    roof = roofline_objects(scene, stage_ms, stage_launches, peaks, counts, clk.get("sm_mhz"), steps)
    # dominant kernel = largest share of the step
    dom = max(roof, key=lambda k: stage_ms.get(k, 0.0) if k != "binning" else 0.0) if roof else None
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": t_max / steps, "higher_is_better": True,
        "scaling": "strong" if split else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_desc(full_scene), "frames_per_step": frames_per_step,
                   "n_gaussians": scene.n, "image": f"{W}x{H}",
                   "l2": "flushed between steps (512 MiB write outside the events)",
                   "parallelism": (f"frame-batch split x{world}: rank r renders frames {{frame_split(F, r, {world})}} "
                                   f"of the {F_all}-frame batch (rank 0: {len(mine)})") if split else
                                  f"replicated x{world} (--weak: each rank its own {F_all}-frame batch)",
                   "max_instances_per_frame": cap,
                   "timed": "CUDA-graph replay of one fgs_frames step" if graph is not None else "eager fgs_frames"},
        "value_eager": value_eager,
        "step_ms": step_stats,
        "gaussians_deformed_per_s": scene.n * frames_per_step * steps / (t_max / 1e3),
        "gaussians_deformed_per_s_deform_stage": scene.n * F * steps / (deform_ms / 1e3) if deform_ms else None,
        "stages_ms_per_step": {k: v / steps for k, v in stage_ms.items()},
        "stages_note": "rank 0's per-stage library CUDA events over the eager timed steps (value_eager); the "
                       "graph replays the same kernels",
        "work_per_frame": {k: v for k, v in counts.items() if k != "sms"},
        "roofline": dict(roof[dom], kernel=dom) if dom else None,
        "roofline_stages": roof,
        "peaks": {"source": peaks["_source"], "hbm_gbs": peaks.get("hbm_gbs"),
                  "fp32_note": "FP32 lane peak = SMs x 128 x median SM clock under load"},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / steps,
        "clocks": clk,
        "e2e": e2e,
    }
    if tile_cull is not None:
        line["tile_cull"] = tile_cull
    if split_check is not None:
        line["frame_split_check"] = split_check
    if not args.no_cpu_baseline and F:
        # the oracle on one FULL frame (rank 0's first frame), rendering the GPU's fp32 G' (protocol P3) so
        # the same run gives the whole-frame parity summary; its own deform output gives the deform error
        P = oracle_procs()
        g_gpu = {k: v.cpu().numpy() for k, v in outs_t[0].items()}
        orc = oracle_full_frame(scene, 0, P, g_render=g_gpu)
        line["parity"] = parity_summary(scene, 0, g_gpu, dbg0, orc)
        single = oracle_single_process(scene, 0, g_gpu, orc["pre"], orc["bins"], orc["stages_s"]["binning"])
        line["cpu_baseline"] = {
            "value": 1.0 / orc["seconds"], "unit": "frames/s", "cores": P, "kind": "oracle",
            "sample": (f"1 full frame of {scene.name} (frame {mine[0]} of the batch): oracle deform of all "
                       f"{scene.n} Gaussians, preprocess of all, binning, blend of every tile; fp64 numpy on "
                       f"{P} host processes (1 BLAS thread each)"),
            "extrapolated": False, "stages_s": orc["stages_s"],
            "gaussians_deformed_per_s": scene.n / orc["stages_s"]["deform"],
            "single_process": single, "cpu_model": cpu_model()}
    print(json.dumps(line), flush=True)


def _first_of_time(scene, f):
    """Index of the first frame of `scene` with frame f's time (fgs_frames deforms each time once and
    the frames sharing it render from that frame's G')."""
    import numpy as np
    tb = np.float32(scene.times[f]).tobytes()
    return next(i for i in range(scene.n_frames) if np.float32(scene.times[i]).tobytes() == tb)


def run_shard(args, scene, rank, world, local_rank):
    """(e2) SURVEY §8(e2): the batch is (time k, view v) frames; views are split across ranks, every rank
    deforms 1/world of the Gaussians at each distinct time and all-gathers X', r', s' (NCCL), overlapped
    with the render of the previous time.  value = all frames of the batch / max-over-ranks time
    ("scaling": "strong": the batch is fixed as N grows)."""
    import torch
    import torch.distributed as dist

    from paper_2310_08528_b200 import build, fgs
    from paper_2310_08528_b200.sharding import ShardedDeform, sharded_frames

    build.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ds = fgs.DeviceScene(scene, dev)
    ts_all = [float(t) for t in scene.times]
    uniq = sorted(set(ts_all), key=ts_all.index)
    frames_of = {t: [f for f in range(scene.n_frames) if ts_all[f] == t] for t in uniq}
    # views split across ranks: rank r renders the frames whose index within their time is in its slice
    from paper_2310_08528_b200.sharding import frame_split
    views = []
    mine = []
    for t in uniq:
        fs = frames_of[t]
        sel = [fs[i] for i in frame_split(len(fs), rank, world)]
        views.append([(ds.cams[f], j) for j, f in enumerate(sel, start=len(mine))])
        mine.extend(sel)
    W, H = scene.cameras[0].width, scene.cameras[0].height
    images = [torch.empty((3, H, W), dtype=torch.float32, device=dev) for _ in mine]
    per_t = max(len(v) for v in views)
    ws = ds.alloc_workspace(max(per_t, 1), 16 * scene.n)
    fused = getattr(args, "fused", False)
    if fused and not (dist.is_available() and dist.is_initialized()):
        # symmetric memory needs a process group: a one-rank NCCL group on 127.0.0.1
        import socket
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=dev)
    sd = ShardedDeform(scene.n, world, rank, dev, n_slots=2, fused=fused)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        sharded_frames(ds, sd, uniq, views, images, ws)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    launches0 = fgs.fgs_launch_count()
    evs = []
    for _ in range(args.steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    launches = fgs.fgs_launch_count() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    t_max = t_ms
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    if rank != 0:
        return
    F = scene.n_frames
    line = {
        "metric": METRIC, "value": F * args.steps / (t_max / 1e3), "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_desc(scene), "frames_per_step": F, "distinct_times": len(uniq),
                   "parallelism": f"views split x{world}; deformation sharded by Gaussian + "
                                  + ("peer stores from the deform epilogue into symmetric memory + barrier (e2 fused)"
                                     if fused else "all_gather (e2)"),
                   "l2": "flushed between steps (512 MiB write outside the events)"},
        "gaussians_deformed_per_s": scene.n * len(uniq) * args.steps / (t_max / 1e3),
        "gpu_launches": launches, "clocks": clk, "mode": "shard-fused" if fused else "shard",
    }
    print(json.dumps(line), flush=True)


def run_train(args, scene, rank, world, local_rank):
    """SURVEY §8(f) rank 4 (§4.3): the training side measured.  A step = every frame of
    the config's batch trained once: fgs_deform at its t, fgs_render, fgs_l1_loss against a synthetic
    target, fgs_render_backward, fgs_deform_backward (field gradients accumulated over the batch), plus
    one fgs_tv_loss.  Replayed from a CUDA graph; per-stage times from a separate eager pass.  The
    autograd oracle (oracle/backward.py) is timed beside it on a bounded sample (cpu_baseline)."""
    import numpy as np
    import torch

    from paper_2310_08528_b200 import build, fgs

    build.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ds = fgs.DeviceScene(scene, dev)
    F = scene.n_frames
    W, H = scene.cameras[0].width, scene.cameras[0].height
    outs, _ = ds.alloc_deformed(1)
    img = torch.empty((3, H, W), device=dev)
    dimg = torch.empty_like(img)
    gen = torch.Generator(device="cpu").manual_seed(5)
    targets = [torch.rand((3, H, W), generator=gen).to(dev) for _ in range(F)]
    ws = ds.alloc_workspace(1, 16 * scene.n)
    part = torch.empty(fgs.FGS_LOSS_PARTIALS, dtype=torch.float64, device=dev)
    l1 = torch.empty(1, device=dev)
    tv = torch.empty(1, device=dev)
    dg, _ = ds.alloc_gaussian_grads()
    dc, _ = ds.alloc_gaussian_grads()
    df, _ = ds.alloc_field_grads()
    rs = torch.empty(fgs.fgs_render_backward_scratch_bytes(scene.n), dtype=torch.uint8, device=dev)
    dsb = torch.empty(fgs.fgs_deform_backward_scratch_bytes(ds.field, ds.mlp), dtype=torch.uint8, device=dev)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    stage_names = ("deform", "render", "l1_loss", "render_backward", "deform_backward", "tv_loss")

    def frame_calls(f):
        t = ds.times[f]
        return (lambda: fgs.fgs_deform(ds.g, ds.field, ds.mlp, t, outs[0]),
                lambda: fgs.fgs_render(ds.cams[f], outs[0], img, ws),
                lambda: fgs.fgs_l1_loss(img, targets[f], dimg, part, l1),
                lambda: fgs.fgs_render_backward(ds.cams[f], outs[0], img, dimg, ws, rs, dg),
                lambda: fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, t, dg, dc, df, dsb))

    def step():
        for f in range(F):
            for c in frame_calls(f):
                c()
        fgs.fgs_tv_loss(ds.field, 0.01, df, part, tv)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # per-stage times (eager, events around each call)
    ms = {k: 0.0 for k in stage_names}
    for f in range(F):
        for name, c in zip(stage_names, frame_calls(f)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            c()
            b.record(stream)
            torch.cuda.synchronize()
            ms[name] += a.elapsed_time(b)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fgs.fgs_tv_loss(ds.field, 0.01, df, part, tv)
    b.record(stream)
    torch.cuda.synchronize()
    ms["tv_loss"] = a.elapsed_time(b)
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        step()
        side.synchronize()
        l0 = fgs.fgs_launch_count()
        with torch.cuda.graph(graph, stream=side):
            step()
        launches_per_step = fgs.fgs_launch_count() - l0
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    evs = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        graph.replay()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    clk = clocks.stop()
    t_ms = sum(x.elapsed_time(y) for x, y in evs)
    fgs.fgs_render_status(ws, 1)
    line = {
        "metric": "training frames/s (deform + render + L1/TV loss + backward) at 800x800, 100k Gaussians",
        "value": F * args.steps / (t_ms / 1e3), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (random target images)", "mode": "train",
        "config": {"workload": workload_desc(scene), "frames_per_step": F,
                   "l2": "flushed between steps (512 MiB write outside the events)",
                   "timed": "CUDA-graph replay of one training step", "tv_weight": 0.01},
        "stages_ms_per_frame": {k: v / (F if k != "tv_loss" else 1) for k, v in ms.items()},
        "gpu_launches": launches_per_step * args.steps, "gpu_launches_per_step": launches_per_step,
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        # the autograd oracle on a bounded sample of one frame: the splat backward of 8 random tiles (with
        # their Gaussians) and the deformation backward of 2000 Gaussians, scaled to the whole frame
        from threadpoolctl import threadpool_limits

        import oracle
        from oracle import backward as OB
        from oracle import render as OR
        cam = scene.cameras[0]
        t = float(scene.times[0])
        G = oracle.deform_ref(scene, t)
        pre = OR.preprocess_ref(G["means"], G["log_scales"], G["quats"], scene.opacity_logits, scene.sh,
                                scene.sh_degree, cam)
        gx, gy = OR.tile_grid(W, H)
        rng = np.random.default_rng(0)
        tiles = rng.choice(gx * gy, 8, replace=False)
        sel = np.unique(np.concatenate([OR.tile_list_ref(pre, cam, int(tl)) for tl in tiles]))
        with threadpool_limits(1):
            t0 = time.perf_counter()
            sub = {k: v[sel] for k, v in G.items()}
            OB.render_grads_ref(sub, scene.opacity_logits[sel], scene.sh[sel], scene.sh_degree, cam,
                                np.random.default_rng(1).normal(size=(3, H, W)))
            t_r = time.perf_counter() - t0
            nd = 2000
            sc = dataclasses_replace_rows(scene, nd)
            t0 = time.perf_counter()
            OB.deform_grads_ref(sc, t, {k: np.ones_like(v[:nd]) for k, v in G.items()})
            t_d = (time.perf_counter() - t0) * scene.n / nd
        # the render sample covers every tile (all pixels, the sample's Gaussians): scale by the share of
        # list entries those 8 tiles hold
        lens = np.array([len(OR.tile_list_ref(pre, cam, int(tl))) for tl in tiles])
        bins = OR.bin_ref(pre, cam)[2]
        share = lens.sum() / max(1, int(np.diff(bins, axis=1).sum()))
        frame_s = t_r / max(share, 1e-9) + t_d
        line["cpu_baseline"] = {"value": 1.0 / frame_s, "unit": "training frames/s", "cores": 1, "kind": "oracle",
                                "extrapolated": True,
                                "sample": (f"1 process: autograd splat backward of the {sel.size} Gaussians of 8 random "
                                           f"tiles over the whole image (scaled by those tiles' {share:.4f} share of "
                                           f"the list entries) + deformation backward of {nd}/{scene.n} Gaussians "
                                           f"(scaled); fp64 PyTorch CPU autograd"),
                                "cpu_model": cpu_model()}
    print(json.dumps(line), flush=True)


def dataclasses_replace_rows(scene, n):
    import dataclasses
    return dataclasses.replace(scene, means=scene.means[:n], log_scales=scene.log_scales[:n],
                               quats=scene.quats[:n], opacity_logits=scene.opacity_logits[:n], sh=scene.sh[:n])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fgs", choices=["fgs", "reference"])
    ap.add_argument("--config", default="dnerf")
    ap.add_argument("--frames", type=int, default=None)
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager fgs_frames calls instead of replaying the step captured in a CUDA graph")
    ap.add_argument("--colour-heads", action="store_true",
                    help="P:1232 variant: add the colour / opacity decoders phi_C, phi_alpha (SURVEY 8(f) rank 2)")
    ap.add_argument("--n", type=int, default=None,
                    help="override the number of Gaussians (SURVEY 8(f) N-sweep: same distributions)")
    ap.add_argument("--radix", type=int, default=None, choices=[0, 1, 2],
                    help="FGS_TUNE_RADIX: 0 per-tile sorts, 1 auto (library default), 2 radix binning path")
    ap.add_argument("--radix-min-list", type=int, default=None, help="FGS_TUNE_RADIX_MIN_LIST (auto threshold)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tile-cull", action="store_true",
                    help="also time the step with FGS_TUNE_TILE_CULL = 1 (adds a tile_cull object to the line)")
    ap.add_argument("--e2e-depth", type=int, default=2, help="fgs_frames_host calls in flight in the pipelined e2e")
    ap.add_argument("--no-e2e-pipeline", action="store_true",
                    help="e2e: one fgs_frames_host call at a time only (no two-in-flight pipelined measurement)")
    ap.add_argument("--weak", action="store_true",
                    help="frames mode under torchrun: every rank renders its own copy of the whole batch (weak "
                         "scaling) instead of its frame_split chunk of it (strong scaling, the default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="frames", choices=["frames", "shard", "train"],
                    help="frames: the frame batch split across ranks (e1); shard: multi-view batch, views "
                         "split across ranks, deformation sharded by Gaussian + NCCL all-gather (e2); train: "
                         "the training side (forward + L1/TV loss + backward, SURVEY 8(f) rank 4)")
    ap.add_argument("--fused", action="store_true",
                    help="with --mode shard: the deform epilogue stores every rank's copy into symmetric "
                         "memory (fgs_deform_range_peers) instead of the NCCL all-gather (SURVEY 8(e2) fused)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "fgs":
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2310_08528_b200.inputs import make_scene
    scene = make_scene(args.config, n_frames=args.frames, n=args.n)
    if args.colour_heads:
        from paper_2310_08528_b200.inputs import with_colour_heads
        scene = with_colour_heads(scene, 0.05, 0.05)

    if args.impl == "reference":
        run_reference(args, scene, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.mode == "shard":
            run_shard(args, scene, rank, world, local_rank)
        elif args.mode == "train":
            run_train(args, scene, rank, world, local_rank)
        else:
            run_fgs(args, scene, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
