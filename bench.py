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
Under torchrun (N > 1) every rank renders its own F-frame batch (frame-batch split, no collective):
value = all frames of all ranks / max-over-ranks time ("scaling": "weak").

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
# state shared with the oracle worker processes (fork start method: inherited, not pickled)
_ORACLE = {}


def _oracle_task(task):
    """One unit of oracle work in a worker process (single-threaded BLAS): ("deform", t, lo, hi),
    ("pre", lo, hi) or ("blend", tiles)."""
    from threadpoolctl import threadpool_limits

    import oracle
    from oracle import render as OR
    sc, cam = _ORACLE["scene"], _ORACLE["cam"]
    t0 = time.perf_counter()
    with threadpool_limits(1):
        if task[0] == "deform":
            oracle.deform_ref(sc, task[1], begin=task[2], end=task[3])
        elif task[0] == "pre":
            lo, hi = task[1], task[2]
            OR.preprocess_ref(sc.means[lo:hi], sc.log_scales[lo:hi], sc.quats[lo:hi], sc.opacity_logits[lo:hi],
                              sc.sh[lo:hi], sc.sh_degree, cam)
        else:
            d = {"means": sc.means, "log_scales": sc.log_scales, "quats": sc.quats}
            OR.render_ref(d, sc.opacity_logits, sc.sh, sc.sh_degree, cam, tiles_subset=task[1],
                          pre=_ORACLE["pre"], full_bins=False)
    return time.perf_counter() - t0


def oracle_procs():
    try:
        return max(1, min(32, len(os.sched_getaffinity(0))))
    except Exception:
        return max(1, min(32, os.cpu_count() or 1))


def oracle_sample(scene, frame, n_tiles, rng_seed=0, deform_per_proc=2_000, procs=None):
    """Time the fp64 oracle on a bounded sample of one frame on `procs` host cores and extrapolate the
    frame time (SURVEY 8(d) oracle timing (ii): a process pool over Gaussian chunks and tiles).

    Sample: deform of procs x deform_per_proc Gaussians (scaled to N), preprocess of all N (chunks),
    binning (bin_ref, serial), blend of n_tiles random tiles (scaled to all tiles).  Each stage's wall
    time is measured around its pool map.  Returns (frame_seconds, deform_seconds_per_N, desc, procs).
    """
    import multiprocessing as mp

    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import render as OR

    P = procs or oracle_procs()
    N = scene.n
    cam = scene.cameras[frame]
    t = float(scene.times[frame])
    _ORACLE.update(scene=scene, cam=cam, pre=None)
    with threadpool_limits(1):
        pre = OR.preprocess_ref(scene.means, scene.log_scales, scene.quats, scene.opacity_logits, scene.sh,
                                scene.sh_degree, cam)                  # the blend's input (not timed)
    _ORACLE["pre"] = pre
    gx, gy = OR.tile_grid(cam.width, cam.height)
    rng = np.random.default_rng(rng_seed)
    tiles = sorted(rng.choice(gx * gy, min(n_tiles, gx * gy), replace=False).tolist())
    sub = min(N, P * deform_per_proc)
    ctx = mp.get_context("fork")
    with ctx.Pool(P) as pool:
        pool.map(_oracle_task, [("pre", 0, 1)] * P)          # start the workers (not timed)

        def timed_map(tasks):
            t0 = time.perf_counter()
            pool.map(_oracle_task, tasks)
            return time.perf_counter() - t0
        edges = np.linspace(0, sub, P + 1).astype(int)
        t_def = timed_map([("deform", t, int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a])
        t_def *= N / max(sub, 1)
        edges = np.linspace(0, N, P + 1).astype(int)
        t_pre = timed_map([("pre", int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a])
        chunks = [tiles[i::P] for i in range(P) if tiles[i::P]]
        t_blend = timed_map([("blend", c) for c in chunks]) * (gx * gy) / len(tiles)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        OR.bin_ref(pre, cam)
        t_bin = time.perf_counter() - t0
    frame_s = t_def + t_pre + t_bin + t_blend
    desc = (f"1 frame of {scene.name} on {P} host processes: oracle deform of {sub}/{N} Gaussians "
            f"(x{N / max(sub, 1):.0f}), preprocess of all {N}, binning (serial), blend of {len(tiles)}/{gx * gy} "
            f"random tiles (x{gx * gy / len(tiles):.1f}) of the canonical G; fp64 numpy, 1 BLAS thread per process")
    return frame_s, t_def, desc, P


def run_reference(args, scene, rank):
    if rank != 0:
        return
    P = oracle_procs()
    n_tiles = 24 * P
    for w in range(args.warmup):
        oracle_sample(scene, w % scene.n_frames, n_tiles, rng_seed=w, procs=P)
    frame_s = []
    t_defs = []
    for k in range(args.steps):
        fs, td, desc, _ = oracle_sample(scene, k % scene.n_frames, n_tiles, rng_seed=100 + k, procs=P)
        frame_s.append(fs)
        t_defs.append(td)
    F = scene.n_frames
    step_s = [F * s for s in frame_s]
    total = sum(step_s)
    value = F * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_desc(scene), "frames_per_step": F, "parallelism": f"{P} host processes (oracle over Gaussian chunks and tiles)"},
        "gaussians_deformed_per_s": scene.n * len(t_defs) / sum(t_defs),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": P, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
STAGE_KERNELS = {"deform": ["deform_tc3_kernel", "deform_tc2_kernel", "deform_tc_kernel"],
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
                             "algorithmic": f"{44 + 12 * K + 72} B per Gaussian-frame"}
    # blend: 9 FP32 inst per evaluated pair + 4 per contributing pair
    E, C = counts.get("evaluated_per_frame"), counts.get("contrib_per_frame")
    t = avg_launch_s("blend")
    if t > 0 and E:
        work = (9 * E + 4 * C) * F / 1e12
        out["blend"] = {"bound": "alu", "achieved": work / t, "peak": fp32_peak, "unit": "Tinst/s",
                        "frac": work / t / fp32_peak, "traffic": None,
                        "algorithmic": f"9 inst x {E:.3g} evaluated + 4 x {C:.3g} contributing pairs per frame"}
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


def run_fgs(args, scene, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2310_08528_b200 import build, fgs

    build.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ds = fgs.DeviceScene(scene, dev)
    F = scene.n_frames
    W, H = scene.cameras[0].width, scene.cameras[0].height
    outs, outs_t = ds.alloc_deformed(F)     # keep the tensors alive (structs hold raw pointers)
    images = [torch.empty((3, H, W), dtype=torch.float32, device=dev) for _ in range(F)]
    cap = 16 * scene.n
    ws = ds.alloc_workspace(F, cap)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)   # 512 MiB > 126 MB L2
    stream = torch.cuda.current_stream()

    def step_eager():
        fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, images, ws)

    for _ in range(args.warmup):
        step_eager()
    fgs.fgs_render_status(ws, F)
    graph = None
    launches_per_step = None
    if not args.no_graph:
        # one step captured in a CUDA graph: the timed steps replay it (same kernels, no launch gaps)
        graph = torch.cuda.CUDAGraph()
        l0 = fgs.fgs_launch_count()
        with torch.cuda.graph(graph):
            fgs.fgs_frames(ds.g, ds.field, ds.mlp, ds.times, ds.cams, outs, images, ws,
                           stream=torch.cuda.current_stream())
        launches_per_step = fgs.fgs_launch_count() - l0
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()

    # work counts of this workload (deterministic; one debug render per frame, untimed)
    counts = {"sms": torch.cuda.get_device_properties(dev).multi_processor_count}
    if rank == 0:
        Ev, Cv, Mv, Wv, Tv = [], [], [], [], []
        for fi in range(F):
            ne = torch.zeros((H, W), dtype=torch.int32, device=dev)
            nc = torch.zeros((H, W), dtype=torch.int32, device=dev)
            ni = torch.zeros(1, dtype=torch.int32, device=dev)
            bw = torch.zeros(2, dtype=torch.int64, device=dev)
            aux = fgs.fgs_render_aux(n_evaluated=ne.data_ptr(), n_contrib=nc.data_ptr(), n_instances=ni.data_ptr(),
                                     blend_work=bw.data_ptr())
            ws1 = ds.alloc_workspace(1, cap)
            im = torch.empty((3, H, W), device=dev)
            fgs.fgs_render_debug(ds.cams[fi], outs[fi], im, ws1, aux)
            torch.cuda.synchronize()
            Ev.append(int(ne.sum()))
            Cv.append(int(nc.sum()))
            Mv.append(int(ni[0]))
            Wv.append(int(bw[0]) * 32)
            Tv.append(int(bw[1]))
            del ws1
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
        t_max, launches = t_eager, launches_eager
    per_step = sorted(timed.per_step)
    step_stats = {"median": statistics.median(per_step), "p10": per_step[int(0.1 * (len(per_step) - 1))],
                  "p90": per_step[int(round(0.9 * (len(per_step) - 1)))], "unit": "ms (this rank)"}
    clk = clocks.stop()
    value = F * args.steps * world / (t_max / 1e3)
    value_eager = F * args.steps * world / (t_eager / 1e3)
    deform_ms = stages["deform"][0]

    # ---- e2e through the C ABI with host (pinned) buffers ----
    e2e = None
    if not args.no_e2e:
        hs = fgs.HostScene(scene)
        himgs = [torch.empty((3, H, W), dtype=torch.float32).pin_memory() for _ in range(F)]
        nbytes = fgs.fgs_frames_host_workspace_bytes(hs.g, hs.field, hs.mlp, F, W, H, cap)
        dws = torch.empty(nbytes, dtype=torch.uint8, device=dev)

        def step_host():
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
        if world > 1:
            tt = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        # parity of the host path against the device path (same inputs -> same images)
        same = all(torch.equal(himgs[i], images[i].cpu()) for i in range(F))
        e2e = {"value": F * args.steps * world / (e_ms / 1e3), "unit": "frames/s",
               "h2d_bytes_per_step": hs.h2d_bytes() + F * 4, "d2h_bytes_per_step": F * 3 * H * W * 4,
               "api": "fgs_frames_host (pinned host model in, host images out)", "matches_device_path": same}
        del dws

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
        "warmup": args.warmup, "ms_per_step": t_max / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_desc(scene), "frames_per_step": F, "n_gaussians": scene.n,
                   "image": f"{W}x{H}", "l2": "flushed between steps (512 MiB write outside the events)",
                   "parallelism": f"frame-split x{world} (each rank its own {F}-frame batch)",
                   "max_instances_per_frame": cap,
                   "timed": "CUDA-graph replay of one fgs_frames step" if graph is not None else "eager fgs_frames"},
        "value_eager": value_eager,
        "step_ms": step_stats,
        "gaussians_deformed_per_s": scene.n * F * steps * world / (t_max / 1e3),
        "gaussians_deformed_per_s_deform_stage": scene.n * F * steps / (deform_ms / 1e3) if deform_ms else None,
        "stages_ms_per_step": {k: v / steps for k, v in stage_ms.items()},
        "stages_note": "per-stage library CUDA events over the eager timed steps (value_eager); the graph "
                       "replays the same kernels",
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
    if not args.no_cpu_baseline and world >= 1:
        P = oracle_procs()
        fs, td, desc, P = oracle_sample(scene, 0, n_tiles=24 * P, procs=P)
        line["cpu_baseline"] = {"value": 1.0 / fs, "unit": "frames/s", "cores": P, "kind": "oracle",
                                "sample": desc, "gaussians_deformed_per_s": scene.n / td}
    print(json.dumps(line), flush=True)


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
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="frames", choices=["frames", "shard"],
                    help="frames: every rank renders its own frame batch (e1); shard: multi-view batch, views "
                         "split across ranks, deformation sharded by Gaussian + NCCL all-gather (e2)")
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
        else:
            run_fgs(args, scene, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
