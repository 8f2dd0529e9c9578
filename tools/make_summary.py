"""Assemble profiles/<name>_summary.md from one evidence pass (tools/gpu_round_evidence.sh TAG):
headline bench line, per-stage times and rooflines, other configurations, colour heads, shard mode,
reference arm, N sweep, ncu launch list and the ncu --set full key metrics of every kernel.

    python tools/make_summary.py TAG NAME "title"
"""
import glob
import json
import os
import subprocess
import sys

TAG, NAME = sys.argv[1], sys.argv[2]
TITLE = sys.argv[3] if len(sys.argv) > 3 else f"{NAME} on B200"
G = "gpurun_out"


def line(path):
    try:
        return json.loads([x for x in open(path) if x.startswith("{")][-1])
    except (OSError, IndexError):
        return None


def stages_us(d):
    F = d["config"].get("frames_per_step", 1)
    return {k: v * 1e3 / F for k, v in d.get("stages_ms_per_step", {}).items()}


out = [f"# {TITLE}", ""]
out.append(f"Commands (gpurun, 1x B200): `bash tools/gpu_round_evidence.sh {TAG}` — `python bench.py` (defaults: "
           "D-NeRF-like config, 20 frames/step, K=20, W=5; headline = CUDA-graph replay of one fgs_frames step), "
           "the ncu launch list (`ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py "
           "--steps 2 --warmup 3 --no-e2e --no-cpu-baseline`), one `ncu --set full --clock-control none "
           "--import-source on` capture per kernel of the step, `bench.py --config hypernerf|neu3d|scaling`, "
           "`--colour-heads`, `--config scaling --mode shard`, `--impl reference`, `tools/sweep_n.sh`.  "
           f"Summary written by `python tools/make_summary.py {TAG} {NAME}`.")
out.append("")
d = line(f"{G}/{TAG}_bench.log")
if d:
    F = d["config"]["frames_per_step"]
    out += ["## Headline (bench.py default)", ""]
    out.append(f"* value **{d['value']:.0f} frames/s** (graph replay; eager {d.get('value_eager', 0):.0f}); "
               f"{d['ms_per_step']:.3f} ms per {F}-frame step; step p10/p50/p90 "
               f"{d.get('step_ms', {}).get('p10', 0):.3f}/{d.get('step_ms', {}).get('median', 0):.3f}/"
               f"{d.get('step_ms', {}).get('p90', 0):.3f} ms")
    e = d.get("e2e") or {}
    if e:
        out.append(f"* e2e (fgs_frames_host: pinned host model in, host images out, copies inside the timed "
                   f"region): {e['value']:.0f} frames/s"
                   + (f" with two calls in flight ({e['serial_value']:.0f} one call at a time)" if "serial_value" in e else "")
                   + f"; {e['h2d_bytes_per_step'] / 1e6:.1f} MB in, "
                   f"{e['d2h_bytes_per_step'] / 1e6:.1f} MB out per step (PCIe: 54-57 GB/s measured each way, "
                   "`tools/numa_probe.py`)")
    for tl in open(f"profiles/{NAME}_tile_cull.jsonl") if os.path.exists(f"profiles/{NAME}_tile_cull.jsonl") else []:
        t = json.loads(tl)
        tc = t.get("tile_cull") or {}
        if tc:
            out.append(f"* `--tile-cull` ({t['config']['workload'].split(':')[0]}): {t['value']:.0f} -> {tc['value']:.0f} frames/s with "
                       f"FGS_TUNE_TILE_CULL = 1 (opt-in, default off), images identical: {tc['images_identical']}")
    cb = d.get("cpu_baseline") or {}
    if cb:
        out.append(f"* oracle (fp64 numpy, {cb.get('cores')} host processes, bounded sample): {cb.get('value'):.3g} "
                   f"{cb.get('unit')} — {cb.get('sample', '')}")
    pa = d.get("parity") or {}
    if pa:
        out.append(f"* whole-frame parity vs the oracle (frame {pa['frame']}, every Gaussian and every pixel): deform max "
                   f"|err| {pa['deform_max_abs_err']:.3g} (tol 1e-4); integer mismatches {pa['integer_mismatches']} "
                   f"outside {pa['boundary_gaussians']} boundary Gaussians; PSNR {pa['psnr_db']:.1f} dB; max |err| on "
                   f"unflagged pixels {pa['max_abs_err_unflagged']:.3g} (tol 2e-3); {pa['flagged_pixels']} flagged of "
                   f"{pa['pixels']} pixels; pass = {pa['pass']}")
    out.append(f"* clocks during the timed region: {d.get('clocks')}; launches per step "
               f"{d.get('gpu_launches_per_step')}")
    r = d.get("roofline") or {}
    if r:
        out.append(f"* roofline (dominant kernel, {r.get('kernel')}): {r['achieved']:.4g} {r['unit']} of "
                   f"{r['peak']:.4g} = **{r['frac']:.3f}**, DRAM traffic {r.get('traffic')} B per launch")
    out += ["", "## Stage times (library CUDA events, eager timed region)", "",
            "| stage | us per step | us per frame | share |", "|---|---|---|---|"]
    st = d.get("stages_ms_per_step", {})
    tot = sum(st.values()) or 1.0
    for k, v in st.items():
        out.append(f"| {k} | {v * 1e3:.1f} | {v * 1e3 / F:.1f} | {100 * v / tot:.1f}% |")
    out += ["", "## Roofline per stage", "",
            "| stage | bound | achieved | peak | frac | ncu DRAM bytes/launch | algorithmic work |",
            "|---|---|---|---|---|---|---|"]
    for k, v in (d.get("roofline_stages") or {}).items():
        out.append(f"| {k} | {v['bound']} | {v['achieved']:.4g} {v['unit']} | {v['peak']:.5g} | {v['frac']:.3f} | "
                   f"{v.get('traffic')} | {v.get('algorithmic', '')} |")
    w = d.get("work_per_frame") or {}
    if w:
        out += ["", "Work per frame: " + ", ".join(f"{k} {v:.4g}" for k, v in w.items())]

out += ["", "## Other configurations (frame mode, 1 GPU)", "",
        "| config | N | image | frames/step | frames/s | e2e frames/s | deform / preprocess / tile sort / duplicate / blend (us per frame) |",
        "|---|---|---|---|---|---|---|"]
for c in ("hypernerf", "neu3d", "scaling"):
    d2 = line(f"{G}/{TAG}_cfg_{c}.log")
    if not d2:
        continue
    su = stages_us(d2)
    cf = d2["config"]
    e2 = (d2.get("e2e") or {}).get("value")
    out.append(f"| {c} | {cf.get('n_gaussians', 0):,} | {cf.get('image')} | {cf['frames_per_step']} | {d2['value']:.0f} | "
               f"{e2 and round(e2)} | {su.get('deform', 0):.1f} / {su.get('preprocess', 0):.1f} / "
               f"{su.get('tile_sort', 0):.1f} / {su.get('duplicate', 0):.1f} / {su.get('blend', 0):.1f} |")
out.append("")
dc = line(f"{G}/{TAG}_colour.log")
if dc:
    out.append(f"* D with the colour/opacity decoders (P:1232, `--colour-heads`): {dc['value']:.0f} frames/s "
               f"(deform {stages_us(dc).get('deform', 0):.1f} us/frame)")
ds = line(f"{G}/{TAG}_shard.log")
if ds:
    out.append(f"* S config, `--mode shard` (e2: deformation sharded by Gaussian + NCCL all-gather per distinct "
               f"time, world 1): {ds['value']:.0f} frames/s")
dr = line(f"{G}/{TAG}_reference.log")
if dr:
    out.append(f"* reference arm (`bench.py --impl reference`: the fp64 oracle on {dr.get('cpu_baseline', {}).get('cores')} "
               f"host processes): {dr['value']:.3g} frames/s")

tr = [x for x in (line(f"{G}/{TAG}_train.log"), line(f"{G}/{TAG}_train_neu3d.log")) if x]
if tr:
    out += ["", "## Training side (SURVEY 8(f) rank 4: `bench.py --mode train`)", "",
            "| config | training frames/s | deform / render / L1 / render backward / deform backward / TV (ms per frame) |",
            "|---|---|---|"]
    for d4 in tr:
        st = d4.get("stages_ms_per_frame", {})
        out.append(f"| {d4['config']['workload'].split(':')[0]} | {d4['value']:.0f} | "
                   + " / ".join(f"{st.get(k, 0):.3f}" for k in ("deform", "render", "l1_loss", "render_backward",
                                                                  "deform_backward", "tv_loss")) + " |")
    cb4 = tr[0].get("cpu_baseline")
    if cb4:
        out.append(f"\nAutograd oracle (extrapolated from a bounded sample): {cb4['value']:.3g} {cb4['unit']} — {cb4['sample']}")
try:
    br = json.load(open(f"{G}/{TAG}_bwd_report.json"))
    errs = br["errors"]["grad_rel_err"]
    out.append(f"\nGradient parity (GPU chain vs the autograd oracle, one frame of a 60-Gaussian 40x32 scene, max |diff| / "
               f"max |ref| per tensor): worst {max(errs.values()):.2g} ({max(errs, key=errs.get)}), loss rel. err "
               f"{br['errors']['loss_rel_err']:.2g}")
except (OSError, KeyError, ValueError):
    pass

sw = []
try:
    sw = [json.loads(x) for x in open(f"{G}/{TAG}_sweep.jsonl") if x.startswith("{")]
except OSError:
    pass
if sw:
    out += ["", "## N sweep (SURVEY 8(f) rank 1; D distributions at 800x800, 20 frames per step)", "",
            "| N | frames/s | ms/step | instances/frame | deform / preprocess / tile sort / blend (us per frame) |",
            "|---|---|---|---|---|"]
    for d3 in sw:
        su = stages_us(d3)
        inst = (d3.get("work_per_frame") or {}).get("instances_per_frame", 0)
        out.append(f"| {d3['config'].get('n_gaussians', 0):,} | {d3['value']:.0f} | {d3['ms_per_step']:.2f} | {inst:.3g} | "
                   f"{su.get('deform', 0):.1f} / {su.get('preprocess', 0):.1f} / {su.get('tile_sort', 0):.1f} / "
                   f"{su.get('blend', 0):.1f} |")

lc = f"{G}/{TAG}_launches.csv"
if os.path.exists(lc):
    out += ["", "## ncu launch list (cold-cache, serialised; includes warm-up and the untimed debug renders "
            "`blend_kernel<1>`)", ""]
    out.append(subprocess.run([sys.executable, "tools/ncu_launches.py", lc], capture_output=True, text=True).stdout.strip())
reps = sorted(glob.glob(f"{G}/{TAG}_*.ncu-rep"))
txts = sorted(glob.glob(f"{G}/{TAG}_*.summary.txt"))
if reps or txts:
    out += ["", "## ncu --set full, one launch per kernel (20-frame batch; backward: one D frame)", ""]
    for rep in reps:
        out.append(subprocess.run([sys.executable, "tools/ncu_summary.py", rep], capture_output=True, text=True).stdout.strip())
        out.append("")
    for t in txts:
        if t.replace(".summary.txt", ".ncu-rep") in reps:
            continue
        out.append(open(t).read().strip())
        out.append("")
open(f"profiles/{NAME}_summary.md", "w").write("\n".join(out) + "\n")
print(f"profiles/{NAME}_summary.md", len(out), "lines")
