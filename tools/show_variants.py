"""Summarise gpurun_out/v_<V>_<config>.log (tools/gpu_variants.sh): frames/s and per-stage us/frame."""
import glob
import json
import os
import re
import sys

root = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
rows = []
for p in sorted(glob.glob(os.path.join(root, "v_*.log"))):
    m = re.match(r"v_(.+)_(dnerf|neu3d|hypernerf|scaling|tiny)\.log", os.path.basename(p))
    if not m:
        continue
    d = None
    for line in open(p):
        if line.startswith("{"):
            d = json.loads(line)
    if d is None:
        print(m.group(1), m.group(2), "no result")
        continue
    F = d["config"]["frames_per_step"]
    st = {k: 1e3 * v / F for k, v in d["stages_ms_per_step"].items()}
    print(f"{m.group(1):10s} {m.group(2):10s} {d['value']:9.1f} fps  " +
          " ".join(f"{k}={v:6.1f}" for k, v in st.items()))
