"""Deformation-kernel timeline (analysis aid, not product code): needs a library built with
-DFGS_EXP_TRACE (tools/build_variant.sh trace deform_tc3.cu -DFGS_EXP_TRACE).  Runs the batch
deformation of a config twice and prints, from CTA 0's clock64 events, where each role's cycles go
per tile-frame: producers (prologue, staging, A compute, wait for A free, A store), the MMA issuer
(wait for A full / D free) and the epilogue (wait for D full, heads + stores).
Usage: python tools/deform_trace.py [config] [frames]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2310_08528_b200 import fgs  # noqa: E402
from paper_2310_08528_b200.inputs import make_scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "dnerf"
F = int(sys.argv[2]) if len(sys.argv) > 2 else None
s = make_scene(name, n_frames=F)
ds = fgs.DeviceScene(s, "cuda:0")
ts = [float(t) for t in s.times]
outs, _ = ds.alloc_deformed(len(ts))
for _ in range(2):
    fgs.fgs_deform_batch(ds.g, ds.field, ds.mlp, ts, outs)
torch.cuda.synchronize()
L = fgs.lib()
KN = 2048
buf = np.zeros((24, KN), dtype=np.uint64)
assert L.fgs_exp_trace(ctypes.c_void_p(buf.ctypes.data)) == 0
tag = (buf >> np.uint64(56)).astype(int)
clk = (buf & np.uint64((1 << 56) - 1)).astype(np.int64)


def events(w):
    n = int(np.count_nonzero(buf[w]))
    return list(zip(tag[w, :n], clk[w, :n]))


t0 = min(c for w in range(24) for _, c in events(w) if c > 0)
print(f"{name}: {len(ts)} frames; CTA 0 timeline (cycles)")
# producers: per-warp sums of the phases
P = {"prologue (1->2)": 0, "group setup (2->3)": 0, "staging issue (3->4)": 0, "staging barrier (4->5)": 0,
     "A compute (5|8 -> 6)": 0, "wait A free (6->7)": 0, "A store (7->8)": 0}
nw = 0
end_all = 0
for w in range(16):
    ev = events(w)
    if not ev:
        continue
    nw += 1
    prev = None
    for (tg, c) in ev:
        if prev is not None:
            ptg, pc = prev
            d = c - pc
            key = {(1, 2): "prologue (1->2)", (2, 3): "group setup (2->3)", (3, 4): "staging issue (3->4)",
                   (4, 5): "staging barrier (4->5)", (5, 6): "A compute (5|8 -> 6)", (8, 6): "A compute (5|8 -> 6)",
                   (6, 7): "wait A free (6->7)", (7, 8): "A store (7->8)"}.get((ptg, tg))
            if key:
                P[key] += d
        prev = (tg, c)
    end_all = max(end_all, ev[-1][1])
ntf = sum(1 for tg, _ in events(0) if tg == 8)
span = end_all - t0
print(f"span {span} cycles, {ntf} tile-frames in CTA 0 -> {span / max(ntf, 1):.0f} cycles per tile-frame")
print("producers (mean over warps, cycles per tile-frame):")
for k, v in P.items():
    print(f"  {k:24s} {v / max(nw, 1) / max(ntf, 1):8.0f}")
M = {"wait A full (10->11)": 0, "wait D free (11->12)": 0, "issue (12->13)": 0, "loop (13->10)": 0}
ev = events(20)
for (a, b) in zip(ev, ev[1:]):
    key = {(10, 11): "wait A full (10->11)", (11, 12): "wait D free (11->12)", (12, 13): "issue (12->13)",
           (13, 10): "loop (13->10)"}.get((a[0], b[0]))
    if key:
        M[key] += b[1] - a[1]
print("MMA issuer (cycles per tile-frame):")
for k, v in M.items():
    print(f"  {k:24s} {v / max(ntf, 1):8.0f}")
E = {"wait D full (20->21)": 0, "heads + stores (21->22)": 0, "loop (22->20)": 0}
ne = 0
for w in range(16, 20):
    ev = events(w)
    if not ev:
        continue
    ne += 1
    for (a, b) in zip(ev, ev[1:]):
        key = {(20, 21): "wait D full (20->21)", (21, 22): "heads + stores (21->22)", (22, 20): "loop (22->20)"}.get(
            (a[0], b[0]))
        if key:
            E[key] += b[1] - a[1]
print("epilogue (mean over warps, cycles per tile-frame):")
for k, v in E.items():
    print(f"  {k:24s} {v / max(ne, 1) / max(ntf, 1):8.0f}")
# first few tile-frames of warp 0 / MMA / epilogue 16, relative times
for w in (0, 20, 16):
    ev = events(w)[:40]
    print(f"warp {w}: " + " ".join(f"{tg}@{c - t0}" for tg, c in ev))
