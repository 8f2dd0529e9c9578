"""Per-CUDA-source-line aggregation of an ncu --set full --import-source report: stall samples,
instructions executed and shared-memory wavefronts.  Usage: python tools/ncu_lines.py REP [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data, fname = None, [], ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        data.append((fname, r))
cols = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared"]
idx = [hdr.index(c) for c in cols]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


agg = {}
for fname, r in data:
    a = agg.setdefault((fname, r[0], r[1].strip()), [0.0, 0.0, 0.0])
    for k, i in enumerate(idx):
        a[k] += num(r[i])
tot = [sum(v[k] for v in agg.values()) or 1.0 for k in range(3)]
print(f"totals: samples {tot[0]:.0f}  inst {tot[1]:.4g}  shared wavefronts {tot[2]:.4g}")
for (fn, ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{fn[:12]:12s}{ln:>5} {100*v[0]/tot[0]:5.1f}% smp {100*v[1]/tot[1]:5.1f}% inst {100*v[2]/tot[2]:5.1f}% wf  {src[:70]}")
