"""Per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of `ncu --set full` reports
-> profiles/ncu_traffic.json, which bench.py reads for the roofline `traffic` field.

    python tools/ncu_traffic.py --frames 20 --config dnerf gpurun_out/r1y_*.ncu-rep
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def kernel_traffic(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        base = name.split("(")[0].split("<")[0] if "::" not in name else name.split("(")[0]
        base = base.split("::")[-1].split("<")[0]
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            tot += float(r[i].replace(",", "")) * UNITS.get(u[i], 1)
        dur = float(r[h.index("gpu__time_duration.sum")].replace(",", ""))
        du = u[h.index("gpu__time_duration.sum")]
        dur_s = dur * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(du, 1e-9)
        res[base] = {"dram_bytes_per_launch": tot, "ncu_duration_s": dur_s, "report": os.path.basename(rep)}
    return res


def summary_traffic(path):
    """The same numbers from a tools/ncu_summary.py text summary (the .ncu-rep deleted on the GPU box)."""
    res, name, vals = {}, None, {}
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def flush():
        if name and "gpu__time_duration.sum" in vals:
            d, du = vals["gpu__time_duration.sum"]
            dur_s = d * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(du, 1e-9)
            tot = sum(v * units.get(uu, 1) for k, (v, uu) in vals.items() if k.startswith("dram__bytes_"))
            res[name] = {"dram_bytes_per_launch": tot, "ncu_duration_s": dur_s, "report": os.path.basename(path)}
    for line in open(path):
        if line.startswith("### "):
            flush()
            name = line[4:].strip().split("(")[0].split("::")[-1].split("<")[0]
            vals = {}
        elif line.startswith("| ") and name:
            parts = [x.strip() for x in line.strip().strip("|").split("|")]
            if len(parts) == 3:
                try:
                    vals[parts[0]] = (float(parts[1].replace(",", "")), parts[2])
                except ValueError:
                    pass
    flush()
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, required=True)
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "profiles", "ncu_traffic.json"))
    ap.add_argument("reports", nargs="+")
    a = ap.parse_args()
    data = {"config": a.config, "frames_per_launch": a.frames,
            "how": "ncu --set full --clock-control none, one launch per kernel of bench.py's default step",
            "kernels": {}}
    for rep in a.reports:
        data["kernels"].update(summary_traffic(rep) if rep.endswith(".txt") else kernel_traffic(rep))
    json.dump(data, open(a.out, "w"), indent=1)
    print(json.dumps(data, indent=1))
