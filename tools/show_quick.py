"""Print frames/s and per-frame stage times of the bench logs written by tools/gpu_quick.sh TAG."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "q"
for c in ("dnerf", "neu3d", "hypernerf"):
    try:
        line = [x for x in open(f"gpurun_out/{tag}_bench_{c}.log") if x.startswith("{")][-1]
    except (OSError, IndexError):
        print(c, "no result")
        continue
    d = json.loads(line)
    F = d["config"].get("frames_per_step", 1)
    st = {k: round(v * 1e3 / F, 1) for k, v in d.get("stages_ms_per_step", {}).items()}
    print(f"{c:10s} {d['value']:8.0f} frames/s  eager {d.get('value_eager', 0):8.0f}  us/frame {st}")
