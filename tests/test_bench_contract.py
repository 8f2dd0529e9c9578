"""bench.py host logic (no GPU): the reference arm's JSON line (the oracle timed on host cores —
the one bench.py leg that may execute oracle/) and the roofline arithmetic of roofline_objects."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2310_08528_b200.inputs import make_scene  # noqa: E402

REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e")


def test_reference_arm_json_line():
    """`bench.py --impl reference` prints ONE JSON line with the base contract's keys, the oracle's
    cpu_baseline (kind, cores, sample) and an e2e object with zero copy bytes."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny",
                          "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in REQUIRED:
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]


def test_roofline_work_per_step_with_several_launches():
    """A stage launched twice per step (render batches longer than one launch) must not count the
    step's work against one launch's time: achieved = step work / step time of the stage."""
    s = make_scene("dnerf", n=1000, n_frames=4)
    peaks = {"hbm_gbs": 6000.0, "sm_max_mhz": 2000.0}
    counts = {"sms": 148, "evaluated_per_frame": 1e6, "contrib_per_frame": 2e5, "instances_per_frame": 5e3}
    steps = 3
    stage_ms = {"deform": 0.3, "preprocess": 0.6, "blend": 1.5, "tile_scan": 0.03, "duplicate": 0.06,
                "tile_sort": 0.09}
    one = bench.roofline_objects(s, stage_ms, {k: steps for k in stage_ms}, peaks, counts, 2000.0, steps)
    two = bench.roofline_objects(s, stage_ms, {k: 2 * steps for k in stage_ms}, peaks, counts, 2000.0, steps)
    for k in ("deform", "preprocess", "blend", "binning"):
        assert one[k]["achieved"] == pytest.approx(two[k]["achieved"]), k
        assert one[k]["frac"] == pytest.approx(one[k]["achieved"] / one[k]["peak"]), k
    # preprocess: 308 B per Gaussian-frame at SH degree 3 over the per-step stage time
    by = s.n * (44 + 12 * 16 + 72) * s.n_frames
    assert one["preprocess"]["achieved"] == pytest.approx(by / (0.6e-3 / steps) / 1e9)
    # blend: (9 E + 4 C) per frame instructions over the per-step time, against 148 x 128 x clock
    work = (9 * 1e6 + 4 * 2e5) * s.n_frames / 1e12
    assert one["blend"]["achieved"] == pytest.approx(work / (1.5e-3 / steps))
    assert one["blend"]["peak"] == pytest.approx(148 * 128 * 2000e6 / 1e12)


def test_blend_c_basis_fraction():
    """roofline.frac_C: 13 instructions per contributing pair (SURVEY 8(d) C basis) over the same time."""
    s = make_scene("dnerf", n=1000, n_frames=2)
    counts = {"sms": 148, "evaluated_per_frame": 1e6, "contrib_per_frame": 2e5, "instances_per_frame": 5e3}
    r = bench.roofline_objects(s, {"blend": 1.0}, {"blend": 1}, {"hbm_gbs": 6000.0}, counts, 2000.0, 1)
    assert r["blend"]["achieved_C"] == pytest.approx(13 * 2e5 * 2 / 1e12 / 1e-3)
    assert r["blend"]["frac_C"] == pytest.approx(r["blend"]["achieved_C"] / r["blend"]["peak"])
    assert r["blend"]["frac_C"] < r["blend"]["frac"]


def test_oracle_full_frame_is_complete_and_matches_render_ref():
    """The oracle arm times a FULL frame (every Gaussian, every tile, no extrapolation): its pooled
    deform / preprocess / blend equal the single-process oracle exactly (tiny config, ragged tiles)."""
    import numpy as np

    import oracle
    s = make_scene("tiny", n=700, width=70, height=50)
    r = bench.oracle_full_frame(s, 0, 3)
    d = oracle.deform_ref(s, float(s.times[0]))
    for k in d:      # chunked vs whole-array matmul: equal up to BLAS summation order
        assert np.allclose(r["deformed"][k], d[k], rtol=0, atol=1e-13)
    ref = oracle.render_ref(r["deformed"], s.opacity_logits, s.sh, s.sh_degree, s.cameras[0])
    assert np.array_equal(r["image"], ref["image"])
    assert np.array_equal(r["n_contrib"], ref["n_contrib"]) and np.array_equal(r["flagged"], ref["flagged"])
    assert set(r["stages_s"]) == {"deform", "preprocess", "binning", "blend"}
