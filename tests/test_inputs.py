"""Seeded input generator (paper_2310_08528_b200/inputs.py): shapes, determinism,
and the recipe of SURVEY §8(d) — CPU only."""
import numpy as np
import pytest

from paper_2310_08528_b200.inputs import CONFIGS, make_scene, morton_order


def test_tiny_recipe():
    s = make_scene("tiny")
    assert s.n == 2000 and s.n_frames == 1 and s.sh.shape == (2000, 1, 3)
    assert abs(s.cameras[0].fx - 68.62) < 0.01 and float(s.times[0]) == np.float32(0.37)
    assert s.field.planes[0][0].shape == (32, 32, 16) and s.field.planes[0][3].shape == (8, 32, 16)
    assert np.all((s.means >= -1) & (s.means <= 1))
    assert np.allclose(np.linalg.norm(s.quats.astype(np.float64), axis=1), 1.0, atol=1e-6)
    sp = s.field.planes[0][0]
    assert sp.min() >= 0.1 and sp.max() <= 0.5
    assert np.all(s.mlp.b_x == 0) and s.mlp.w_d.shape == (32, 16)


def test_dnerf_recipe_and_determinism():
    a = make_scene("dnerf", n=1000)
    b = make_scene("dnerf", n=1000)
    assert np.array_equal(a.means, b.means) and np.array_equal(a.field.planes[1][5], b.field.planes[1][5])
    assert a.n_frames == 20 and a.sh.shape == (1000, 16, 3) and a.mlp.w_d.shape == (64, 64)
    assert abs(a.cameras[0].fx - 857.80) < 0.01
    assert np.allclose(a.times, np.arange(20) / 19, atol=1e-7)
    for c in a.cameras:
        eye = -c.R.T.astype(np.float64) @ c.t.astype(np.float64)
        assert abs(np.linalg.norm(eye) - 4.0) < 1e-5
        assert np.allclose(c.R.astype(np.float64) @ c.R.T.astype(np.float64), np.eye(3), atol=1e-6)


@pytest.mark.parametrize("name,fx", [("hypernerf", 1029.36), ("neu3d", 1449.69), ("scaling", 2058.73)])
def test_other_configs_small(name, fx):
    s = make_scene(name, n=500)
    assert abs(s.cameras[0].fx - fx) < 0.01
    assert s.n_frames == {"hypernerf": 50, "neu3d": 8, "scaling": 64}[name]
    assert s.mlp.width == 128 and s.field.res == CONFIGS[name]["res"]


def test_morton_order_is_a_reordering_of_the_draw():
    a = make_scene("dnerf", n=3000, order="draw")
    b = make_scene("dnerf", n=3000)
    perm = morton_order(a.means, a.field.bmin, a.field.bmax)
    assert sorted(perm.tolist()) == list(range(3000))
    for k in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        assert np.array_equal(getattr(b, k), getattr(a, k)[perm]), k
    # neighbours in index space are close in space (Z-order locality): mean step << random step
    step_sorted = np.linalg.norm(np.diff(b.means.astype(np.float64), axis=0), axis=1).mean()
    step_draw = np.linalg.norm(np.diff(a.means.astype(np.float64), axis=0), axis=1).mean()
    assert step_sorted < 0.25 * step_draw


def test_morton_code_order_brute_force():
    """Z-order of a 2x2x2 grid of cell centres: code bit layout x (msb) y z per level."""
    pts = np.array([[x, y, z] for x in (0.25, 0.75) for y in (0.25, 0.75) for z in (0.25, 0.75)])
    rng = np.random.default_rng(0)
    sh = rng.permutation(8)
    perm = morton_order(pts[sh], (0, 0, 0), (1, 1, 1), bits=1)
    got = pts[sh][perm]
    want = sorted(pts.tolist(), key=lambda p: (p[0] > 0.5) * 4 + (p[1] > 0.5) * 2 + (p[2] > 0.5))
    assert np.array_equal(got, np.array(want))
