"""Pins for the Adam oracle (oracle/optim.py) — CPU only."""
import numpy as np
import pytest

from oracle import optim


def test_zero_gradient_keeps_parameters_and_decays_moments():
    """grad 0 everywhere -> params unchanged, moments decay by b1 / b2."""
    rng = np.random.default_rng(0)
    p, m, v = rng.normal(size=50), rng.normal(size=50), rng.uniform(size=50)
    p2, m2, v2 = optim.adam_step(p, np.zeros(50), m, v, 7, 1e-3)
    # m^ != 0 still moves p unless m == 0: with m == 0 nothing moves
    p3, m3, v3 = optim.adam_step(p, np.zeros(50), np.zeros(50), v, 7, 1e-3)
    assert np.array_equal(p3, p) and np.all(m3 == 0)
    assert np.allclose(m2, 0.9 * m, rtol=0, atol=1e-15) and np.allclose(v2, 0.999 * v, rtol=0, atol=1e-15)


def test_first_step_magnitude_is_lr():
    """first step, scalar g > 0 -> dp = -lr g / (|g| + eps) (bias-corrected magnitude lr)."""
    for g in (1e-3, 0.5, 7.0):
        p, _, _ = optim.adam_step(np.array([2.0]), np.array([g]), np.zeros(1), np.zeros(1), 1, 1.6e-3)
        assert abs((2.0 - p[0]) - 1.6e-3 * g / (g + 1e-8)) < 1e-15


def test_matches_torch_adam_trace():
    """100 random steps against torch.optim.Adam (a library routine) in float64."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    p0 = rng.normal(size=64)
    P = torch.tensor(p0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([P], lr=1.6e-3, betas=(0.9, 0.999), eps=1e-8)
    p, m, v = p0.copy(), np.zeros(64), np.zeros(64)
    for t in range(1, 101):
        g = rng.normal(size=64) * (0.1 + t % 7)
        P.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        p, m, v = optim.adam_step(p, g, m, v, t, 1.6e-3)
    assert np.max(np.abs(P.detach().numpy() - p)) <= 1e-12
