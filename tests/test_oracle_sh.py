"""Pins for the SH oracle (oracle/sh.py) against scipy's complex SH — CPU only.

P:706 leaves the basis to [3dgs]; reading R10 = real SH with the Condon-Shortley
phase.  scipy.special.sph_harm_y(l, m, theta, phi) includes the CS phase; the
real basis is sqrt(2) Re(Y_l^|m|) for m > 0, sqrt(2) Im(Y_l^|m|) for m < 0 and
Y_l^0 for m = 0 (SURVEY §8(c.4) SH row).
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import sph_harm_y

from oracle.sh import sh_basis, sh_to_rgb

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _real_sh_scipy(l, m, d):
    theta = np.arccos(np.clip(d[:, 2], -1, 1))
    phi = np.arctan2(d[:, 1], d[:, 0])
    Y = sph_harm_y(l, abs(m), theta, phi)
    if m > 0:
        return math.sqrt(2) * Y.real
    if m < 0:
        return math.sqrt(2) * Y.imag
    return Y.real


@pytest.mark.parametrize("degree", [0, 1, 2, 3])
def test_basis_matches_scipy(degree):
    rng = np.random.default_rng(degree)
    d = rng.normal(size=(1000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    B = sh_basis(d, degree)
    assert B.shape == (1000, (degree + 1) ** 2)
    for l in range(degree + 1):
        for m in range(-l, l + 1):
            k = l * l + l + m
            assert np.max(np.abs(B[:, k] - _real_sh_scipy(l, m, d))) < 1e-13, (l, m)


def test_golden_sh_examples():
    g = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))["sh"]
    d = np.array([[0.3, -0.4, 0.866]])
    d /= np.linalg.norm(d)
    zero = g[0]
    rgb = sh_to_rgb(np.zeros((1, 16, 3)), d, zero["degree"])
    assert np.allclose(rgb, zero["rgb"], atol=0, rtol=0)
    dc = g[1]
    sh = np.zeros((1, 1, 3))
    sh[0, 0] = dc["dc"]
    assert np.allclose(sh_to_rgb(sh, d, 0)[0], dc["rgb"], atol=1e-15)


def test_clamp_at_zero_only():
    d = np.array([[0.0, 0.0, 1.0]])
    sh = np.zeros((1, 1, 3))
    sh[0, 0] = [-10.0, 10.0, 0.0]
    rgb = sh_to_rgb(sh, d, 0)[0]
    assert rgb[0] == 0.0 and rgb[1] > 1.0 and rgb[2] == 0.5
