"""Oracle: view-dependent SH colour — PAPER.md P:706 ("colour defined by spherical
harmonic (SH) coefficients C in R^k, where k represents nums of SH functions").

TEST INFRASTRUCTURE (see oracle/__init__.py).  numpy float64.

The paper does not give the basis; reading R10 takes the [3dgs] convention the
paper renders with: real SH with the Condon-Shortley phase, degree <= 3,
coefficient index k = l^2 + l + m (m = -l..l), colour = sum Y_k C_k + 0.5,
clamped at 0 only.  The table below is written from the standard real-SH
definitions (pinned against scipy.special.sph_harm_y in tests/test_oracle_sh.py).
"""
from __future__ import annotations

import math

import numpy as np

C0 = 0.5 / math.sqrt(math.pi)                      # Y_00 = 1/(2 sqrt(pi))
C1 = math.sqrt(3.0 / (4.0 * math.pi))
C2_K = 0.5 * math.sqrt(15.0 / math.pi)
C2_0 = 0.25 * math.sqrt(5.0 / math.pi)
C2_2 = 0.25 * math.sqrt(15.0 / math.pi)
C3_A = 0.25 * math.sqrt(35.0 / (2.0 * math.pi))
C3_B = 0.5 * math.sqrt(105.0 / math.pi)
C3_C = 0.25 * math.sqrt(21.0 / (2.0 * math.pi))
C3_E = 0.25 * math.sqrt(7.0 / math.pi)


def sh_basis(dirs, degree):
    """Real SH basis values Y_k(d) for unit directions d [N,3]; returns [N, (deg+1)^2].

    Order k = l^2 + l + m (m = -l..l); CS phase included.
    """
    d = np.asarray(dirs, np.float64)
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    cols = [np.full_like(x, C0)]
    if degree >= 1:
        cols += [-C1 * y, C1 * z, -C1 * x]
    if degree >= 2:
        xx, yy, zz = x * x, y * y, z * z
        cols += [C2_K * x * y, -C2_K * y * z, C2_0 * (2 * zz - xx - yy), -C2_K * x * z,
                 C2_2 * (xx - yy)]
    if degree >= 3:
        cols += [-C3_A * y * (3 * xx - yy), C3_B * x * y * z, -C3_C * y * (4 * zz - xx - yy),
                 C3_E * z * (2 * zz - 3 * xx - 3 * yy), -C3_C * x * (4 * zz - xx - yy),
                 0.5 * C3_B * z * (xx - yy), -C3_A * x * (xx - 3 * yy)]
    return np.stack(cols, axis=1)


def sh_to_rgb(sh, dirs, degree):
    """rgb = max(0, sum_k Y_k(d) C_k + 0.5) per channel (reading R10).

    sh: [N, K, 3]; dirs: [N, 3] unit.  Returns [N, 3] float64.
    """
    Y = sh_basis(dirs, degree)
    C = np.asarray(sh, np.float64)[:, : Y.shape[1], :]
    return np.maximum(0.0, np.einsum("nk,nkc->nc", Y, C) + 0.5)
