"""Oracle: the Adam update the paper's training uses ("The learning rate is set as 1.6e-3 ...",
[3dgs] / 4D-GS train with Adam; SURVEY §8(f) rank 4 "Adam").  TEST INFRASTRUCTURE (see oracle/__init__.py).

Standard bias-corrected Adam (Kingma & Ba), written out per element in float64, in the textbook order:
    m_t = b1 m_{t-1} + (1 - b1) g
    v_t = b2 v_{t-1} + (1 - b2) g^2
    m^ = m_t / (1 - b1^t),  v^ = v_t / (1 - b2^t)
    p_t = p_{t-1} - lr m^ / (sqrt(v^) + eps)
Reading A1: eps is added to sqrt(v^) (the PyTorch / [3dgs] convention), t counts from 1.
Pinned by tests/test_oracle_optim.py: zero gradient -> parameters unchanged and moments decayed by b1, b2
(SPEC S:358); first step with g != 0 -> |dp| = lr g / (|g| + eps) ~ lr; torch.optim.Adam (a
library routine) on the same trace.
"""
from __future__ import annotations

import numpy as np


def adam_step(p, g, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    """One Adam step at step number t (1-based); returns (p, m, v) as new float64 arrays."""
    p = np.asarray(p, np.float64)
    g = np.asarray(g, np.float64)
    m = b1 * np.asarray(m, np.float64) + (1.0 - b1) * g
    v = b2 * np.asarray(v, np.float64) + (1.0 - b2) * g * g
    mh = m / (1.0 - b1 ** t)
    vh = v / (1.0 - b2 ** t)
    return p - lr * mh / (np.sqrt(vh) + eps), m, v
