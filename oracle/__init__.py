"""fp64 CPU ORACLE for the 4D-GS per-frame deform + render path — TEST INFRASTRUCTURE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything under `oracle/`.  The product path
(`paper_2310_08528_b200`) never imports it, and this package never imports the
product path (it shares no code, header, helper or constant generator with
`paper_2310_08528_b200/csrc`).  The only shared module is the seeded input
generator `paper_2310_08528_b200.inputs`, which holds none of the method's
arithmetic.

Plain numpy, float64 throughout (inputs are the fp32 arrays promoted exactly),
vectorised only across independent Gaussians / pixels; every function follows
the paper passage cited in its docstring, in the paper's order and notation.
Citations: `P:n` = /root/reference/PAPER.md line n (later, camera-ready version
P:611-1251 is authoritative); readings D*/R* are listed in DESIGN.md §3 and
SURVEY.md §8(c.3).

`oracle.backward` (imported explicitly; it needs torch) restates the forward in PyTorch CPU float64
ops and differentiates it with autograd: the gradients of the training loss of PAPER.md §4.3.

Pinned by `tests/test_oracle_*.py` (-m "not gpu") against closed forms, worked
examples (tests/golden/), library routines (scipy SH) and brute force.  The
only unpinned item is end-to-end image parity with the paper's figures (no
trained weights / datasets): "parity unpinned" for that, and only that.
"""
from . import deform, render, sh  # noqa: F401
from .deform import deform_ref, hexplane_features  # noqa: F401
from .render import preprocess_ref, render_ref, render_ref_bruteforce  # noqa: F401
