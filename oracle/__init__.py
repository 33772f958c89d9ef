"""fp64 CPU oracle of the TPO hot path (arXiv 2405.11922) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product path (paper_2405_11922_b200) never imports it and
shares no code with it.

* ``oracle.core``  -- ctypes wrapper of the plain-C fp64 oracle ``tpo_oracle.c``.
* ``oracle.dense`` -- tiny-size dense definitions (explicit L L^T series, the exact MSA
  matrix of Eq. s, brute-force Eq. obj1, robust principal angles) in numpy.

Parity status: all functions are pinned by tests/test_oracle_pins.py (see DESIGN.md
"Pins"); none is "parity unpinned".
"""
from . import core, dense  # noqa: F401
