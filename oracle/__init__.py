"""fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg may
import, call, link or execute anything under oracle/.  The product path
(paper_2202_07235_b200/) never imports it and shares no code with it.  See oracle/ref.py for the
function list and the PAPER.md passages each one follows.

Parity pinned: O1, O2, O3, O4, O5, P8 (tests/test_oracle_pins.py); F1-F3 (same file); the f4 volume
oracle V1-V6 in oracle/vol.py (tests/test_oracle_vol_pins.py).  "Parity unpinned": the
generator's absolute scale and SNR calibration beyond self-consistency.
"""
from . import ref  # noqa: F401
from . import vol  # noqa: F401
