"""CPU oracle for the asynchronous-RAS hot path (arxiv 2003.05361).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import, call or
execute anything under `oracle/`.  The product path (`paper_2003_05361_b200`,
the CUDA library behind `include/ras.h`) never imports it and shares no code
with it; the only shared module is `ras_inputs` (seeded input generators,
none of the method's arithmetic).
"""
from .ras_oracle import *  # noqa: F401,F403
from .ras_oracle import __all__  # noqa: F401
