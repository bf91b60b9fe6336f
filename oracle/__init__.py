"""CPU oracle for the MWU hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import anything from this package.  The product
path (`paper_2307_03307_b200`) never imports it and shares no code with it.
"""
from .mwu_oracle import *  # noqa: F401,F403
