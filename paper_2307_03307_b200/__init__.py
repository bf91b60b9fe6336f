"""B200-native MWU positive-LP hot path (arXiv 2307.03307): CUDA library libmwu.so behind the
C ABI of include/mwu.h, with a thin ctypes binding.  See DESIGN.md."""
from .mwu import (  # noqa: F401
    Solver, MwuError, default_options, lib, EXPORTS, GRAPH_KINDS, VEC, ST,
    MIXED, PURE_PACKING, PURE_COVERING,
)
