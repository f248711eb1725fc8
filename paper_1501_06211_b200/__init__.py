"""B200-native interface-PCG for SIMP-weighted Q1 elasticity by non-overlapping domain
decomposition (arXiv 1501.06211).  The product is the C-ABI library libde.so
(include/de.h; sources in csrc/); `binding` is its thin ctypes mirror."""
from . import binding  # noqa: F401
from .binding import Solver, DEError  # noqa: F401
