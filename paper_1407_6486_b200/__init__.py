"""B200-native (sm_100a) PFASST x multigrid hot path, a drop-in for the
reference package ``pintlab`` (arXiv:1407.6486, "Interweaving PFASST and
Parallel Multigrid").

The module layout and public names mirror the reference (heat, transfers,
multigrid, quadrature, sdc, hierarchy, pfasst); every computation on the
path runs in lib/libpintlab_b200.so through the C ABI declared in
include/pintlab_b200.h.  There is no CPU fallback.
"""
from . import heat, hierarchy, multigrid, pfasst, quadrature, sdc, transfers  # noqa: F401
from ._build import LIB  # noqa: F401

__all__ = ["heat", "hierarchy", "multigrid", "pfasst", "quadrature", "sdc", "transfers"]
