"""B200-native extrapolated GBS time stepper (Ellison & Fornberg, arXiv 1907.11771).

The hot path (FE start, leap-frog substeps over an FD MOL right-hand side,
averaging, weighted extrapolation; Eq. (1) and lines 109-115) runs in
the sm_100a kernels of ``lib/libgbs_b200.so`` behind the C ABI of
``include/gbs.h``; ``gbs`` is its thin binding and ``scheme`` the host-side
weight / H setup.  This package never imports ``oracle/``.
"""

from . import scheme  # noqa: F401

__all__ = ["gbs", "scheme"]
