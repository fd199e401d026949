"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package is input plumbing only (SURVEY.md
§8(c) S11/S12): workload descriptions (grid, PDE kind, stencil order, step
counts, macro-step count, weight-set *name*) and seeded initial-condition
generators.  It holds none of the method's arithmetic: no FE/LF/averaging,
no extrapolation weights, no stencils, no stability analysis.  Both
``oracle/`` and ``paper_1907_11771_b200/`` may import it; it imports neither.
"""

from .configs import CONFIGS, Workload, get_config, reduced  # noqa: F401
from .ic import make_ic  # noqa: F401
