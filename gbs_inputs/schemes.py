"""Free extrapolation weights of the Appendix-B optimised sets (input data).

``optimized_schemes.json`` holds, per set, the order, n_dep, n_free and the free
weights c_free as exact "num/den" strings -- the same kind of data the paper prints
for GBS_8,6 / GBS_8,8 / GBS_12,8.  It is written by
``tools/optimize_schemes.py`` (App. B optimiser, host side) and read here
as plain data; the dependent weights are computed from it independently by
``paper_1907_11771_b200.scheme`` and ``oracle.weights`` (Eq. (6)).  No method
arithmetic lives here.
"""

from __future__ import annotations

import json
import os
from typing import Dict, Sequence

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "optimized_schemes.json")


def optimized_sets() -> Dict[str, dict]:
    with open(_PATH) as f:
        return json.load(f)


def optimized_for(steps: Sequence[int]) -> dict:
    """The optimised order-8 set whose step counts are exactly `steps` ("opt8")."""
    want = sorted(steps)
    for name, s in optimized_sets().items():
        if sorted(s["n_dep"] + s["n_free"]) == want:
            return dict(s, name=name)
    raise KeyError(f"no optimised weight set on step counts {want}")
