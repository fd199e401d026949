"""Workload table: the five BASELINE.json configs, restated as plain data.

Each entry is a description only (what to run), never how: the step counts,
the *name* of the weight set, the H rule's factor, the macro-step count and
the IC recipe.  Weights and H are computed from these names on each side
independently (``paper_1907_11771_b200.scheme`` for the product,
``oracle.weights`` / ``oracle.stability`` for the oracle).

Sources: BASELINE.json ``configs[0..4]``; SURVEY.md §8(c) S3 (weight
fallback), S6 (unit periodic box), S7 (H rule), S11 (IC recipe), §8(d)
table (sizes).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Tuple

PDE_FIELDS = {"adv1d": 1, "acoustic2d": 3, "wave3d": 2}
PDE_NDIM = {"adv1d": 1, "acoustic2d": 2, "wave3d": 3}


@dataclass(frozen=True)
class Workload:
    name: str
    pde: str                      # 'adv1d' | 'acoustic2d' | 'wave3d'
    n: Tuple[int, int, int]       # grid points (nx, ny, nz); unused axes = 1
    order: int                    # centered FD order (4 or 8)
    steps: Tuple[int, ...]        # GBS step counts n_k (even, distinct)
    weights: str                  # weight-set name (see module doc)
    macro_steps: int              # M
    ic: str                       # IC recipe name (gbs_inputs.ic)
    seed: int
    h_factor: float = 0.5         # H = h_factor * ISB(R) / rho  (S7)
    notes: str = field(default="", compare=False)

    @property
    def ndim(self) -> int:
        return PDE_NDIM[self.pde]

    @property
    def fields(self) -> int:
        return PDE_FIELDS[self.pde]

    @property
    def points(self) -> int:
        nx, ny, nz = self.n
        return nx * ny * nz

    @property
    def state_shape(self) -> Tuple[int, ...]:
        """numpy shape of the SoA state: [F][nz][ny][nx] with unused axes dropped."""
        nx, ny, nz = self.n
        if self.ndim == 1:
            return (self.fields, nx)
        if self.ndim == 2:
            return (self.fields, ny, nx)
        return (self.fields, nz, ny, nx)

    @property
    def substeps(self) -> int:
        """S = sum_k (n_k + 1): RHS-evaluating substeps per macro step (S16)."""
        return sum(k + 1 for k in self.steps)

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]
    "c1": Workload("c1", "adv1d", (256, 1, 1), 4, (2, 4, 6, 8), "square8", 200,
                   "gauss1d", 1001,
                   notes="1D advection u_t=-u_x, FD4, square order-8 weights"),
    # configs[1]: paper's optimized order-8 weights on {2..12} are not tabulated
    # (SURVEY §0 finding 3, S3) -> square {2,4,6,8} weights, 0 on 10 and 12.
    "c2": Workload("c2", "acoustic2d", (1024, 1024, 1), 4, (2, 4, 6, 8, 10, 12),
                   "fallback8", 50, "gauss2d_sum8", 1002),
    "c3": Workload("c3", "acoustic2d", (4096, 4096, 1), 8, (2, 4, 6, 8, 10, 12),
                   "fallback8", 20, "bandlimited2d", 1003),
    "c4": Workload("c4", "wave3d", (512, 512, 512), 8, (2, 4, 6, 8, 10, 12),
                   "fallback8", 10, "gauss3d", 1004),
    "c5": Workload("c5", "wave3d", (1024, 1024, 1024), 8,
                   (2, 4, 6, 8, 10, 12, 14, 16), "fallback8", 4,
                   "bandlimited3d", 1005),
}

# The paper's own experiment (§4.1), not a
# BASELINE.json config: one-way wave u_t + u_x = 0 on [0,1), spectral derivative (order 0),
    # IC (1 - cos 2 pi x)/2, GBS_8,6, lambda = dt/dx = 0.99/pi ISB (h_factor 0.99 with
    # rho = pi N), one period (macro steps = ceil(1 / H_max), H = 1 / macro steps).
PAPER_WORKLOADS = {
    "s41": Workload("s41", "adv1d", (64, 1, 1), 0, tuple(range(2, 23, 2)), "GBS_8_6", 0,
                    "cos1d", 0, h_factor=0.99,
                    notes="PAPER.md 4.1 one-way wave, spectral, one period"),
}


def get_config(name: str) -> Workload:
    key = name.lower()
    if key in CONFIGS:
        return CONFIGS[key]
    if key in PAPER_WORKLOADS:
        return PAPER_WORKLOADS[key]
    raise KeyError(f"unknown config {name!r}; known: {sorted(CONFIGS) + sorted(PAPER_WORKLOADS)}")


def reduced(name: str, n: Tuple[int, int, int], macro_steps: int | None = None,
            weights: str | None = None) -> Workload:
    """Same PDE, stencil, step counts and IC recipe as config `name`, smaller grid."""
    w = get_config(name)
    kw = {"n": tuple(n), "name": f"{w.name}-reduced-{'x'.join(map(str, n))}"}
    if macro_steps is not None:
        kw["macro_steps"] = macro_steps
    if weights is not None:
        kw["weights"] = weights
    return w.with_(**kw)
