"""The sequence-group partition (gbs_plan, the planner gbs_create uses) is optimal.

PAPER.md §3.6 (lines 388-400) folds the sequences onto cores so that every core does the
same number of RHS evaluations; SURVEY.md §8(e) asks for the exact optimum (brute force,
m <= 16) of the critical path = max over groups of sum (n_k + 1).  Pinned against:
* SURVEY.md §8(e)'s brute-force table (2 / 4 / 8 GPUs for {2,4,6,8}, {2..12}, {2..16});
* the lower bound max(ceil(S / g), n_max + 1), which the optimum reaches for the sets the
  round-1 planner missed ({2..12}/2 -> 24, {2..16}/3 -> 27, {2..22}/4 -> 36, {2..30}/3 -> 85);
* an exhaustive search over every assignment, written here independently, on random sets.
"""

import itertools
import random

import pytest

from paper_1907_11771_b200 import gbs


def plan_groups(counts, g):
    plans = [gbs.gbs_plan("wave3d", (64, 64, 64), 8, counts, g, r, g) for r in range(g)]
    groups = [tuple(p["my_n_k"]) for p in plans]
    return plans[0]["critical_substeps"], groups


def brute_force(counts, g):
    best = None
    for asg in itertools.product(range(g), repeat=len(counts)):
        load = [0] * g
        for n, q in zip(counts, asg):
            load[q] += n + 1
        best = max(load) if best is None else min(best, max(load))
    return best


@pytest.mark.parametrize("counts,g,crit", [
    ((2, 4, 6, 8), 2, 12), ((2, 4, 6, 8), 4, 9),
    (tuple(range(2, 13, 2)), 2, 24), (tuple(range(2, 13, 2)), 4, 13), (tuple(range(2, 13, 2)), 6, 13),
    (tuple(range(2, 17, 2)), 2, 40), (tuple(range(2, 17, 2)), 4, 20), (tuple(range(2, 17, 2)), 8, 17),
])
def test_survey_table(counts, g, crit):
    """SURVEY.md §8(e) '[derived] Best sequence-only partitions, by brute force'."""
    got, groups = plan_groups(list(counts), g)
    assert got == crit
    assert sorted(n for grp in set(groups) for n in grp) == sorted(counts)


@pytest.mark.parametrize("nmax,g", [(12, 2), (16, 3), (22, 4), (30, 3), (30, 8), (22, 6), (30, 5), (16, 5)])
def test_reaches_the_lower_bound(nmax, g):
    counts = list(range(2, nmax + 1, 2))
    S = sum(n + 1 for n in counts)
    lower = max(-(-S // g), nmax + 1)
    got, groups = plan_groups(counts, g)
    assert got == lower, (counts, g, groups)


def test_matches_exhaustive_search_on_random_sets():
    rng = random.Random(1907)
    for _ in range(40):
        m = rng.randint(1, 8)
        counts = sorted(rng.sample(range(2, 61, 2), m))
        g = rng.randint(1, min(m, 4))
        got, groups = plan_groups(counts, g)
        assert got == brute_force(counts, g), (counts, g, groups)
        loads = [sum(n + 1 for n in grp) for grp in set(groups)]
        assert max(loads) == got


def test_large_set_finishes():
    """m = 32 (the ABI's maximum) still plans quickly and reaches the bound."""
    counts = list(range(2, 65, 2))
    got, _ = plan_groups(counts, 8)
    S = sum(n + 1 for n in counts)
    assert got == max(-(-S // 8), 65)
