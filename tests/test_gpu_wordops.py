"""The roofline's work counter against an independent host
count: per selected step 12 (V - 1) W_E + 8 W_E + m, plus the coins drawn
(sum of candidate degrees) for a Greedy-Intersections step and m (V - 2) 4 W_E
for a Greedy-Potential step.  The kernel sums the V terms in closed form after
its loop; here every step's list comes from the oracle's count_pairs on the
replayed prefix."""
import random

import pytest

import paper_2512_13365_b200 as T
from helpers import fixture_systems, o_count_pairs

pytestmark = pytest.mark.gpu


def expected_wops(sys_, subs, strategy):
    n_x, rows = sys_
    we = (len(rows) + 63) // 64
    total = 0
    for t in range(len(subs)):
        cands = [k for k, c in o_count_pairs(sys_, subs[:t], min_count=2)]
        m = len(cands)
        V = n_x + t
        total += 12 * (V - 1) * we + 8 * we + m
        if strategy == 4:  # coins: candidates sharing a variable, q and its twin excluded
            per_var = {}
            for (i, j, s) in cands:
                per_var[i] = per_var.get(i, 0) + 1
                per_var[j] = per_var.get(j, 0) + 1
            keys = set(cands)
            for (i, j, s) in cands:
                twin = 1 if (i, j, -s) in keys else 0
                total += per_var[i] + per_var[j] - 2 - twin
        elif strategy == 6:
            total += m * (V - 2) * 4 * we
    return total


@pytest.mark.parametrize("name,comp", [("laderman", 2), ("sxs", 0), ("sxs", 2)])
@pytest.mark.parametrize("strategy", [0, 1, 2, 4, 6])
def test_wordops_match_host_count(name, comp, strategy):
    sys_ = fixture_systems(name)[comp]
    rng = random.Random(100 * strategy + comp)
    cfgs = [T.ProcessConfig(strategy, alpha=0.1 + 0.4 * rng.random(), beta=0.5 + 0.5 * rng.random(),
                            seed=rng.getrandbits(64)) for _ in range(3)]
    st = {}
    recs = T.run_cse(sys_, cfgs, stats=st)
    want = sum(expected_wops(sys_, r.substitutions, strategy) for r in recs)
    assert st["wops"] == want
