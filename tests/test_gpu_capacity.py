"""Shrunk session capacity and its exact fallback (host.cpp shrink_capacity /
search_step_begin): session layouts are sized for the starting candidate list
plus slack; a process whose list outgrows it flags an overflow and the session
re-runs that iteration at full capacity.  Results must equal the oracle's
whether or not the fallback fires."""
import pytest

import paper_2512_13365_b200 as T
from helpers import fixture_systems, o_count_pairs, o_optimize_system

# m grows: substituting (1,2) consumes one candidate and leaves (1,3), (2,3),
# (1,4), (2,4) at count 2 while creating (3,5), (4,5): 6 -> 7 candidates
GROW = (4, [[1, 2, 3, 4], [1, 2, 3, 4], [1, 3], [1, 3], [2, 3], [2, 3], [1, 4], [1, 4], [2, 4], [2, 4]])


def test_growth_system_grows():
    assert len(o_count_pairs(GROW, (), 2)) == 6
    assert len(o_count_pairs(GROW, [(1, 2, 1)], 2)) == 7


@pytest.mark.gpu
@pytest.mark.parametrize("slack", ["0", "1", "64"])
def test_overflow_rerun_matches_oracle(dev, monkeypatch, slack):
    monkeypatch.setenv("TCSE_MCAP_SLACK", slack)
    for seed in range(1, 7):
        cfg = T.SearchConfig(n_processes=64, patience=4, master_seed=seed)
        st = {}
        rec, it = T.optimize_system(GROW, cfg, stats=st)
        o = o_optimize_system(GROW, cfg)
        assert (rec.substitutions, rec.cost, it, st["steps"]) == (o["subs"], o["cost"], o["iterations"], o["steps"])
        if slack == "0" and seed == 1:
            assert st["retries"] >= 1  # the fallback fired and changed nothing


@pytest.mark.gpu
def test_tight_slack_on_fixtures(dev, monkeypatch):
    monkeypatch.setenv("TCSE_MCAP_SLACK", "0")
    for name in ("laderman", "sxs"):
        for sys_ in fixture_systems(name):
            cfg = T.SearchConfig(n_processes=48, patience=2, master_seed=3)
            st = {}
            rec, it = T.optimize_system(sys_, cfg, stats=st)
            o = o_optimize_system(sys_, cfg)
            assert (rec.substitutions, rec.cost, it, st["steps"]) == (o["subs"], o["cost"], o["iterations"],
                                                                   o["steps"])
