"""Prefix snapshots (search.cu build_snapshots) never change results: every
reinit process ends in the same state whether it copies a snapshot, part of
one, or replays the whole prefix itself (TCSE_SNAP=0) — records, costs,
iteration and step counts equal the oracle's either way, on the headline
scheme and a 5x5x5 one, including a capacity-retry run (shrunk lists)."""
import pytest

import paper_2512_13365_b200 as T
from helpers import fixture_systems, o_optimize_system

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("snap", ["1", "0"])
@pytest.mark.parametrize("name,comp,n", [("sxs", 2, 512), ("sxs", 0, 384), ("naive555_f1000", 2, 256)])
def test_snapshots_match_oracle(dev, monkeypatch, snap, name, comp, n):
    monkeypatch.setenv("TCSE_SNAP", snap)
    sys_ = fixture_systems(name)[comp]
    cfg = T.SearchConfig(n_processes=n, patience=3, master_seed=11, max_iterations=4)
    st = {}
    rec, it = T.optimize_system(sys_, cfg, stream_salt=comp, stats=st)
    o = o_optimize_system(sys_, cfg, salt=comp)
    assert (rec.substitutions, rec.cost, it, st["steps"]) == (o["subs"], o["cost"], o["iterations"], o["steps"])
    assert st["replayed"] > 0  # reinit processes ran (iterations 2..)


def test_snapshots_with_capacity_retry(dev, monkeypatch):
    # zero capacity slack: lists that grow force full-capacity re-runs of an
    # iteration, whose builder publishes the snapshots again
    monkeypatch.setenv("TCSE_MCAP_SLACK", "0")
    sys_ = fixture_systems("sxs")[2]
    cfg = T.SearchConfig(n_processes=512, patience=3, master_seed=5, max_iterations=4)
    rec, it = T.optimize_system(sys_, cfg, stream_salt=2)
    o = o_optimize_system(sys_, cfg, salt=2)
    assert (rec.substitutions, rec.cost, it) == (o["subs"], o["cost"], o["iterations"])
