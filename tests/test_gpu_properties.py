"""The reference's own acceptance properties (proj/tests/acceptance.cpp and
test_strategies.cpp / test_parallel_search.cpp), asserted on the device path:

* every record the device produces replays, expands back to the original
  system and carries its total_cost (acceptance 3-4, expand_and_verify);
* alpha = 0 collapses Greedy-Intersections and Greedy-Potential to greedy
  (acceptance 6; test_strategies.cpp:159-169, 252-259);
* mixed weights (1,0,0,0) are Greedy-Intersections on the same stream
  (test_strategies.cpp:203-215: a single positive weight draws nothing);
* the portfolio is never worse than deterministic greedy on flipped schemes
  (acceptance 7);
* reports are byte-identical for any number of ranks (the GPU-count form of
  the reference's thread-count invariance, test_parallel_search.cpp:187-202).
"""
import os
import random

import pytest

import paper_2512_13365_b200 as T
from helpers import fixture_systems, random_system

pytestmark = pytest.mark.gpu


def _records_verify(sys_, recs):
    for rec in recs:
        ok, cost = T.verify_record(sys_, rec.substitutions)
        assert ok and cost == rec.cost


@pytest.mark.parametrize("name", ["laderman", "sxs", "sxs_border"])
def test_every_record_expands_and_costs(dev, name):
    rng = random.Random(11)
    for sys_ in fixture_systems(name):
        cfgs = [T.ProcessConfig(k % 7, alpha=rng.random() * 0.5, beta=0.5 + rng.random() * 0.5,
                                p_greedy=0.5 + rng.random() * 0.5, seed=rng.getrandbits(64)) for k in range(210)]
        _records_verify(sys_, T.run_cse(sys_, cfgs))


def test_every_record_expands_random_systems(dev):
    rng = random.Random(5)
    for _ in range(60):
        sys_ = random_system(rng, 14, 10)
        cfgs = [T.ProcessConfig(k, seed=rng.getrandbits(64)) for k in range(7)]
        _records_verify(sys_, T.run_cse(sys_, cfgs))


def test_alpha_zero_collapses_to_greedy(dev):
    rng = random.Random(3)
    for _ in range(100):
        sys_ = random_system(rng, 12, 9)
        seed = rng.getrandbits(64)
        g, gi, gp = T.run_cse(sys_, [T.ProcessConfig(0, seed=seed), T.ProcessConfig(4, alpha=0.0, seed=seed),
                                     T.ProcessConfig(6, alpha=0.0, seed=seed)])
        assert gi.substitutions == g.substitutions and gp.substitutions == g.substitutions
        assert gi.cost == g.cost == gp.cost


def test_mixed_single_weight_is_gi(dev):
    rng = random.Random(90)
    for r in range(60):
        sys_ = random_system(rng, 12, 8)
        mixed, gi = T.run_cse(sys_, [T.ProcessConfig(5, alpha=0.35, beta=0.8, seed=r, mix_weights=(1, 0, 0, 0)),
                                     T.ProcessConfig(4, alpha=0.35, beta=0.8, seed=r)])
        assert mixed.substitutions == gi.substitutions and mixed.cost == gi.cost


def test_portfolio_never_worse_than_greedy_on_flipped(dev):
    naive = T.naive_scheme(3, 3, 3)
    for seed in range(8):
        s = T.flip_walk(naive, 1000 + seed, 40)
        greedy = T.optimize_scheme(s, T.SearchConfig(n_processes=1, forced_strategy="greedy", patience=1))
        best = T.optimize_scheme(s, T.SearchConfig(n_processes=64, patience=3, master_seed=seed))
        assert best["total"] <= greedy["total"]


def test_reports_identical_for_any_world_size():
    s = T.load_scheme(os.path.join(os.path.dirname(__file__), "golden", "schemes", "laderman.json"))
    cfg = T.SearchConfig(n_processes=96, patience=3, master_seed=4)
    texts = []
    for world in (1, 2, 3):
        os.environ["TCSE_SHARED_DEVICES"] = "1"
        try:
            d = T.Device([0] * world) if world > 1 else T.Device(0)
        finally:
            os.environ.pop("TCSE_SHARED_DEVICES", None)
        texts.append(T.report_to_json(T.optimize_scheme(s, cfg, device=d)))
        d.close()
    assert texts[0] == texts[1] == texts[2]
