"""GPU parity: the sm_100a search path (through the C ABI) against the oracle.

Bit-exact integer parity everywhere: pair counts, candidate lists at every
step, substitution sequences and costs for ALL seven strategies (the device
replays the reference's mt19937_64 streams), optimize_system records,
iteration counts and step counts.  The oracle (oracle/liboracle.so) is itself
pinned against the compiled reference in test_oracle_pin.py.
"""
import random

import pytest

import paper_2512_13365_b200 as T
from helpers import (EXAMPLE, fixture_systems, o_count_pairs, o_optimize_system, o_run_cse,
                     o_sequence_fnv, random_system)

pytestmark = pytest.mark.gpu


def rand_cfg(rng, strategy):
    return T.ProcessConfig(strategy, alpha=rng.choice([0.0, rng.random() * 0.5]), beta=0.5 + rng.random() * 0.5,
                           p_greedy=0.5 + rng.random() * 0.5, seed=rng.getrandbits(64))


def test_worked_example_counts(dev):
    # test_linear_system.cpp:48-58
    got = dict(T.count_pairs(EXAMPLE, min_count=1))
    assert got[(2, 4, 1)] == 2
    assert got[(1, 3, -1)] == 2
    assert got[(1, 2, 1)] == 1
    assert got[(1, 2, -1)] == 2
    assert T.count_pairs(EXAMPLE, min_count=1) == o_count_pairs(EXAMPLE)


def test_count_pairs_random_states(dev):
    rng = random.Random(2024)
    for _ in range(60):
        sys = random_system(rng, 50, 12)
        # walk a few random substitutions so fresh variables enter the counts
        prefix = []
        for _ in range(rng.randint(0, 4)):
            cands = o_count_pairs(sys, prefix, 2)
            if not cands:
                break
            prefix.append(rng.choice(cands)[0])
        for minc in (1, 2):
            assert T.count_pairs(sys, prefix, minc) == o_count_pairs(sys, prefix, minc)


@pytest.mark.parametrize("name", ["laderman", "sxs", "sxs_border", "naive555_f1000"])
def test_count_pairs_fixtures(dev, name):
    for sys in fixture_systems(name):
        assert T.count_pairs(sys, (), 2) == o_count_pairs(sys, (), 2)


def test_run_cse_all_strategies_random(dev):
    rng = random.Random(606)
    for _ in range(25):
        sys = random_system(rng, 14, 10)
        cfgs = [rand_cfg(rng, k) for k in range(7) for _ in range(6)]
        recs, traces = T.run_cse(sys, cfgs, trace_stride=64)
        for cfg, rec, tr in zip(cfgs, recs, traces):
            subs, cost, otr = o_run_cse(sys, cfg, trace_cap=64)
            assert rec.substitutions == subs, (sys, cfg)
            assert rec.cost == cost
            assert tr == otr
            assert rec.strategy == cfg["strategy"] and rec.seed == cfg["seed"]


@pytest.mark.parametrize("name", ["laderman", "sxs"])
def test_run_cse_all_strategies_fixtures(dev, name):
    rng = random.Random(hash(name) & 0xffff)
    for sys in fixture_systems(name):
        cfgs = [rand_cfg(rng, k) for k in range(7) for _ in range(3)]
        recs = T.run_cse(sys, cfgs)
        for cfg, rec in zip(cfgs, recs):
            subs, cost = o_run_cse(sys, cfg)
            assert rec.substitutions == subs and rec.cost == cost, cfg


def test_run_cse_with_prefix(dev):
    rng = random.Random(77)
    sys = fixture_systems("sxs")[2]
    g = T.run_cse(sys, [T.ProcessConfig(0)])[0]
    for k in (1, 5, 20):
        prefix = g.substitutions[:k]
        cfgs = [rand_cfg(rng, s) for s in range(7)]
        recs = T.run_cse(sys, cfgs, prefix)
        for cfg, rec in zip(cfgs, recs):
            assert (rec.substitutions, rec.cost) == o_run_cse(sys, cfg, prefix)


# SURVEY.md Appendix C, regenerated from the reference (tests/golden/greedy.json)
GREEDY = {
    "laderman": [(18, 6, 0x60e62426707cfa4c), (18, 6, 0xc11c64a1e07d531c), (34, 5, 0x551124fab2393785)],
    "sxs": [(59, 18, 0x36fd7a5f61c82d89), (59, 18, 0x36fd7a5f61c82d89), (88, 40, 0x751888f0b0445915)],
    "sxl": [(185, 73, 0x00cc607c22dccea6), (189, 71, 0x4ee7134f288b34b0), (303, 163, 0x12ca999b253e94c2)],
    "strassen": [(5, 0, 0xcbf29ce484222325), (5, 0, 0xcbf29ce484222325), (8, 0, 0xcbf29ce484222325)],
}


@pytest.mark.parametrize("name", sorted(GREEDY))
def test_greedy_goldens(dev, name):
    for sys, (cost, steps, fnv) in zip(fixture_systems(name), GREEDY[name]):
        rec = T.run_cse(sys, [T.ProcessConfig(0)])[0]
        assert rec.cost == cost
        assert len(rec.substitutions) == steps
        assert o_sequence_fnv(rec.substitutions) == fnv
        ok, c = T.verify_record(sys, rec.substitutions)
        assert ok and c == cost


def test_replay_error_names_position(dev):
    # test_cse_engine.cpp:87-91
    with pytest.raises(T.TcseError) as e:
        T.run_cse(EXAMPLE, [T.ProcessConfig(0)], prefix=[(2, 4, 1), (2, 4, 1)])
    assert "position 1" in str(e.value)


@pytest.mark.parametrize("forced", [None, 0, 4])
def test_optimize_system_matches_oracle(dev, forced):
    rng = random.Random(1234 + (forced or 9))
    for _ in range(4):
        sys = random_system(rng, 20, 10, 15, 8)
        cfg = T.SearchConfig(n_processes=12, patience=3, master_seed=rng.getrandbits(64), forced_strategy=forced)
        st = {}
        rec, it = T.optimize_system(sys, cfg, stats=st)
        o = o_optimize_system(sys, cfg)
        assert rec.substitutions == o["subs"] and rec.cost == o["cost"]
        assert (rec.strategy, rec.seed, it) == (o["strategy"], o["seed"], o["iterations"])
        assert st["steps"] == o["steps"]


@pytest.mark.parametrize("name", ["laderman", "sxs"])
def test_optimize_scheme_components_match_oracle(dev, name):
    systems = fixture_systems(name)
    cfg = T.SearchConfig(n_processes=64, patience=3, master_seed=1)
    st = {}
    got = T.optimize_systems(systems, cfg, [0, 1, 2], stats=st)
    steps = 0
    for c, (sys, (rec, it)) in enumerate(zip(systems, got)):
        o = o_optimize_system(sys, cfg, salt=c)
        assert rec.substitutions == o["subs"] and rec.cost == o["cost"] and it == o["iterations"]
        steps += o["steps"]
    assert st["steps"] == steps


def test_strassen_scheme_18(dev):
    # test_parallel_search.cpp:129-141
    s = T.load_scheme(__import__("helpers").SCHEMES + "/strassen.json")
    rep = T.optimize_scheme(s, T.SearchConfig(n_processes=16, patience=2))
    assert rep["total"] == 18
    assert [c["cost"] for c in rep["components"]] == [5, 5, 8]
    assert all(not c["record"].substitutions for c in rep["components"])


def test_worked_example_portfolio_reaches_6(dev):
    # test_parallel_search.cpp:89-98
    rec, _ = T.optimize_system(EXAMPLE, T.SearchConfig(n_processes=64, patience=3, master_seed=42))
    assert rec.cost == 6
    assert T.verify_record(EXAMPLE, rec.substitutions) == (True, 6)


def test_single_process_greedy_portfolio_equals_run_cse(dev):
    # test_parallel_search.cpp:73-87
    w = [0.0] * 7
    w[0] = 1.0
    rec, _ = T.optimize_system(EXAMPLE, T.SearchConfig(n_processes=1, patience=1, strategy_weights=w))
    direct = T.run_cse(EXAMPLE, [T.ProcessConfig(0)])[0]
    assert rec.substitutions == direct.substitutions and rec.cost == direct.cost


def test_incumbent_non_increasing(dev):
    rng = random.Random(88)
    sys = random_system(rng, 25, 12, 20, 10)
    seen = []
    T.optimize_system(sys, T.SearchConfig(n_processes=16, patience=4, master_seed=5),
                      on_iteration=lambda it, rec: seen.append((it, rec.cost)) and False)
    assert [it for it, _ in seen] == list(range(1, len(seen) + 1))
    assert all(a[1] >= b[1] for a, b in zip(seen, seen[1:]))


def test_config_errors(dev):
    with pytest.raises(T.TcseError, match="reinit_fraction"):
        T.optimize_system(EXAMPLE, T.SearchConfig(reinit_fraction=1.5))
    with pytest.raises(T.TcseError, match="patience"):
        T.optimize_system(EXAMPLE, T.SearchConfig(patience=0))
    with pytest.raises(T.TcseError, match="all strategy weights are zero"):
        T.optimize_system(EXAMPLE, T.SearchConfig(strategy_weights=[0.0] * 7))
