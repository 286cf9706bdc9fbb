"""Randomized parity at scale (a stand-in for racecheck, which is closed on
this pool): any shared-memory race or ordering bug shows up as a record that
differs from the oracle or between block sizes.

* thousands of run_cse processes over random systems, all strategies, random
  alpha/beta/p/seed, including multi-word masks (65-250 expressions, W = 2..4)
* identical records for every block size the kernel is instantiated with
* optimize_system on multi-word systems against the oracle
"""
import os
import random

import pytest

import paper_2512_13365_b200 as T
from helpers import o_optimize_system, o_run_cse, random_system

pytestmark = pytest.mark.gpu


def rand_cfg(rng):
    return T.ProcessConfig(rng.randrange(7), alpha=rng.choice([0.0, rng.random() * 0.5]), beta=0.5 + rng.random() * 0.5,
                           p_greedy=0.5 + rng.random() * 0.5, seed=rng.getrandbits(64))


def tall_system(rng, n_e, n_x, density):
    rows = []
    for _ in range(n_e):
        row = [v if rng.random() < 0.5 else -v for v in range(1, n_x + 1) if rng.random() < density]
        rows.append(row)
    return n_x, rows


def test_run_cse_random_at_scale(dev):
    rng = random.Random(4242)
    checked = 0
    for _ in range(24):
        sys_ = random_system(rng, 30, 14)
        cfgs = [rand_cfg(rng) for _ in range(48)]
        recs = T.run_cse(sys_, cfgs)
        for cfg, rec in zip(cfgs, recs):
            assert (rec.substitutions, rec.cost) == o_run_cse(sys_, cfg), cfg
            checked += 1
    assert checked == 24 * 48


@pytest.mark.parametrize("n_e,n_x,density", [(70, 10, 0.3), (130, 12, 0.25), (200, 9, 0.3), (250, 14, 0.15)])
def test_run_cse_multiword(dev, n_e, n_x, density):
    rng = random.Random(n_e * 7 + n_x)
    sys_ = tall_system(rng, n_e, n_x, density)
    cfgs = [rand_cfg(rng) for _ in range(21)]
    recs = T.run_cse(sys_, cfgs)
    for cfg, rec in zip(cfgs, recs):
        assert (rec.substitutions, rec.cost) == o_run_cse(sys_, cfg), cfg


def test_block_sizes_agree():
    rng = random.Random(77)
    systems = [random_system(rng, 30, 14) for _ in range(6)] + [tall_system(rng, 90, 10, 0.3)]
    cfgs = [rand_cfg(rng) for _ in range(40)]
    results = {}
    old = os.environ.get("TCSE_NT")
    try:
        for nt in ("32", "64", "128", "256"):
            os.environ["TCSE_NT"] = nt
            d = T.Device(0)  # the block size is read when a context is created
            results[nt] = [[(r.substitutions, r.cost) for r in T.run_cse(s, cfgs, device=d)] for s in systems]
            d.close()
    finally:
        if old is None:
            os.environ.pop("TCSE_NT", None)
        else:
            os.environ["TCSE_NT"] = old
    base = results["64"]
    for nt, r in results.items():
        assert r == base, nt


def test_optimize_multiword_against_oracle(dev):
    rng = random.Random(9)
    for n_e, n_x in ((80, 9), (150, 8)):
        sys_ = tall_system(rng, n_e, n_x, 0.3)
        cfg = T.SearchConfig(n_processes=24, patience=2, master_seed=rng.getrandbits(64))
        rec, it = T.optimize_system(sys_, cfg, stream_salt=1)
        o = o_optimize_system(sys_, cfg, salt=1)
        assert (rec.substitutions, rec.cost, it) == (o["subs"], o["cost"], o["iterations"])


def test_bench_workload_parity_at_scale(dev):
    """The bench workload itself (S(x)S 4x4x4:49, default mixed weights,
    reinit 0.4, U/V/W concurrent) at 4096 processes for 2 iterations (the
    second with prefix sharing) against the oracle: identical incumbents and
    identical substitution-step counts."""
    from helpers import fixture_systems
    systems = fixture_systems("sxs")
    cfg = T.SearchConfig(n_processes=4096, patience=1 << 20, master_seed=1, max_iterations=2)
    st = {}
    got = T.optimize_systems(systems, cfg, [0, 1, 2], stats=st)
    steps = 0
    for c, (sys_, (rec, it)) in enumerate(zip(systems, got)):
        o = o_optimize_system(sys_, cfg, salt=c)
        assert (rec.substitutions, rec.cost, rec.strategy, rec.seed, it) == (o["subs"], o["cost"], o["strategy"],
                                                                             o["seed"], o["iterations"])
        steps += o["steps"]
    assert st["steps"] == steps
