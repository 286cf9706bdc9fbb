"""Pins the C restatement (oracle/liboracle.so) against the reference itself
(oracle/_ref/libterncse_ref.so, compiled from /root/reference): bit-identical
RNG streams, pair counts, run_cse records for all 7 strategies,
assign_strategies slots, pick_reinit sets and optimize_system results."""
import ctypes as C
import random

import pytest

import paper_2512_13365_b200 as T
from helpers import o_count_pairs, o_optimize_system, o_run_cse, random_system
from oracle_lib import have_reference, oracle, reference
from paper_2512_13365_b200 import _abi

pytestmark = pytest.mark.skipif(not have_reference(), reason="reference build unavailable")


@pytest.mark.parametrize("seed", [0, 1, 5489, 2**63 + 11, 2**64 - 1])
def test_mt19937_64_and_distributions(seed):
    o, r = oracle(), reference()
    a, b = (C.c_uint64 * 2000)(), (C.c_uint64 * 2000)()
    o.or_mt19937_64(seed, 2000, a)
    r.ref_mt19937_64(seed, 2000, b)
    assert list(a) == list(b)
    for lo, hi in [(0, 1), (1, 1), (0, 0), (1, 7), (0, 2**40), (3, 2**63), (1, 3), (0, 12)]:
        o.or_uniform_int(seed, lo, hi, 2000, a)
        r.ref_uniform_int(seed, lo, hi, 2000, b)
        assert list(a) == list(b), (lo, hi)
    x, y = (C.c_double * 2000)(), (C.c_double * 2000)()
    for lo, hi in [(0.0, 1.0), (0.0, 0.5), (0.5, 1.0)]:
        o.or_uniform_real(seed, lo, hi, 2000, x)
        r.ref_uniform_real(seed, lo, hi, 2000, y)
        assert list(x) == list(y)


def test_mix_seed():
    o, r = oracle(), reference()
    rng = random.Random(3)
    for _ in range(200):
        parts = (C.c_uint64 * 4)(*[rng.getrandbits(64) for _ in range(4)])
        assert o.or_mix_seed(parts, 4) == r.ref_mix_seed(parts, 4)


def test_count_pairs_random_states():
    rng = random.Random(2024)
    for _ in range(150):
        sys_ = random_system(rng, 50, 12)
        prefix = []
        for _ in range(rng.randint(0, 3)):
            cands = o_count_pairs(sys_, prefix, 2)
            if not cands:
                break
            prefix.append(rng.choice(cands)[0])
        assert o_count_pairs(sys_, prefix, 1) == o_count_pairs(sys_, prefix, 1, which="reference")


def test_run_cse_all_strategies():
    rng = random.Random(606)
    for _ in range(120):
        sys_ = random_system(rng, 14, 10)
        for k in range(7):
            cfg = T.ProcessConfig(k, alpha=rng.choice([0.0, rng.random() * 0.5]), beta=0.5 + rng.random() * 0.5,
                                  p_greedy=0.5 + rng.random() * 0.5, seed=rng.getrandbits(64))
            assert o_run_cse(sys_, cfg) == o_run_cse(sys_, cfg, which="reference")


def test_assign_strategies_and_reinit():
    o, r = oracle(), reference()
    a, b = (_abi.ProcessConfig * 700)(), (_abi.ProcessConfig * 700)()
    for forced in (-1, 0, 4):
        cfg = T.SearchConfig(master_seed=31, forced_strategy=None if forced < 0 else forced).to_c()
        for it in (1, 2, 9):
            for salt in (0, 1, 2):
                assert o.or_assign_strategies(C.byref(cfg), it, 700, salt, a) == 0
                assert r.ref_assign_strategies(C.byref(cfg), it, 700, salt, b) == 0
                assert all(bytes(a[p]) == bytes(b[p]) for p in range(700))
    rng = random.Random(1)
    for _ in range(60):
        n = rng.randint(1, 400)
        costs = (C.c_int32 * n)(*[rng.randint(0, 12) for _ in range(n)])
        f = rng.choice([0.0, 0.4, 0.5, 1.0, 0.33, 0.999])
        x, y = (C.c_uint8 * n)(), (C.c_uint8 * n)()
        o.or_pick_reinit(costs, n, f, x)
        r.ref_pick_reinit(costs, n, f, y)
        assert list(x) == list(y)


@pytest.mark.parametrize("forced", [None, 0, 1, 4, 5])
def test_optimize_system(forced):
    rng = random.Random(77 + (forced or 0))
    for _ in range(3):
        sys_ = random_system(rng, 20, 10, 15, 8)
        cfg = T.SearchConfig(n_processes=16, patience=3, master_seed=rng.getrandbits(64), forced_strategy=forced)
        a = o_optimize_system(sys_, cfg, salt=2)
        b = o_optimize_system(sys_, cfg, salt=2, which="reference", threads=3)
        assert a == b


def test_counted_replica_equals_real_optimize_system():
    rng = random.Random(5)
    for _ in range(4):
        sys_ = random_system(rng, 20, 10, 15, 8)
        cfg = T.SearchConfig(n_processes=24, patience=3, master_seed=rng.getrandbits(64))
        s = _abi.make_system(*sys_)
        rec = _abi.make_record(200)
        it = C.c_int32()
        assert reference().ref_optimize_system(C.byref(s), C.byref(cfg.to_c()), 1, 4, C.byref(rec), C.byref(it)) == 0
        b = o_optimize_system(sys_, cfg, salt=1, which="reference", threads=4)
        assert _abi.record_subs(rec) == b["subs"] and rec.cost == b["cost"] and it.value == b["iterations"]
