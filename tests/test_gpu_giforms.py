"""Both exact Greedy-Intersections forms against the oracle (search.cu
sel_gi / add_run): the dense layout (TCSE_GI_DENSE=1) and the O(deg) walk
(TCSE_GI_DENSE=0), forced on the same processes — each both with near-best
pruning (default: approximate scores from exact integer sums, exact folds only
within the rounding bound of the best; dense: gi_score_bm or gi_pass, then
gi_fold_dense) and
without it (TCSE_GI_PRUNE=0: the walk folds every candidate, the dense layout
runs the reference loop itself, branch-free over bitmaps for lists of at most
32 candidates).

The walk adds runs of disjoint candidates in O(1), including the binade
crossings of the running double sum: by binary search below max(c-1)+1 and
in closed form above it.  The cases below push both regimes: high pair counts
(tall systems: many expressions over few variables, so c-1 is large and the
sum crosses many binades), betas whose products have full 52-bit fractions,
beta = 0 (integer sums), beta > 1, tiny beta, and negative beta (the walk
layout then runs the reference loop); negative alpha (every score below -1:
the block argmax must still return a real candidate, as the reference's
first-candidate rule does — for gp too).  Records and per-step candidate-list
traces must equal the oracle's in every case."""
import random

import pytest

import paper_2512_13365_b200 as T
from helpers import fixture_systems, o_optimize_system, o_run_cse, random_system

pytestmark = pytest.mark.gpu

BETAS = [0.5, 0.75, 0.6180339887498949, 1.0, 0.0, 3.7, 1e-300, 0.9999999999999999, -0.6]


def tall_system(rng, n_e, n_x, density):
    rows = []
    for _ in range(n_e):
        rows.append([v if rng.random() < 0.5 else -v for v in range(1, n_x + 1) if rng.random() < density])
    return n_x, rows


def gi_cfgs(rng, n):
    out = []
    for t in range(n):
        beta = BETAS[t % len(BETAS)] if t < len(BETAS) else 0.5 + rng.random() * 0.5
        strategy = 4 if t % 3 else 5  # gi, and mixed (which draws gi among others)
        out.append(T.ProcessConfig(strategy, alpha=rng.choice([0.05, 0.3, 0.5, 1.7, -0.4, -3.0]), beta=beta,
                                   p_greedy=0.5 + rng.random() * 0.5, seed=rng.getrandbits(64)))
    return out


def cyclic_system(n, offsets, copies):
    """Rows {r, r+o1, r+o2, ...} (mod n), each repeated: every candidate has the
    same count and the same number of intersecting candidates, so approximate
    gi scores tie exactly whenever coin sums do (the pruned walk then folds
    several near-best candidates per thread, including its rescan path)."""
    rows = []
    for r in range(n):
        row = [(r + o) % n + 1 for o in offsets]
        for k in range(copies):
            rows.append([v if (k + i) % 3 else -v for i, v in enumerate(row)] if k % 2 else list(row))
    return n, rows


def systems(rng):
    # small lists first (<= 32 candidates: the small-list instantiation)
    out = [fixture_systems("laderman")[0], fixture_systems("laderman")[2], random_system(rng, 18, 8)]
    out += [random_system(rng, 40, 12) for _ in range(4)]
    out += [cyclic_system(100, (0, 1, 3), 2), cyclic_system(64, (0, 1, 2, 5), 3)]
    out += [tall_system(rng, 90, 8, 0.45), tall_system(rng, 200, 9, 0.35), tall_system(rng, 250, 14, 0.2)]
    out += [fixture_systems("sxs")[2], fixture_systems("naive555_f1000")[2]]
    return out


def set_form(monkeypatch, form):
    """form: '<dense>[-exact][-nobm|-plain]'.  Dense pruned scoring uses the
    per-variable candidate bitmaps (gi_score_bm) or the full-list pass
    (gi_pass, -nobm); dense without pruning (-exact) runs the reference loop —
    branch-free over the bitmaps in the small-list instantiation for lists of
    at most 32 candidates (gi_dense_small), the plain loop otherwise or with
    -plain (TCSE_GI_SMALL=0)."""
    monkeypatch.setenv("TCSE_GI_DENSE", form[0])
    monkeypatch.setenv("TCSE_GI_PRUNE", "0" if "exact" in form else "1")
    monkeypatch.setenv("TCSE_GI_BM", "0" if form.endswith("nobm") else "1")
    monkeypatch.setenv("TCSE_GI_SMALL", "0" if form.endswith("plain") else "1")


@pytest.mark.parametrize("form", ["1", "1-nobm", "1-exact", "1-exact-plain", "0", "0-exact"])
def test_gi_forms_match_oracle(dev, monkeypatch, form):
    set_form(monkeypatch, form)
    rng = random.Random(4242)
    for sys_ in systems(rng):
        cfgs = gi_cfgs(rng, 18)
        recs, traces = T.run_cse(sys_, cfgs, trace_stride=32)
        for cfg, rec, tr in zip(cfgs, recs, traces):
            subs, cost, otr = o_run_cse(sys_, cfg, trace_cap=32)
            assert (rec.substitutions, rec.cost) == (subs, cost), (form, cfg)
            assert tr == otr, (form, cfg)


@pytest.mark.parametrize("form", ["1", "0"])
def test_gi_forms_optimize_system(dev, monkeypatch, form):
    monkeypatch.setenv("TCSE_GI_DENSE", form)
    rng = random.Random(99)
    for sys_ in (tall_system(rng, 160, 10, 0.3), fixture_systems("naive555_f1000")[2]):
        cfg = T.SearchConfig(n_processes=96, patience=3, master_seed=5, forced_strategy=4)
        st = {}
        rec, it = T.optimize_system(sys_, cfg, stats=st)
        o = o_optimize_system(sys_, cfg)
        assert (rec.substitutions, rec.cost, it, st["steps"]) == (o["subs"], o["cost"], o["iterations"], o["steps"])


def test_negative_scores_gp(dev):
    rng = random.Random(31)
    for _ in range(6):
        sys_ = random_system(rng, 30, 10)
        cfgs = [T.ProcessConfig(6, alpha=rng.choice([-0.5, -2.0, -7.5]), seed=rng.getrandbits(64)) for _ in range(8)]
        for cfg, rec in zip(cfgs, T.run_cse(sys_, cfgs)):
            assert (rec.substitutions, rec.cost) == o_run_cse(sys_, cfg), cfg


@pytest.mark.parametrize("form", ["1", "1-nobm", "1-exact", "1-exact-plain", "0"])
def test_gi_forms_many_coin_chunks(dev, monkeypatch, form):
    """A coin buffer of one candidate's worth (TCSE_COIN_MAX) splits every gi
    step into many chunks: chunk boundaries, the precleared first chunk and the
    per-chunk near-best folds must still reproduce the oracle."""
    monkeypatch.setenv("TCSE_COIN_MAX", "1")
    set_form(monkeypatch, form)
    rng = random.Random(777)
    for sys_ in systems(rng)[:8]:
        cfgs = gi_cfgs(rng, 12)
        recs, traces = T.run_cse(sys_, cfgs, trace_stride=32)
        for cfg, rec, tr in zip(cfgs, recs, traces):
            subs, cost, otr = o_run_cse(sys_, cfg, trace_cap=32)
            assert (rec.substitutions, rec.cost) == (subs, cost), (form, cfg)
            assert tr == otr, (form, cfg)
