"""BASELINE configs 3-5 pinned on the device against the reference itself
(oracle/_ref, the unmodified headers compiled here) under the bench's own
workload: default mixed strategy weights, reinit fraction 0.4, hundreds of
processes, several iterations (so iterations >= 2 replay incumbent prefixes),
the bench's launch shapes (NT = 64 / 128 / 256 by list length, the O(deg)
Greedy-Intersections walk on long lists, shrunk candidate capacity with the
full-capacity re-run).  Records, costs, strategies, seeds, iteration counts
and substitution-step counts must all be equal (parallel_search.hpp:220-273).
"""
import json
import os
import subprocess
import sys

import pytest

import paper_2512_13365_b200 as T
from helpers import fixture_systems, o_optimize_system
from oracle_lib import REF_SO

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build absent")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
THREADS = os.cpu_count() or 1


def ref_all(systems, cfg):
    out, steps = [], 0
    for c, s in enumerate(systems):
        o = o_optimize_system(s, cfg, salt=c, which="reference", threads=THREADS)
        out.append((o["subs"], o["cost"], o["strategy"], o["seed"], o["iterations"]))
        steps += o["steps"]
    return out, steps


# (fixture, processes, iterations): config 3 (5x5x5 stand-ins), config 4/5 (6x6x6 stand-ins)
CASES = [("sxs_border", 1024, 3), ("naive555_f1000", 1024, 3), ("sxl", 512, 2), ("naive666_f3000", 512, 2)]


@pytest.mark.parametrize("name,n,its", CASES)
def test_bench_workload_matches_reference(name, n, its):
    systems = fixture_systems(name)
    cfg = T.SearchConfig(n_processes=n, patience=1 << 30, master_seed=1, max_iterations=its)
    st = {}
    got = T.optimize_systems(systems, cfg, [0, 1, 2], stats=st)
    want, steps = ref_all(systems, cfg)
    for (rec, it), w in zip(got, want):
        assert (rec.substitutions, rec.cost, rec.strategy, rec.seed, it) == w
    assert st["steps"] == steps
    assert st["replayed"] > 0  # iterations >= 2 replayed incumbent prefixes
    assert sum(st["steps_by_strategy"]) == st["steps"]


def _run_sub(name, n, its, env):
    prog = ("import json,sys; sys.path[:0]=[%r,%r]\n"
            "import paper_2512_13365_b200 as T\n"
            "from helpers import fixture_systems\n"
            "st={}\n"
            "r=T.optimize_systems(fixture_systems(%r),T.SearchConfig(n_processes=%d,patience=1<<30,master_seed=1,"
            "max_iterations=%d),[0,1,2],stats=st)\n"
            "print(json.dumps([[rec.substitutions,rec.cost,rec.strategy,rec.seed,it] for rec,it in r]"
            "+[st['steps'],st['retries']]))\n" % (ROOT, os.path.join(ROOT, "tests"), name, n, its))
    p = subprocess.run([sys.executable, "-c", prog], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("name,env", [
    ("naive555_f1000", {"TCSE_NT": "256", "TCSE_GI_DENSE": "0"}),   # every system on the walk, 8 warps
    ("naive555_f1000", {"TCSE_NT": "128", "TCSE_MCAP_SLACK": "0"}),  # tightest capacity: re-runs at full size
    ("sxl", {"TCSE_NT": "256", "TCSE_GI_DENSE": "1", "TCSE_GI_BM": "0"}),  # long lists on the dense form
])
def test_forced_launch_shapes_match_reference(name, env):
    n, its = 512, 2
    got = _run_sub(name, n, its, env)
    systems = fixture_systems(name)
    cfg = T.SearchConfig(n_processes=n, patience=1 << 30, master_seed=1, max_iterations=its)
    want, steps = ref_all(systems, cfg)
    for g, w in zip(got[:3], want):
        assert ([tuple(q) for q in g[0]], g[1], g[2], g[3], g[4]) == w
    assert got[3] == steps
