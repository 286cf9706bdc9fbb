"""The multi-rank path on one GPU: two ranks (processes) split every
iteration's processes and exchange payloads over gloo; the result must be
identical to the single-rank search and to the oracle (GPU-count
invariance).  No kernel waits on another rank: the exchange
happens on the host between iterations."""
import json
import os
import subprocess
import sys

import pytest

import paper_2512_13365_b200 as T
from helpers import fixture_systems, o_optimize_system

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def run_ranks(mode, name, n, tmp_path, port):
    out = str(tmp_path / ("mr_%s_%s" % (mode, name)))
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "mr_worker.py"), mode, name, str(n), out],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    for p in procs:
        o = p.communicate(timeout=600)[0].decode()
        assert p.returncode == 0, o[-3000:]
    return [json.load(open(out + ".%d" % r)) for r in range(2)]


@pytest.mark.parametrize("mode,port", [("callback", 29611), ("device", 29612)])
@pytest.mark.parametrize("name", ["laderman", "sxs"])
def test_two_ranks_equal_one(tmp_path, mode, port, name):
    n = 96
    port += 10 if name == "sxs" else 0
    ranks = run_ranks(mode, name, n, tmp_path, port)
    cfg = T.SearchConfig(n_processes=n, patience=3, master_seed=11)
    one = T.optimize_systems(fixture_systems(name), cfg, [0, 1, 2])
    for r in ranks:
        assert len(r["records"]) == 3
        for (subs, cost, strat, seed, it), (rec, it1) in zip(r["records"], one):
            assert [tuple(q) for q in subs] == rec.substitutions
            assert (cost, strat, seed, it) == (rec.cost, rec.strategy, rec.seed, it1)
    # steps split across ranks add up to the single-rank count (= the oracle's)
    total = sum(r["steps"] for r in ranks)
    o = sum(o_optimize_system(s, cfg, salt=c)["steps"] for c, s in enumerate(fixture_systems(name)))
    assert total == o
