"""World-size-2 gloo test of the multi-rank exchange protocol on CPU (no
GPU): each rank runs its slice of global process ids, all-gathers its costs
and local best record, and applies the global argmin / pick_reinit rules of
the device reduce kernel (search.cu reduce_kernel).  The result must equal
the single-process optimize_system (oracle restatement, pinned to the
reference).  The device side of the same protocol is exercised on a GPU by
tests/test_gpu_multirank.py."""
import json
import os
import random
import subprocess
import sys

import pytest

import paper_2512_13365_b200 as T
from helpers import o_optimize_system, random_system

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("seed,n,port", [(3, 12, 29531), (8, 17, 29532)])
def test_two_rank_protocol_equals_single_process(tmp_path, seed, n, port):
    out = str(tmp_path / "mrcpu")
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "mr_cpu_worker.py"), str(seed), str(n), out],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    for p in procs:
        o = p.communicate(timeout=300)[0].decode()
        assert p.returncode == 0, o[-3000:]
    res = [json.load(open(out + ".%d" % r)) for r in range(2)]
    sys_ = random_system(random.Random(seed), 20, 10, 15, 8)
    ref = o_optimize_system(sys_, T.SearchConfig(n_processes=n, patience=3, master_seed=seed))
    for r in res:
        assert [tuple(q) for q in r["subs"]] == ref["subs"]
        assert (r["cost"], r["strategy"], r["seed"], r["iterations"], r["steps"]) == (
            ref["cost"], ref["strategy"], ref["seed"], ref["iterations"], ref["steps"])
