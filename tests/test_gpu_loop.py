"""The device-resident optimize_system loop (session.inc): barrier kernels
advance the loop state in HBM, iterations replay a captured CUDA graph in
batches with one host synchronisation each, and every transport (none, NCCL,
host all-gather between rank threads) gives the single-rank result — which
is the oracle's (parallel_search.hpp:220-273)."""
import json
import os
import subprocess
import sys

import pytest

import paper_2512_13365_b200 as T
from helpers import fixture_systems, o_optimize_system

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rec_tuple(rec, it):
    return (rec.substitutions, rec.cost, rec.strategy, rec.seed, it)


def oracle_tuple(sys_, cfg, salt):
    o = o_optimize_system(sys_, cfg, salt=salt)
    return (o["subs"], o["cost"], o["strategy"], o["seed"], o["iterations"]), o["steps"]


@pytest.mark.parametrize("name,n,patience", [("laderman", 64, 4), ("sxs", 128, 3), ("sxs_border", 48, 3)])
def test_batched_run_matches_oracle(dev, name, n, patience):
    systems = fixture_systems(name)
    cfg = T.SearchConfig(n_processes=n, patience=patience, master_seed=5)
    s = T.Search(systems, cfg, [0, 1, 2], device=dev)
    assert s.run() == 0
    res, st = s.result()
    s.close()
    steps = 0
    for c, (sys_, (rec, it)) in enumerate(zip(systems, res)):
        want, o_steps = oracle_tuple(sys_, cfg, c)
        assert rec_tuple(rec, it) == want
        steps += o_steps
    assert st["steps"] == steps
    assert sum(st["steps_by_strategy"]) == st["steps"]
    its = max(it for _, it in res)
    # graph replays, far fewer host synchronisations than iterations
    assert st["graph_launches"] == its
    assert st["host_syncs"] < its
    assert st["kernel_launches"] > 0 and st["kernel_ms"] > 0 and st["exchange_ms"] > 0


def test_step_by_step_equals_batched(dev):
    systems = fixture_systems("sxs")
    cfg = T.SearchConfig(n_processes=96, patience=3, master_seed=21)
    a = T.Search(systems, cfg, [0, 1, 2], device=dev)
    while a.step() > 0:
        pass
    ra, sa = a.result()
    a.close()
    b = T.Search(systems, cfg, [0, 1, 2], device=dev)
    b.run()
    rb, sb = b.result()
    b.close()
    assert [rec_tuple(r, i) for r, i in ra] == [rec_tuple(r, i) for r, i in rb]
    assert sa["steps"] == sb["steps"] and sa["host_syncs"] > sb["host_syncs"]


def test_max_iterations_on_device(dev):
    systems = fixture_systems("laderman")
    cfg = T.SearchConfig(n_processes=64, patience=1 << 30, master_seed=2, max_iterations=7)
    res = T.optimize_systems(systems, cfg, [0, 1, 2])
    assert [it for _, it in res] == [7, 7, 7]
    for c, (sys_, (rec, it)) in enumerate(zip(systems, res)):
        assert rec_tuple(rec, it) == oracle_tuple(sys_, cfg, c)[0]


def test_eager_and_graph_identical(tmp_path):
    """TCSE_GRAPH=0 enqueues the same sequence without capture."""
    prog = ("import json,sys; sys.path[:0]=[%r,%r]\n"
            "import paper_2512_13365_b200 as T\n"
            "from helpers import fixture_systems\n"
            "st={}\n"
            "r=T.optimize_systems(fixture_systems('sxs'),T.SearchConfig(n_processes=80,patience=3,master_seed=9),"
            "[0,1,2],stats=st)\n"
            "print(json.dumps([[rec.substitutions,rec.cost,rec.seed,it] for rec,it in r]+[st['graph_launches']]))\n"
            % (ROOT, os.path.join(ROOT, "tests")))
    outs = []
    for g in ("1", "0"):
        p = subprocess.run([sys.executable, "-c", prog], env=dict(os.environ, TCSE_GRAPH=g), capture_output=True,
                           text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    assert outs[0][:-1] == outs[1][:-1]
    assert outs[0][-1] > 0 and outs[1][-1] == 0


def test_callback_runs_every_iteration_and_stops(dev):
    systems = fixture_systems("sxs")
    cfg = T.SearchConfig(n_processes=64, patience=1 << 30, master_seed=3)
    seen = []

    def cb(s, it, rec):
        seen.append((s, it, rec.cost))
        return it >= 4  # stop at the 4th barrier (fixed wall-time budgets work this way)
    res = T.optimize_systems(systems, cfg, [0, 1, 2], on_iteration=cb)
    assert [it for _, it in res] == [4, 4, 4]
    assert sorted((s, it) for s, it, _ in seen) == [(s, it) for s in range(3) for it in range(1, 5)]
    for s, (rec, _) in enumerate(res):
        assert [c for s2, it, c in sorted(seen) if s2 == s][-1] == rec.cost


def test_nccl_one_rank_in_graph():
    """The NCCL transport through the library (ncclAllGather on the context
    stream, captured in the iteration graph) on a one-rank communicator."""
    if not T.lib().tcse_nccl_available():
        pytest.skip("NCCL not loadable")
    d = T.Device(0)
    d.set_nccl(T.Device.nccl_unique_id(), 0, 1)
    systems = fixture_systems("sxs")
    cfg = T.SearchConfig(n_processes=100, patience=3, master_seed=13)
    st = {}
    res = T.optimize_systems(systems, cfg, [0, 1, 2], device=d, stats=st)
    for c, (sys_, (rec, it)) in enumerate(zip(systems, res)):
        assert rec_tuple(rec, it) == oracle_tuple(sys_, cfg, c)[0]
    assert st["graph_launches"] > 0
    d.close()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_device_context_shared_gpu(world):
    """tcse_create_devices' rank threads on one GPU (test transport: host
    all-gather between the threads; NCCL refuses a GPU twice): identical to
    one rank, with and without a callback."""
    os.environ["TCSE_SHARED_DEVICES"] = "1"
    try:
        d = T.Device([0] * world)
    finally:
        os.environ.pop("TCSE_SHARED_DEVICES", None)
    assert d.n_devices == world
    systems = fixture_systems("laderman")
    cfg = T.SearchConfig(n_processes=77, patience=3, master_seed=17)
    res = T.optimize_systems(systems, cfg, [0, 1, 2], device=d)
    for c, (sys_, (rec, it)) in enumerate(zip(systems, res)):
        assert rec_tuple(rec, it) == oracle_tuple(sys_, cfg, c)[0]
    seen = []
    res2 = T.optimize_systems(systems, cfg, [0, 1, 2], device=d,
                              on_iteration=lambda s, it, rec: seen.append(it) or it >= 2)
    assert [it for _, it in res2] == [2, 2, 2] and len(seen) == 6
    d.close()


def test_duplicate_devices_refused():
    with pytest.raises(T.TcseError, match="listed twice"):
        T.Device([0, 0])


def test_wall_budget_on_device_stops_every_system_at_one_barrier(dev):
    """wall_budget_s: the device stops every system at the first barrier after
    the budget (no host turn per iteration); the state is exactly the one
    max_iterations = that many iterations gives (the oracle)."""
    systems = fixture_systems("sxs")
    cfg = T.SearchConfig(n_processes=2048, patience=1 << 30, master_seed=6, wall_budget_s=0.02)
    st = {}
    res = T.optimize_systems(systems, cfg, [0, 1, 2], stats=st)
    its = {it for _, it in res}
    assert len(its) == 1
    k = its.pop()
    assert 1 <= k < 1000 and st["graph_launches"] >= k
    ocfg = T.SearchConfig(n_processes=2048, patience=1 << 30, master_seed=6, max_iterations=k)
    for c, (sys_, (rec, it)) in enumerate(zip(systems, res)):
        assert rec_tuple(rec, it) == oracle_tuple(sys_, ocfg, c)[0]


def test_wall_budget_rank0_decides_for_every_rank():
    os.environ["TCSE_SHARED_DEVICES"] = "1"
    try:
        d = T.Device([0, 0])
    finally:
        os.environ.pop("TCSE_SHARED_DEVICES", None)
    systems = fixture_systems("laderman")
    cfg = T.SearchConfig(n_processes=512, patience=1 << 30, master_seed=8, wall_budget_s=0.01)
    res = T.optimize_systems(systems, cfg, [0, 1, 2], device=d)
    k = res[0][1]
    assert all(it == k for _, it in res)
    ocfg = T.SearchConfig(n_processes=512, patience=1 << 30, master_seed=8, max_iterations=k)
    for c, (sys_, (rec, it)) in enumerate(zip(systems, res)):
        assert rec_tuple(rec, it) == oracle_tuple(sys_, ocfg, c)[0]
    d.close()


def test_negative_wall_budget_rejected(dev):
    with pytest.raises(T.TcseError, match="wall_budget_s"):
        T.optimize_system(fixture_systems("laderman")[0], T.SearchConfig(wall_budget_s=-1.0))
