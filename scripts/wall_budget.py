"""Best additions at a fixed wall time, reference CPU path vs the B200 search.

For each scheme: the reference optimize_scheme (oracle/_ref, all host cores,
default config: tier process count, patience 10) runs to convergence; its wall
time T_ref is the budget.  The GPU search (same weights, reinit, patience,
seed) runs with the paper's GPU process counts (16384 for
rank < 100, 8192 below 200, 2048 above) and stops at the first iteration
barrier after T_ref (SearchConfig.wall_budget_s, decided on the device; the
reference side of SURVEY.md 8(d) uses an on_iteration abort).  Every GPU record is re-verified (replay + expand_and_verify).
"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2512_13365_b200 as T  # noqa: E402
from oracle_lib import reference  # noqa: E402


def gpu_count(r):
    return 16384 if r < 100 else (8192 if r < 200 else 2048)


def run(name, seed=1):
    path = os.path.join(ROOT, "tests", "golden", "schemes", name + ".json")
    text = open(path).read()
    s = T.parse_scheme(text)
    ref = reference()
    cfg = T.SearchConfig(master_seed=seed)
    buf = C.create_string_buffer(1 << 24)
    n = C.c_int32()
    t0 = time.time()
    rc = ref.ref_optimize_scheme_json(text.encode(), C.byref(cfg.to_c()), os.cpu_count(), buf, len(buf), C.byref(n))
    t_ref = time.time() - t0
    assert rc == 0, ref.ref_last_error()
    rj = json.loads(buf.value.decode())
    systems = [T.LinearSystem(nx, rows) for nx, rows in T.extract_systems(s)]
    N = gpu_count(s["r"])
    # load this scheme's kernel shapes once (lazy module loading is a one-time
    # process cost, not search time)
    T.optimize_systems(systems, T.SearchConfig(n_processes=64, patience=1, max_iterations=1), [0, 1, 2])
    # the budget is enforced on the device (wall_budget_s: every system stops
    # at the first barrier after it, no host turn per iteration)
    gcfg = T.SearchConfig(n_processes=N, master_seed=seed, wall_budget_s=t_ref)
    start = time.time()
    st = {}
    res = T.optimize_systems(systems, gcfg, [0, 1, 2], stats=st)
    t_gpu = time.time() - start
    stopped_first = any(it > 0 for _, it in res) and t_gpu >= t_ref
    costs = []
    for sys_, (rec, it) in zip(systems, res):
        ok, cost = T.verify_record(sys_, rec.substitutions)
        assert ok and cost == rec.cost
        costs.append(rec.cost)
    # the rest of the budget: more seeds, then the reference's own component-
    # wise combine (parallel_search.hpp:522-547) over every run
    best = list(costs)
    seeds = [seed]
    nxt = seed + 1
    while time.time() - start < t_ref:
        left = t_ref - (time.time() - start)
        scfg = T.SearchConfig(n_processes=N, master_seed=nxt, wall_budget_s=max(left, 1e-6))
        r2 = T.optimize_systems(systems, scfg, [0, 1, 2])
        for c, (sys_, (rec, _)) in enumerate(zip(systems, r2)):
            ok, cost = T.verify_record(sys_, rec.substitutions)
            assert ok and cost == rec.cost
            best[c] = min(best[c], rec.cost)
        seeds.append(nxt)
        nxt += 1
    t_all = time.time() - start
    return {
        "scheme": name, "digest": T.scheme_digest(s), "shape": "%dx%dx%d:%d" % (s["m"], s["n"], s["p"], s["r"]),
        "naive": [T.naive_cost(r) for _, r in T.extract_systems(s)],
        "reference": {"total": rj["total"], "components": [rj["components"][k]["cost"] for k in "uvw"],
                      "processes": rj["config"]["n_processes"], "iterations": rj["iterations"],
                      "wall_s": round(t_ref, 3), "threads": os.cpu_count()},
        "gpu": {"total": sum(costs), "components": costs, "processes": N, "iterations": [it for _, it in res],
                "wall_s": round(t_gpu, 3), "stopped_at_budget": stopped_first, "steps": st["steps"],
                "steps_per_s_device": st["steps"] / max(1e-9, st["kernel_ms"]) * 1e3},
        "gpu_le_reference": sum(costs) <= rj["total"],
        "gpu_seeds_combined": {"total": sum(best), "components": best, "seeds": seeds, "wall_s": round(t_all, 3),
                               "note": "runs with master seeds %d..%d until the reference's wall time, "
                                       "component-wise minimum (the reference's combine)" % (seeds[0], seeds[-1])},
    }


if __name__ == "__main__":
    names = sys.argv[1:] or ["laderman", "sxs", "sxs_border", "naive555_f1000", "sxl", "naive666_f3000"]
    # one untimed call first: CUDA context creation and module load are a
    # one-time process cost, not part of any search (the reference arm runs
    # in an already-loaded library too)
    T.optimize_system((4, [[1, 2, -3, 4], [1, -2, -4], [1, -2, -3, 4]]), T.SearchConfig(n_processes=64, patience=1))
    rows = []
    for nm in names:
        r = run(nm)
        rows.append(r)
        print(json.dumps(r), flush=True)
    out = os.path.join(ROOT, "gpurun_out", "wall_budget.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(rows, open(out, "w"), indent=1)
