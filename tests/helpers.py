"""Shared test helpers: seeded random systems (test_util.hpp:74-91 shape),
fixture loading, oracle calls returning Python values."""
import ctypes as C
import json
import os
import random

from oracle_lib import oracle, reference
from paper_2512_13365_b200 import _abi
from paper_2512_13365_b200.scheme import extract_systems, load_scheme

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
SCHEMES = os.path.join(GOLDEN, "schemes")

EXAMPLE = (4, [[1, 2, -3, 4], [1, -2, -4], [1, -2, -3, 4]])  # test_util.hpp:49-53


def random_system(rng, max_exprs, max_vars, min_exprs=1, min_vars=2):
    """random_system (test_util.hpp:74-91) with Python's RNG."""
    n_x = rng.randint(min_vars, max_vars)
    n_e = rng.randint(min_exprs, max_exprs)
    rows = []
    for _ in range(n_e):
        ids = list(range(1, n_x + 1))
        rng.shuffle(ids)
        t = rng.randint(0, n_x)
        rows.append([i if rng.random() < 0.5 else -i for i in ids[:t]])
    return n_x, rows


def fixture_systems(name):
    return extract_systems(load_scheme(os.path.join(SCHEMES, name + ".json")))


def fixture_index():
    with open(os.path.join(SCHEMES, "index.json")) as f:
        return json.load(f)


def lib_of(which):
    return oracle() if which == "oracle" else reference()


def o_count_pairs(sys, prefix=(), min_count=1, which="oracle"):
    L = lib_of(which)
    pfx = "or_" if which == "oracle" else "ref_"
    s = _abi.make_system(*sys)
    pre, npre = _abi.make_pairs(list(prefix))
    cap = 200000
    out = (_abi.PairCount * cap)()
    n = C.c_int32()
    rc = getattr(L, pfx + "count_pairs")(C.byref(s), pre, npre, min_count, out, cap, C.byref(n))
    if rc:
        raise RuntimeError(rc, getattr(L, pfx + "last_error")().decode())
    return [((out[t].pair.i, out[t].pair.j, out[t].pair.rel_sign), out[t].count) for t in range(n.value)]


def o_run_cse(sys, cfg, prefix=(), trace_cap=0, which="oracle"):
    """cfg: paper_2512_13365_b200.ProcessConfig -> (subs, cost[, trace])."""
    s = _abi.make_system(*sys)
    pre, npre = _abi.make_pairs(list(prefix))
    rec = _abi.make_record(_naive(sys) + 1)
    c = cfg.to_c() if hasattr(cfg, "to_c") else cfg
    if which == "oracle":
        tr = (C.c_uint64 * max(1, trace_cap))()
        rc = oracle().or_run_cse(C.byref(s), pre, npre, C.byref(c), C.byref(rec), tr if trace_cap else None,
                                 trace_cap)
        if rc:
            raise RuntimeError(rc, oracle().or_last_error().decode())
        out = (_abi.record_subs(rec), rec.cost)
        if trace_cap:
            return out + ([tr[t] for t in range(min(trace_cap, rec.n_subs + 1))],)
        return out
    rc = reference().ref_run_cse(C.byref(s), pre, npre, C.byref(c), C.byref(rec))
    if rc:
        raise RuntimeError(rc, reference().ref_last_error().decode())
    return _abi.record_subs(rec), rec.cost


def o_optimize_system(sys, cfg, salt=0, which="oracle", threads=1):
    s = _abi.make_system(*sys)
    c = cfg.to_c() if hasattr(cfg, "to_c") else cfg
    rec = _abi.make_record(_naive(sys) + 1)
    it = C.c_int32()
    steps = C.c_uint64()
    if which == "oracle":
        rc = oracle().or_optimize_system(C.byref(s), C.byref(c), salt, C.byref(rec), C.byref(it), C.byref(steps))
        err = oracle().or_last_error
    else:
        secs = C.c_double()
        rc = reference().ref_optimize_system_counted(C.byref(s), C.byref(c), salt, threads, 0.0, C.byref(rec),
                                                     C.byref(it), C.byref(steps), C.byref(secs))
        err = reference().ref_last_error
    if rc:
        raise RuntimeError(rc, err().decode())
    return dict(subs=_abi.record_subs(rec), cost=rec.cost, strategy=rec.strategy, seed=rec.seed,
                iterations=it.value, steps=steps.value)


def o_sequence_fnv(subs):
    arr, n = _abi.make_pairs(list(subs))
    return oracle().or_sequence_fnv(arr, n)


def _naive(sys):
    return sum(len(r) - 1 for r in sys[1] if r)


CHECK_METHOD = {"auto": -1, "exact_brent": 0, "randomized_product": 1}


def ref_check_scheme(s, method="auto", trials=16, seed=0):
    """The reference's verify_brent / verify_by_product / check_scheme_auto
    -> (valid, first_violation or None, method name); raises ValueError with
    the reference's message on a structural error."""
    flat = [(C.c_int8 * max(1, sum(len(r) for r in x)))(*[v for row in x for v in row]) for x in (s["u"], s["v"], s["w"])]
    cs = _abi.Scheme(s["m"], s["n"], s["p"], s["r"], *flat)
    out = _abi.CheckReport()
    lib = reference()
    rc = lib.ref_check_scheme(C.byref(cs), CHECK_METHOD[method], trials, seed, C.byref(out))
    if rc != 0:
        raise ValueError(lib.ref_last_error().decode())
    name = "exact_brent" if out.method == 0 else "randomized_product"
    return (bool(out.valid), None if out.valid else out.first_violation.decode(), name)
