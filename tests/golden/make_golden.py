"""Generates tests/golden/golden.json from the REFERENCE ITSELF (oracle/_ref,
compiled from /root/reference).  Run here: python tests/golden/make_golden.py

Contents (all produced by the unmodified reference code paths):
  greedy         forced-greedy run_cse per fixture component
  run_cse        seeded random systems x 7 strategies: record + cost
  optimize       optimize_system results (record, iterations, counted steps)
  reports        optimize_scheme -> report_to_json bytes (io.hpp:250-266)
"""
import ctypes as C
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from helpers import fixture_systems, o_optimize_system, o_run_cse, o_sequence_fnv, random_system  # noqa: E402
from oracle_lib import reference  # noqa: E402

import paper_2512_13365_b200 as T  # noqa: E402
from paper_2512_13365_b200 import _abi  # noqa: E402


def main():
    g = {"greedy": {}, "run_cse": [], "optimize": [], "reports": {}}
    for name in ("strassen", "laderman", "sxs", "sxl", "sxs_border"):
        rows = []
        for sys_ in fixture_systems(name):
            subs, cost = o_run_cse(sys_, T.ProcessConfig(0), which="reference")
            rows.append(dict(cost=cost, steps=len(subs), fnv="%016x" % o_sequence_fnv(subs), first=subs[:3]))
        g["greedy"][name] = rows
    rng = random.Random(20251218)
    for case in range(40):
        sys_ = random_system(rng, 12, 9)
        for k in range(7):
            cfg = T.ProcessConfig(k, alpha=rng.choice([0.0, round(rng.random() * 0.5, 6)]),
                                  beta=round(0.5 + rng.random() * 0.5, 6), p_greedy=round(0.5 + rng.random() * 0.5, 6),
                                  seed=rng.getrandbits(64))
            subs, cost = o_run_cse(sys_, cfg, which="reference")
            g["run_cse"].append(dict(sys=sys_, cfg=dict(cfg), subs=subs, cost=cost))
    for case in range(6):
        sys_ = random_system(rng, 20, 10, 15, 8)
        cfg = T.SearchConfig(n_processes=12, patience=3, master_seed=rng.getrandbits(64),
                             forced_strategy=[None, None, 0, 4, 6, 1][case])
        o = o_optimize_system(sys_, cfg, salt=case % 3, which="reference", threads=4)
        g["optimize"].append(dict(sys=sys_, cfg=dict(cfg), salt=case % 3, **o))
    ref = reference()
    for name, cfg in (("strassen", T.SearchConfig(n_processes=16, patience=2)),
                      ("laderman", T.SearchConfig(n_processes=32, patience=3, master_seed=7)),
                      ("sxs", T.SearchConfig(n_processes=24, patience=2, master_seed=11))):
        with open(os.path.join(HERE, "schemes", name + ".json")) as f:
            text = f.read()
        buf = C.create_string_buffer(1 << 22)
        n = C.c_int32()
        c = cfg.to_c()
        rc = ref.ref_optimize_scheme_json(text.encode(), C.byref(c), 4, buf, len(buf), C.byref(n))
        assert rc == 0, ref.ref_last_error()
        g["reports"][name] = dict(cfg=dict(cfg), json=buf.value.decode())
    # emit_slp (io.hpp:352-393) of each report, and combine_componentwise of two
    # laderman reports (parallel_search.hpp:522-547), from the reference
    ref.ref_emit_slp.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int32, C.POINTER(C.c_int32)]
    ref.ref_combine_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int32, C.POINTER(C.c_int32)]
    for name, r in g["reports"].items():
        with open(os.path.join(HERE, "schemes", name + ".json")) as f:
            text = f.read()
        buf = C.create_string_buffer(1 << 22)
        n = C.c_int32()
        assert ref.ref_emit_slp(text.encode(), r["json"].encode(), buf, len(buf), C.byref(n)) == 0
        r["slp"] = buf.value.decode()
    with open(os.path.join(HERE, "schemes", "laderman.json")) as f:
        text = f.read()
    other = {}
    for seed in (3, 4):
        cfg = T.SearchConfig(n_processes=16, patience=2, master_seed=seed)
        buf = C.create_string_buffer(1 << 22)
        n = C.c_int32()
        assert ref.ref_optimize_scheme_json(text.encode(), C.byref(cfg.to_c()), 4, buf, len(buf), C.byref(n)) == 0
        other[seed] = buf.value.decode()
    buf = C.create_string_buffer(1 << 22)
    n = C.c_int32()
    joined = (other[3] + "\x1e" + other[4]).encode()
    assert ref.ref_combine_json(joined, buf, len(buf), C.byref(n)) == 0, ref.ref_last_error()
    g["combine"] = dict(inputs=[other[3], other[4]], json=buf.value.decode())
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, separators=(",", ":"))
        f.write("\n")
    print("run_cse cases", len(g["run_cse"]), "optimize", len(g["optimize"]))


if __name__ == "__main__":
    main()
