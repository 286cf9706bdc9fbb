"""Golden vectors generated from the reference itself (tests/golden/
make_golden.py): the oracle must reproduce every one (runs without the
reference present), and the report writer must reproduce the reference's
report_to_json bytes."""
import json
import os

import paper_2512_13365_b200 as T
from helpers import EXAMPLE, GOLDEN, fixture_systems, o_count_pairs, o_optimize_system, o_run_cse, o_sequence_fnv

with open(os.path.join(GOLDEN, "golden.json")) as f:
    G = json.load(f)


def test_worked_example_golden():
    # test_linear_system.cpp:48-58 and 66-90
    c = dict(o_count_pairs(EXAMPLE))
    assert c[(2, 4, 1)] == 2 and c[(1, 3, -1)] == 2 and c[(1, 2, 1)] == 1 and c[(1, 2, -1)] == 2
    assert sum(len(r) - 1 for r in EXAMPLE[1]) == 8
    subs, cost = o_run_cse(EXAMPLE, T.ProcessConfig(0))
    assert cost <= 6


def test_greedy_goldens():
    for name, rows in G["greedy"].items():
        for sys_, want in zip(fixture_systems(name), rows):
            subs, cost = o_run_cse(sys_, T.ProcessConfig(0))
            assert cost == want["cost"] and len(subs) == want["steps"]
            assert "%016x" % o_sequence_fnv(subs) == want["fnv"]
            assert [list(q) for q in subs[:3]] == want["first"]


def test_appendix_c_values():
    # SURVEY.md Appendix C (survey-derived; regenerated from the reference)
    g = G["greedy"]
    assert [r["cost"] for r in g["laderman"]] == [18, 18, 34]
    assert [r["cost"] for r in g["sxs"]] == [59, 59, 88]
    assert [r["cost"] for r in g["sxl"]] == [185, 189, 303]
    assert [r["fnv"] for r in g["sxs"]] == ["36fd7a5f61c82d89", "36fd7a5f61c82d89", "751888f0b0445915"]


def test_run_cse_goldens():
    for case in G["run_cse"]:
        cfg = T.ProcessConfig(**{k: (tuple(v) if k == "mix_weights" else v) for k, v in case["cfg"].items()})
        subs, cost = o_run_cse(tuple(case["sys"]), cfg)
        assert [list(q) for q in subs] == case["subs"] and cost == case["cost"]


def test_optimize_goldens():
    for case in G["optimize"]:
        cfg = T.SearchConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in case["cfg"].items()})
        o = o_optimize_system(tuple(case["sys"]), cfg, salt=case["salt"])
        assert [list(q) for q in o["subs"]] == case["subs"]
        assert (o["cost"], o["iterations"], o["steps"], o["seed"]) == (case["cost"], case["iterations"],
                                                                        case["steps"], case["seed"])


def test_report_json_bytes_match_reference():
    for name, r in G["reports"].items():
        ref = r["json"]
        j = json.loads(ref)
        comps = []
        for key in "uvw":
            c = j["components"][key]
            rec = T.SolutionRecord([tuple(q) for q in c["substitutions"]], c["cost"],
                                   T.strategy_from_string(c["strategy"]), c["seed"])
            comps.append(dict(record=rec, cost=c["cost"], naive=c["naive"], iterations=c["iterations"]))
        cfg = T.SearchConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in r["cfg"].items()})
        cfg["n_processes"] = j["config"]["n_processes"]
        rep = dict(scheme_digest=j["scheme_digest"], config=cfg, components=comps, total=j["total"],
                   iterations=j["iterations"])
        assert T.report_to_json(rep) == ref


def test_oracle_reports_match_goldens():
    """optimize_scheme's components re-derived by the oracle (U, V, W with
    salts 0, 1, 2) equal the reference report."""
    for name, r in G["reports"].items():
        j = json.loads(r["json"])
        cfg = T.SearchConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in r["cfg"].items()})
        cfg["n_processes"] = j["config"]["n_processes"]
        for c, (key, sys_) in enumerate(zip("uvw", fixture_systems(name))):
            o = o_optimize_system(sys_, cfg, salt=c)
            assert [list(q) for q in o["subs"]] == j["components"][key]["substitutions"]
            assert o["cost"] == j["components"][key]["cost"]
