"""The result/output path, host-side and GPU-free:
emit_slp, parse_report / report_to_json round trip, combine_componentwise and
the CLI front end — byte-identical to the reference (goldens made from it by
tests/golden/make_golden.py; live comparison when oracle/_ref is present)."""
import json
import os
import subprocess
import sys

import pytest

import paper_2512_13365_b200 as T
from helpers import GOLDEN, SCHEMES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(GOLDEN, "golden.json")) as f:
    G = json.load(f)


@pytest.mark.parametrize("name", sorted(G["reports"]))
def test_report_round_trip_and_slp(name):
    r = G["reports"][name]
    rep = T.parse_report(r["json"])
    assert T.report_to_json(rep) == r["json"]
    s = T.load_scheme(os.path.join(SCHEMES, name + ".json"))
    slp = T.emit_slp(rep, s)
    assert slp == r["slp"]
    # one binary operator per addition (test_io.cpp:105-152)
    assert T.count_slp_operators(slp) == rep["total"]


def test_slp_reexpands_to_the_scheme():
    # every output line of the program expands back to its original row (test_io.cpp:154-197)
    r = G["reports"]["laderman"]
    rep = T.parse_report(r["json"])
    s = T.load_scheme(os.path.join(SCHEMES, "laderman.json"))
    slp = T.emit_slp(rep, s)
    defined, outputs = {}, {}
    for line in slp.splitlines():
        if not line or line[0] == "#":
            continue
        name, rhs = line.split(" = ")
        acc, sign = {}, 1
        toks = rhs.split(" ")
        if toks[0].startswith("-"):
            sign, toks[0] = -1, toks[0][1:]
        for tok in toks:
            if tok in "+-":
                sign = 1 if tok == "+" else -1
                continue
            for v, c in defined.get(tok, {tok: 1}).items():
                acc[v] = acc.get(v, 0) + sign * c
        acc = {v: c for v, c in acc.items() if c}
        (defined if name.startswith("t") else outputs)[name] = acc
    for q in range(s["r"]):
        want = {"a[%d][%d]" % (k // 3 + 1, k % 3 + 1): x for k, x in enumerate(s["u"][q]) if x}
        assert outputs.get("u[%d]" % (q + 1), {}) == want


def test_combine_matches_reference():
    c = G["combine"]
    reps = [T.parse_report(x) for x in c["inputs"]]
    assert T.report_to_json(T.combine_componentwise(reps)) == c["json"]
    assert T.report_to_json(T.combine_componentwise(reps[:1])) == c["inputs"][0]
    other = dict(reps[1])
    other["scheme_digest"] = "0000000000000000"
    with pytest.raises(ValueError, match="different schemes"):
        T.combine_componentwise([reps[0], other])


def test_cli_verify_and_combine(tmp_path):
    cli = os.path.join(ROOT, "tools", "tcse_cli.py")
    out = subprocess.run([sys.executable, cli, "verify", os.path.join(SCHEMES, "strassen.json")],
                         capture_output=True, text=True)
    assert out.returncode == 0
    assert "digest: 05ac287a032b2430" in out.stdout and "naive: U=5 V=5 W=8 total=18" in out.stdout
    paths = []
    for t, x in enumerate(G["combine"]["inputs"]):
        p = tmp_path / ("r%d.json" % t)
        p.write_text(x)
        paths.append(str(p))
    dst = tmp_path / "best.json"
    out = subprocess.run([sys.executable, cli, "combine"] + paths + ["--out-report", str(dst)],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert dst.read_text() == G["combine"]["json"]
    bad = subprocess.run([sys.executable, cli, "verify", str(tmp_path / "missing.json")], capture_output=True,
                         text=True)
    assert bad.returncode == 1 and bad.stderr.startswith("error: ")


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(G["reports"]))
def test_cli_reduce_reproduces_reference_files(tmp_path, name):
    """`reduce` on the GPU writes the reference's report JSON and SLP bytes."""
    r = G["reports"][name]
    cfg = r["cfg"]
    rep, slp = tmp_path / "r.json", tmp_path / "p.slp"
    cmd = [sys.executable, os.path.join(ROOT, "tools", "tcse_cli.py"), "reduce", os.path.join(SCHEMES, name + ".json"),
           "--processes", str(cfg["n_processes"]), "--iterations-patience", str(cfg["patience"]),
           "--seed", str(cfg["master_seed"]), "--out-report", str(rep), "--out-slp", str(slp)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    assert rep.read_text() == r["json"]
    assert slp.read_text() == r["slp"]


def test_flip_report_round_trip_and_combine():
    """parse_report keeps flip_mode, per-component scheme_id and the carried
    scheme (io.hpp:190-196, 242, 285-286): flip reports of the reference
    round-trip byte-identically and combine like the reference's."""
    with open(os.path.join(os.path.dirname(__file__), "golden", "flip_reports.json")) as f:
        g = json.load(f)
    reps = [T.parse_report(x) for x in g["reports"]]
    for text, rep in zip(g["reports"], reps):
        assert rep["config"]["flip_enabled"] is True
        assert rep["scheme"]["r"] == 27 and all("scheme_id" in c for c in rep["components"])
        assert T.report_to_json(rep) == text
    a, b = g["combine_pair"]
    assert T.report_to_json(T.combine_componentwise([reps[a], reps[b]])) == g["combined"]
    if reps[0]["scheme_digest"] != reps[1]["scheme_digest"]:
        with pytest.raises(ValueError, match="different schemes"):
            T.combine_componentwise(reps)
