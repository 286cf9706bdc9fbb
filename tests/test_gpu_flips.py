"""Flip mode on the device: optimize_with_flips
(parallel_search.hpp:354-518) vs the reference itself, report JSON byte for
byte (carried scheme, scheme ids, records, iterations), plus the reference's
own flip-mode properties (test_parallel_search.cpp:204-261)."""
import ctypes as C
import json
import os

import pytest

import paper_2512_13365_b200 as T
from helpers import SCHEMES
from oracle_lib import have_reference, reference
from paper_2512_13365_b200 import _abi

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_reference(), reason="reference build unavailable")]


def ref_lib():
    r = reference()
    r.ref_optimize_with_flips_json.argtypes = [C.c_char_p, C.POINTER(_abi.SearchConfig), C.c_int32, C.c_int32,
                                               C.c_int32, C.c_uint32, C.c_char_p, C.c_int32, C.POINTER(C.c_int32)]
    return r


def naive_json(m, n, p, flips=0, seed=0):
    r = reference()
    buf = C.create_string_buffer(1 << 22)
    k = C.c_int32()
    assert r.ref_flipped_naive_json(m, n, p, flips, seed, buf, len(buf), C.byref(k)) == 0
    return buf.value.decode()


def ref_flip_report(text, cfg):
    r = ref_lib()
    buf = C.create_string_buffer(1 << 23)
    k = C.c_int32()
    rc = r.ref_optimize_with_flips_json(text.encode(), C.byref(cfg.to_c()), cfg["m_schemes"], cfg["flips_min"],
                                        cfg["flips_max"], 4, buf, len(buf), C.byref(k))
    assert rc == 0, r.ref_last_error()
    return buf.value.decode()


CASES = [
    ("naive223", dict(n_processes=12, patience=2, master_seed=77, m_schemes=4, flips_min=1, flips_max=6)),
    ("strassen", dict(n_processes=9, patience=2, master_seed=3, m_schemes=3)),
    ("laderman", dict(n_processes=32, patience=2, master_seed=5, m_schemes=4)),
    ("naive223f", dict(n_processes=24, patience=3, master_seed=9, m_schemes=5, flips_min=2, flips_max=8)),
]


@pytest.mark.parametrize("name,kw", CASES)
def test_flip_report_bytes_match_reference(dev, name, kw):
    if name == "naive223":
        text = naive_json(2, 2, 3)
    elif name == "naive223f":
        text = naive_json(2, 2, 3, 10, 3)
    else:
        text = open(os.path.join(SCHEMES, name + ".json")).read()
    cfg = T.SearchConfig(**kw)
    want = ref_flip_report(text, cfg)
    got = T.report_to_json(T.optimize_with_flips(T.parse_scheme(text), cfg))
    assert got == want


def test_flip_results_verify_against_carried_scheme(dev):
    # test_parallel_search.cpp:225-252
    s = T.parse_scheme(naive_json(2, 2, 3))
    rep = T.optimize_with_flips(s, T.SearchConfig(n_processes=12, patience=2, master_seed=77, m_schemes=4,
                                                  flips_min=1, flips_max=6))
    carried = rep["scheme"]
    assert T.verify_brent(carried) == (True, None)
    assert rep["scheme_digest"] == T.scheme_digest(carried)
    total = 0
    for (nx, rows), c in zip(T.extract_systems(carried), rep["components"]):
        ok, cost = T.verify_record(T.LinearSystem(nx, rows), c["record"].substitutions)
        assert ok and cost == c["cost"]
        total += cost
    assert rep["total"] == total
    naive = sum(T.naive_cost(rows) for _, rows in T.extract_systems(s))
    assert rep["total"] <= naive


def test_one_scheme_is_optimize_scheme(dev):
    # test_parallel_search.cpp:204-223
    s = T.parse_scheme(naive_json(2, 2, 3, 10, 3))
    cfg = T.SearchConfig(n_processes=8, patience=2, master_seed=21)
    plain = T.optimize_scheme(s, cfg)
    flip = T.optimize_with_flips(s, T.SearchConfig(n_processes=8, patience=2, master_seed=21, m_schemes=1))
    assert flip["total"] == plain["total"]
    for a, b in zip(flip["components"], plain["components"]):
        assert a["record"].substitutions == b["record"].substitutions


def test_cli_flip_mode_writes_the_reference_report(tmp_path):
    """`tcse_cli.py reduce --flip-mode --flip-schemes M` dispatches to flip
    mode (terncse_cli.cpp:85-86, 163-164) and writes the reference's report."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "s.json"
    src.write_text(open(os.path.join(SCHEMES, "laderman.json")).read())
    out = tmp_path / "r.json"
    cmd = [sys.executable, os.path.join(root, "tools", "tcse_cli.py"), "reduce", str(src), "--flip-mode",
           "--flip-schemes", "4", "--processes", "32", "--iterations-patience", "2", "--seed", "5",
           "--out-report", str(out)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    cfg = T.SearchConfig(n_processes=32, patience=2, master_seed=5, m_schemes=4)
    assert out.read_text() == ref_flip_report(src.read_text(), cfg)
    # the report round-trips and names the carried scheme's variant
    rep = T.parse_report(out.read_text())
    assert rep["config"]["flip_enabled"] and all("scheme_id" in c for c in rep["components"])
