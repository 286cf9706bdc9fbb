"""Scheme fixtures and the host-side scheme loader (io.hpp:22-81,
scheme.hpp:68-157, parallel_search.hpp:276-292)."""
import json
import os

import pytest

import paper_2512_13365_b200 as T
from helpers import SCHEMES, fixture_index

EXPECTED = {"strassen": ("05ac287a032b2430", [5, 5, 8]), "laderman": ("1575a9b2d4014af0", [28, 28, 42]),
            "sxs": ("7da4ac65bf44d830", [95, 95, 128]), "sxl": ("760577d1fad2ec32", [451, 451, 576]),
            "sxs_border": ("c41f03a3eef4d50f", [95, 95, 180]), "naive555_f1000": (None, [200, 185, 282]),
            "naive666_f3000": (None, [441, 413, 627])}


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_fixture_digest_and_naive(name):
    s = T.load_scheme(os.path.join(SCHEMES, name + ".json"))
    digest, naive = EXPECTED[name]
    if digest:
        assert T.scheme_digest(s) == digest
    assert fixture_index()[name]["digest"] == T.scheme_digest(s)
    assert [T.naive_cost(rows) for _, rows in T.extract_systems(s)] == naive


@pytest.mark.parametrize("name", ["strassen", "laderman", "sxs"])
def test_fixtures_are_brent_valid(name):
    s = T.load_scheme(os.path.join(SCHEMES, name + ".json"))
    assert T.verify_brent(s) == (True, None)


def test_flipped_coefficient_fails_brent():
    # test_scheme.cpp:28-35
    s = T.load_scheme(os.path.join(SCHEMES, "strassen.json"))
    s["w"][0][0] = -s["w"][0][0]
    ok, why = T.verify_brent(s)
    assert not ok and why.startswith("brent(")


def test_extract_shapes():
    # test_scheme.cpp:67-81
    s = T.load_scheme(os.path.join(SCHEMES, "strassen.json"))
    (nu, ru), (nv, rv), (nw, rw) = T.extract_systems(s)
    assert (nu, len(ru), nv, len(rv), nw, len(rw)) == (4, 7, 4, 7, 7, 4)


def test_parse_errors_carry_coordinates():
    # test_io.cpp:70-85
    s = json.load(open(os.path.join(SCHEMES, "strassen.json")))
    s["u"][3][1] = 2
    with pytest.raises(T.SchemeError, match=r"u\[3\]\[1\]"):
        T.parse_scheme(json.dumps(s))
    s = json.load(open(os.path.join(SCHEMES, "strassen.json")))
    del s["u"][6]
    with pytest.raises(T.SchemeError, match="tensor u has 6 rows, expected 7"):
        T.parse_scheme(json.dumps(s))
    with pytest.raises(T.SchemeError, match="scheme json"):
        T.parse_scheme("{ not json")
    with pytest.raises(T.SchemeError, match='"r"'):
        T.parse_scheme('{"m":2,"n":2,"p":2}')
