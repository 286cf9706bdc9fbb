"""The library's flip-graph walk (tcse_flip_walk, host only) against the
reference's random_flip chains: the stored flipped-naive fixtures (generated
by the reference, tests/golden/make_fixtures.py) and, where the reference
build is present, fresh chains from ref_flipped_naive_json."""
import ctypes as C
import json
import os

import pytest

import paper_2512_13365_b200 as T
from helpers import SCHEMES
from oracle_lib import REF_SO, reference


def canon(s):
    return {k: s[k] for k in ("m", "n", "p", "r", "u", "v", "w")}


@pytest.mark.parametrize("name,shape,flips", [("naive555_f1000", (5, 5, 5), 1000),
                                              ("naive666_f3000", (6, 6, 6), 3000)])
def test_walk_reproduces_reference_fixtures(name, shape, flips):
    want = T.load_scheme(os.path.join(SCHEMES, name + ".json"))
    got = T.flip_walk(T.naive_scheme(*shape), 12345, flips)
    assert canon(got) == canon(want)
    assert T.verify_brent(got) == (True, None)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build absent")
@pytest.mark.parametrize("shape,flips,seed", [((2, 2, 2), 1, 1), ((2, 2, 3), 7, 99), ((3, 3, 3), 40, 5),
                                              ((4, 4, 4), 200, 12345), ((3, 4, 5), 120, 2024)])
def test_walk_matches_reference_random_flip(shape, flips, seed):
    r = reference()
    buf = C.create_string_buffer(1 << 22)
    k = C.c_int32()
    assert r.ref_flipped_naive_json(*shape, flips, seed, buf, len(buf), C.byref(k)) == 0
    want = T.parse_scheme(buf.value.decode())
    got = T.flip_walk(T.naive_scheme(*shape), seed, flips)
    assert canon(got) == canon(want)


def test_zero_flips_is_identity_and_walks_stay_valid():
    s = T.load_scheme(os.path.join(SCHEMES, "laderman.json"))
    assert canon(T.flip_walk(s, 3, 0)) == canon(s)
    for seed in (1, 2, 3):
        assert T.verify_brent(T.flip_walk(s, seed, 25)) == (True, None)


def test_walk_rejects_non_ternary():
    s = T.naive_scheme(2, 2, 2)
    s["u"][0][0] = 2
    with pytest.raises(T.TcseError, match="coefficient out of range"):
        T.flip_walk(s, 1, 1)
