"""Scheme verification, CPU side: the reference's own
verify_brent / verify_by_product pinned on the golden schemes and corrupted
variants against the host restatement (scheme.verify_brent), and the Python
mirror's structural errors worded like check_structure (scheme.hpp:39-62).
No device calls."""
import copy
import random

import pytest

from helpers import ref_check_scheme
from oracle_lib import have_reference
from paper_2512_13365_b200 import TcseError, verify_schemes
from paper_2512_13365_b200.scheme import load_scheme, verify_brent
import helpers
import os

pytestmark = pytest.mark.skipif(not have_reference(), reason="reference oracle not built")

SMALL = ["strassen", "laderman"]
ALL = ["strassen", "laderman", "sxs", "sxs_border", "naive555_f1000", "sxl", "naive666_f3000"]


def scheme(name):
    return load_scheme(os.path.join(helpers.SCHEMES, name + ".json"))


def corrupt(s, rng):
    s = copy.deepcopy(s)
    t = rng.choice("uvw")
    rows = s[t]
    a = rng.randrange(len(rows))
    b = rng.randrange(len(rows[a]))
    rows[a][b] = rng.choice([x for x in (-1, 0, 1) if x != rows[a][b]])
    return s


@pytest.mark.parametrize("name", ALL)
def test_reference_accepts_goldens(name):
    s = scheme(name)
    valid, fv, method = ref_check_scheme(s, "auto", 16, 1)
    assert valid and fv is None
    assert method == ("randomized_product" if s["r"] >= 200 else "exact_brent")


@pytest.mark.parametrize("name", SMALL)
def test_reference_brent_matches_restatement_on_corruptions(name):
    rng = random.Random(7)
    s0 = scheme(name)
    for _ in range(12):
        s = corrupt(s0, rng)
        valid, fv, _ = ref_check_scheme(s, "exact_brent")
        assert (valid, fv) == verify_brent(s)


def test_reference_known_answers():
    s = scheme("strassen")
    s["w"][0][0] = -1  # test_scheme.cpp:28-35
    valid, fv, _ = ref_check_scheme(s, "exact_brent")
    assert not valid and fv.startswith("brent(")
    s = scheme("strassen")
    s["u"][3][2] = 1  # test_scheme.cpp:57-61
    assert not ref_check_scheme(s, "randomized_product", 10, 42)[0]
    assert ref_check_scheme(scheme("strassen"), "randomized_product", 10, 42) == (True, None, "randomized_product")


def test_mirror_structure_messages_match_reference():
    s = scheme("strassen")
    s["u"].pop()
    # check_tensor's wording (scheme.hpp:41-43)
    with pytest.raises(TcseError, match=r"^scheme: tensor u has 6 rows, expected 7$"):
        verify_schemes([s])
    s2 = scheme("strassen")
    s2["v"][2].append(0)
    with pytest.raises(TcseError, match="tensor v row 2 has 5 entries, expected 4"):
        verify_schemes([s2])
    bad = scheme("strassen")
    bad["m"] = 0
    with pytest.raises(TcseError, match="dimensions and rank must be positive"):
        verify_schemes([bad])

