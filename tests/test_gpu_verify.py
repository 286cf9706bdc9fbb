"""Batched device scheme verification (verify.cu) through the
C ABI: every report (valid, first violation, method) identical to the
reference's verify_brent / verify_by_product / check_scheme_auto."""
import copy
import os
import random

import pytest

import helpers
from helpers import ref_check_scheme
from paper_2512_13365_b200 import TcseError, verify_schemes
from paper_2512_13365_b200.scheme import load_scheme

pytestmark = pytest.mark.gpu

ALL = ["strassen", "laderman", "sxs", "sxs_border", "naive555_f1000", "sxl", "naive666_f3000"]


def scheme(name):
    return load_scheme(os.path.join(helpers.SCHEMES, name + ".json"))


def corrupt(s, rng, k=1):
    s = copy.deepcopy(s)
    for _ in range(k):
        t = rng.choice("uvw")
        rows = s[t]
        a = rng.randrange(len(rows))
        b = rng.randrange(len(rows[a]))
        rows[a][b] = rng.choice([x for x in (-1, 0, 1) if x != rows[a][b]])
    return s


@pytest.mark.parametrize("method", ["auto", "exact_brent", "randomized_product"])
def test_goldens_valid(method):
    schemes = [scheme(n) for n in ALL]
    got = verify_schemes(schemes, method, 16, 1)
    want = [ref_check_scheme(s, method, 16, 1) for s in schemes]
    assert [tuple(g) for g in got] == want
    assert all(g.valid for g in got)


@pytest.mark.parametrize("name", ALL)
def test_corruptions_match_reference(name):
    rng = random.Random(hash(name) & 0xffff)
    s0 = scheme(name)
    batch = [corrupt(s0, rng, k) for k in (1, 1, 1, 2, 3, 8)]
    for method, trials, seed in (("exact_brent", 16, 0), ("randomized_product", 10, 42),
                                 ("randomized_product", 1, 5), ("auto", 16, 3)):
        got = verify_schemes(batch, method, trials, seed)
        want = [ref_check_scheme(s, method, trials, seed) for s in batch]
        assert [tuple(g) for g in got] == want, (name, method)


def test_known_answers():
    s = scheme("strassen")
    s["w"][0][0] = -1  # test_scheme.cpp:28-35
    r = verify_schemes([s], "exact_brent")[0]
    assert not r.valid and r.first_violation.startswith("brent(")
    z = dict(m=2, n=2, p=2, r=7, u=[[0] * 4] * 7, v=[[0] * 4] * 7, w=[[0] * 7] * 4)  # test_scheme.cpp:16-26
    r = verify_schemes([z], "exact_brent")[0]
    assert not r.valid and r.first_violation == ref_check_scheme(z, "exact_brent")[1]
    s = scheme("strassen")
    s["u"][3][2] = 1  # test_scheme.cpp:57-61
    assert not verify_schemes([s], "randomized_product", 10, 42)[0].valid
    assert tuple(verify_schemes([scheme("strassen")], "randomized_product", 10, 42)[0]) == \
        (True, None, "randomized_product")


def test_structural_errors():
    s = scheme("strassen")
    s["w"][1][3] = 2  # test_scheme.cpp:47-48
    with pytest.raises(TcseError, match=r"w\[1\]\[3\]") as e:
        verify_schemes([scheme("laderman"), s])
    with pytest.raises(ValueError) as r:
        ref_check_scheme(s, "exact_brent")
    assert str(e.value) == str(r.value)
    with pytest.raises(TcseError, match="trials must be >= 1"):
        verify_schemes([scheme("strassen")], "randomized_product", 0, 1)  # test_scheme.cpp:63-65


def test_mixed_batch_one_call():
    rng = random.Random(11)
    batch = []
    for n in ALL:
        s = scheme(n)
        batch += [s, corrupt(s, rng)]
    got = verify_schemes(batch, "auto", 16, 9)
    want = [ref_check_scheme(s, "auto", 16, 9) for s in batch]
    assert [tuple(g) for g in got] == want
