"""Scheme verification time: the reference's check_scheme_auto per scheme on
one host core vs one batched device call (tcse_verify_schemes, verify.cu), on
M copies of each golden scheme (flip mode checks M-1 variants per iteration).
Inputs are marshalled once; only the C calls are timed."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2512_13365_b200 as T  # noqa: E402
from paper_2512_13365_b200 import _abi  # noqa: E402
from oracle_lib import reference  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
REPS = 5
dev = T.default_device()
ref = reference()
lib = T.lib()
out = []
for name in ["laderman", "sxs", "sxs_border", "naive555_f1000", "sxl", "naive666_f3000"]:
    s = T.load_scheme(os.path.join(ROOT, "tests/golden/schemes", name + ".json"))
    flat = [(C.c_int8 * sum(len(r) for r in x))(*[v for row in x for v in row]) for x in (s["u"], s["v"], s["w"])]
    cs = (_abi.Scheme * M)(*[_abi.Scheme(s["m"], s["n"], s["p"], s["r"], *flat) for _ in range(M)])
    rep = (_abi.CheckReport * M)()
    assert lib.tcse_verify_schemes(dev.handle, cs, M, -1, 16, 1, rep) == 0  # warm
    t0 = time.perf_counter()
    for _ in range(REPS):
        assert lib.tcse_verify_schemes(dev.handle, cs, M, -1, 16, 1, rep) == 0
    t_dev = (time.perf_counter() - t0) / REPS
    one = _abi.CheckReport()
    t0 = time.perf_counter()
    for t in range(M):
        assert ref.ref_check_scheme(C.byref(cs[t]), -1, 16, 1, C.byref(one)) == 0
    t_ref = time.perf_counter() - t0
    assert all(r.valid for r in rep) and one.valid
    row = dict(scheme=name, r=s["r"], method="randomized_product" if rep[0].method else "exact_brent", batch=M,
               reference_ms=round(t_ref * 1e3, 3), device_ms=round(t_dev * 1e3, 3),
               speedup=round(t_ref / t_dev, 1))
    out.append(row)
    print(json.dumps(row))
