"""Generates tests/golden/flip_reports.json from the reference (oracle/_ref):
two optimize_with_flips reports (parallel_search.hpp:354-518) of a flipped
naive 3x3x3 scheme and their combine_componentwise (522-547), as report JSON text.
Run here (the reference build must exist); the output is committed."""
import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import paper_2512_13365_b200 as T  # noqa: E402
from paper_2512_13365_b200 import _abi  # noqa: E402
from oracle_lib import reference  # noqa: E402


def main():
    ref = reference()
    ref.ref_optimize_with_flips_json.argtypes = [C.c_char_p, C.POINTER(_abi.SearchConfig), C.c_int32, C.c_int32,
                                                 C.c_int32, C.c_uint32, C.c_char_p, C.c_int32, C.POINTER(C.c_int32)]
    ref.ref_combine_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int32, C.POINTER(C.c_int32)]
    buf = C.create_string_buffer(1 << 22)
    n = C.c_int32()
    assert ref.ref_flipped_naive_json(3, 3, 3, 30, 5, buf, len(buf), C.byref(n)) == 0
    text = buf.value.decode()
    reports = []
    for seed in (77, 78):
        cfg = T.SearchConfig(n_processes=12, patience=2, master_seed=seed, m_schemes=4, flips_min=1, flips_max=6)
        rc = ref.ref_optimize_with_flips_json(text.encode(), C.byref(cfg.to_c()), 4, 1, 6, 4, buf, len(buf),
                                              C.byref(n))
        assert rc == 0, ref.ref_last_error()
        reports.append(buf.value.decode())
    # combine needs reports of one (carried) scheme: a report with itself
    pair = (0, 0)
    joined = "\x1e".join([reports[pair[0]], reports[pair[1]]])
    assert ref.ref_combine_json(joined.encode(), buf, len(buf), C.byref(n)) == 0, ref.ref_last_error()
    out = dict(scheme=text, reports=reports, combine_pair=list(pair), combined=buf.value.decode())
    with open(os.path.join(HERE, "flip_reports.json"), "w") as f:
        json.dump(out, f, indent=0)
        f.write("\n")


if __name__ == "__main__":
    main()
