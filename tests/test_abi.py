"""The C-ABI library loads without a GPU, exports every symbol include/tcse.h
declares, and its struct layouts match the ctypes mirror."""
import ctypes as C
import os
import re
import subprocess

import paper_2512_13365_b200 as T
from paper_2512_13365_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tcse.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tcse_[a-z_0-9]+)\s*\(", text)) - {"tcse_iter_cb", "tcse_allgather_fn"})


def test_library_exports_every_declared_symbol():
    lib = T.lib()
    names = declared_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", T.library_path()], capture_output=True, text=True).stdout
    for name in names:
        assert re.search(r" T %s$" % name, out, re.M), name


def test_loads_without_gpu_and_reports_abi():
    lib = T.lib()
    assert lib.tcse_abi_version() == 2
    cfg = _abi.SearchConfig()
    lib.tcse_default_search_config(C.byref(cfg))
    assert list(cfg.strategy_weights) == [0.0, 4.0, 1.0, 2.0, 8.0, 0.1, 0.01]
    assert (cfg.reinit_fraction, cfg.patience, cfg.forced_strategy) == (0.4, 10, -1)
    s = _abi.make_system(4, [[1, 2, -3, 4], [1, -2, -4], [1, -2, -3, 4]])
    assert lib.tcse_naive_cost(C.byref(s)) == 8


def test_host_verification_api_without_gpu():
    # expand_and_verify through the product's host API (no device needed)
    ex = T.LinearSystem(4, [[1, 2, -3, 4], [1, -2, -4], [1, -2, -3, 4]])
    assert T.verify_record(ex, [(2, 4, 1), (1, 3, -1)]) == (True, 6)
    with __import__("pytest").raises(T.TcseError, match="position 1"):
        T.verify_record(ex, [(2, 4, 1), (2, 4, 1)])


def test_struct_layouts_match_header(tmp_path):
    prog = tmp_path / "layout.c"
    structs = {"tcse_pair": _abi.Pair, "tcse_pair_count": _abi.PairCount, "tcse_system": _abi.System,
               "tcse_process_config": _abi.ProcessConfig, "tcse_search_config": _abi.SearchConfig,
               "tcse_record": _abi.Record, "tcse_stats": _abi.Stats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "%s"' % HEADER, "int main(void){"]
    for cname, py in structs.items():
        lines.append('printf("%s %%zu\\n", sizeof(%s));' % (cname, cname))
        for f, _ in py._fields_:
            lines.append('printf("%s.%s %%zu\\n", offsetof(%s, %s));' % (cname, f, cname, f))
    lines.append("return 0;}")
    prog.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(prog)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got["%s.%s" % (cname, f)]) == getattr(py, f).offset, (cname, f)


def test_no_device_fails_loudly():
    if T.lib().tcse_device_count() > 0:
        return
    import pytest
    with pytest.raises(T.TcseError):
        T.Device(0)
