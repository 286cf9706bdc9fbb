"""The C++ drop-in adapter (include/tcse/terncse_gpu.hpp) used through the
reference's own API, built against the unmodified reference headers
(oracle/_ref/adapter_check): identical report_to_json bytes, records,
on_iteration traces and error behaviour, GPU vs the reference CPU path."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.mark.skipif(not os.path.exists(EXE), reason="adapter_check not built (needs the reference headers)")
def test_adapter_matches_reference_api():
    r = subprocess.run([EXE, os.path.join(ROOT, "tests", "golden", "schemes")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "FAIL" not in r.stdout
    assert r.stdout.count("[PASS]") >= 13
