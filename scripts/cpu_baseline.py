"""Reference CPU path on this host: the reference's
optimize_system (oracle/_ref) on the bench workload (S(x)S 4x4x4:49, default
weights, seed 1), iteration 1 of U, V, W, at the tier process count (256) and
at 4096 / 16384, with threads = nproc and threads = 1; CPU model stated."""
import ctypes as C
import json
import os
import platform
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2512_13365_b200 as T  # noqa: E402
from oracle_lib import reference  # noqa: E402
from paper_2512_13365_b200 import _abi  # noqa: E402


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run(n, threads, iters=1):
    ref = reference()
    s = T.load_scheme(os.path.join(ROOT, "tests", "golden", "schemes", "sxs.json"))
    steps = secs = 0.0
    for comp, (nx, rows) in enumerate(T.extract_systems(s)):
        sy = _abi.make_system(nx, rows)
        rec = _abi.make_record(T.naive_cost(rows) + 1)
        it, st, tot = C.c_int32(), C.c_uint64(), C.c_double()
        cfg = T.SearchConfig(n_processes=n, patience=1 << 30, master_seed=1, max_iterations=iters).to_c()
        assert ref.ref_optimize_system_counted(C.byref(sy), C.byref(cfg), comp, threads, 0.0, C.byref(rec),
                                               C.byref(it), C.byref(st), C.byref(tot)) == 0
        steps += st.value
        secs += tot.value
    return steps / secs, steps, secs


if __name__ == "__main__":
    nproc = os.cpu_count()
    rows = []
    for n in (256, 4096, 16384):
        for th in (nproc, 1):
            if th == 1 and n == 16384:
                continue  # ~25 s; the 4096 point already gives the single-core rate
            v, st, sec = run(n, th)
            rows.append(dict(processes=n, threads=th, steps_per_s=v, steps=int(st), seconds=round(sec, 3)))
            print(json.dumps(rows[-1]), flush=True)
    out = dict(cpu=cpu_model(), nproc=nproc, workload="sxs 4x4x4:49, default weights, seed 1, iteration 1 of U,V,W",
               rows=rows)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "cpu_baseline.json"), "w"), indent=1)
