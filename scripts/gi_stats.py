"""gi path counters of a TCSE_GI_STATS build (debug only):
TCSE_LIBRARY=ab/stats.so python scripts/gi_stats.py scheme N iters [strategy]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_13365_b200 as T  # noqa: E402

name, N, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
forced = sys.argv[4] if len(sys.argv) > 4 else None
s = T.load_scheme(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "schemes", name + ".json"))
systems = [T.LinearSystem(nx, rows) for nx, rows in T.extract_systems(s)]
lib = T.lib()
buf = (ctypes.c_ulonglong * 8)()
T.optimize_systems(systems, T.SearchConfig(n_processes=64, patience=1, max_iterations=1))
lib.tcse_debug_gi_stats(buf, 1)
st = {}
T.optimize_systems(systems, T.SearchConfig(n_processes=N, patience=1 << 30, master_seed=1, max_iterations=iters,
                                           forced_strategy=forced), [0, 1, 2], stats=st)
lib.tcse_debug_gi_stats(buf, 1)
a, lone, folds, ovf, ref, msum, multi = [buf[i] for i in range(7)]
print("%s N=%d: steps=%d approx_steps=%d (avg m %.1f) lone=%.1f%% multi=%.1f%% folds/multi=%.2f ovf=%.2f%% ref_steps=%d" % (
    name, N, st["steps"], a, msum / max(1, a), 100.0 * lone / max(1, a), 100.0 * multi / max(1, a),
    folds / max(1, multi), 100.0 * ovf / max(1, a), ref))
