"""Where the time of one public-API call goes (session create / steps / result / close)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_13365_b200 as T  # noqa: E402

name = sys.argv[1]
N = int(sys.argv[2])
s = T.load_scheme(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "schemes", name + ".json"))
systems = [T.LinearSystem(nx, rows) for nx, rows in T.extract_systems(s)]
T.optimize_systems(systems, T.SearchConfig(n_processes=64, patience=1, max_iterations=1))
for rep in range(2):
    t0 = time.perf_counter()
    se = T.Search(systems, T.SearchConfig(n_processes=N, patience=1 << 30, master_seed=1, max_iterations=3), [0, 1, 2])
    t1 = time.perf_counter()
    ts = []
    while se.step() > 0:
        ts.append(time.perf_counter())
    t2 = time.perf_counter()
    res, st = se.result()
    t3 = time.perf_counter()
    se.close()
    t4 = time.perf_counter()
    steps = [b - a for a, b in zip([t1] + ts[:-1], ts)]
    print("%s N=%d create %.1f ms, steps %s ms, result %.1f ms, close %.1f ms, kernel %.1f ms, steps %d" % (
        name, N, (t1 - t0) * 1e3, ["%.1f" % (x * 1e3) for x in steps], (t3 - t2) * 1e3, (t4 - t3) * 1e3,
        st["kernel_ms"], st["steps"]))
