"""Quick device-throughput probe (not the bench): steps/s of the search kernel."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_13365_b200 as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sxs"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 4
forced = sys.argv[4] if len(sys.argv) > 4 else None
s = T.load_scheme(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "schemes", name + ".json"))
systems = [T.LinearSystem(nx, rows) for nx, rows in T.extract_systems(s)]
cfg = T.SearchConfig(n_processes=N, patience=1000, master_seed=1, max_iterations=iters, forced_strategy=forced)
T.optimize_systems(systems, T.SearchConfig(n_processes=64, patience=1, max_iterations=1))  # warm
st = {}
t0 = time.time()
res = T.optimize_systems(systems, cfg, [0, 1, 2], stats=st)
wall = time.time() - t0
print("%s N=%d iters=%d forced=%s nt=%s: steps=%d kernel_ms=%.1f step_ms=%.1f wall_ms=%.1f exch_ms=%.1f -> %.4g steps/s (kernel) %.4g steps/s (step) %.3g steps/s (wall) costs=%s" % (
    name, N, iters, forced, os.environ.get("TCSE_NT", "64"), st["steps"], st["kernel_ms"], st["step_ms"], st["wall_ms"],
    st["exchange_ms"], st["steps"] / st["kernel_ms"] * 1e3, st["steps"] / st["step_ms"] * 1e3, st["steps"] / wall,
    [r.cost for r, _ in res]))
