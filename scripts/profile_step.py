"""Minimal driver for ncu: the bench workload for a few iterations.
Launch order: 3 x search_kernel (dump mode: base candidate lists), then per
iteration 1 x search_kernel + 1 x reduce_kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_13365_b200 as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sxs"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
forced = sys.argv[4] if len(sys.argv) > 4 else None
s = T.load_scheme(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "schemes", name + ".json"))
systems = [T.LinearSystem(nx, rows) for nx, rows in T.extract_systems(s)]
st = {}
res = T.optimize_systems(systems, T.SearchConfig(n_processes=N, patience=1 << 30, master_seed=1, max_iterations=iters,
                                                       forced_strategy=forced),
                         [0, 1, 2], stats=st)
print(name, N, iters, [r.cost for r, _ in res], st["steps"], "%.2f ms kernel" % st["kernel_ms"])
