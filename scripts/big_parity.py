"""Parity + throughput on the large stand-in schemes (multi-word bitsets):
GPU optimize_systems vs the oracle on a small process count, then a timed run."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_13365_b200 as T  # noqa: E402
from helpers import fixture_systems, o_optimize_system  # noqa: E402

name = sys.argv[1]
n_small = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n_big = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
systems = fixture_systems(name)
cfg = T.SearchConfig(n_processes=n_small, patience=1, master_seed=5, max_iterations=2)
t0 = time.time()
got = T.optimize_systems(systems, cfg, [0, 1, 2])
t1 = time.time()
ok = True
for c, (sys_, (rec, it)) in enumerate(zip(systems, got)):
    o = o_optimize_system(sys_, cfg, salt=c)
    same = rec.substitutions == o["subs"] and rec.cost == o["cost"] and it == o["iterations"]
    ok &= same
    print("%s comp %d: gpu %d oracle %d iters %d/%d %s" % (name, c, rec.cost, o["cost"], it, o["iterations"],
                                                          "MATCH" if same else "MISMATCH"))
t2 = time.time()
st = {}
res = T.optimize_systems(systems, T.SearchConfig(n_processes=n_big, patience=1 << 30, master_seed=1, max_iterations=2),
                         [0, 1, 2], stats=st)
print("%s parity %s (gpu %.2fs, oracle %.1fs); N=%d 2 iters: %.3g steps/s kernel, kernel %.1f ms, costs %s" % (
    name, "OK" if ok else "FAILED", t1 - t0, t2 - t1, n_big, st["steps"] / st["kernel_ms"] * 1e3, st["kernel_ms"],
    [r.cost for r, _ in res]))
sys.exit(0 if ok else 1)
