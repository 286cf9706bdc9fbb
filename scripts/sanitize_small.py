"""Small workload for compute-sanitizer (racecheck / memcheck / synccheck):
every strategy on a few systems through run_cse, the dump path, and a short
optimize_systems with reinit (all kernels: prep, search, pack, reduce)."""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_13365_b200 as T  # noqa: E402
from helpers import fixture_systems, random_system  # noqa: E402

rng = random.Random(1)
sys_ = fixture_systems("laderman")[2]
cfgs = [T.ProcessConfig(k, alpha=0.3, beta=0.7, p_greedy=0.6, seed=rng.getrandbits(64)) for k in range(7)]
T.run_cse(sys_, cfgs, trace_stride=8)
T.count_pairs(sys_, (), 1)
T.count_pairs(random_system(rng, 12, 9), (), 2)
res = T.optimize_systems(fixture_systems("sxs"), T.SearchConfig(n_processes=8, patience=1, max_iterations=3,
                                                                 master_seed=3), [0, 1, 2])
print("ok", [r.cost for r, _ in res])
