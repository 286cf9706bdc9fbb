"""One rank of the CPU (gloo) multi-rank protocol test: the exchange protocol
of tcse_search (include/tcse.h: partition by global id, per-rank payload of
costs + local best record, global argmin by (cost, id), pick_reinit over the
gathered costs) executed with oracle process runs in place of the kernel."""
import ctypes as C
import json
import os
import random
import sys

import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from helpers import random_system  # noqa: E402
from oracle_lib import oracle  # noqa: E402
import paper_2512_13365_b200 as T  # noqa: E402
from paper_2512_13365_b200 import _abi  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
seed, n, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
dist.init_process_group("gloo")
O = oracle()
O.or_run_process.argtypes = [C.POINTER(_abi.System), C.POINTER(_abi.ProcessConfig), C.c_int32,
                             C.POINTER(_abi.Pair), C.c_int32, C.POINTER(_abi.Record), C.POINTER(C.c_int32)]
sys_ = random_system(random.Random(seed), 20, 10, 15, 8)
s = _abi.make_system(*sys_)
cap = sum(len(r) - 1 for r in sys_[1] if r) + 1
cfg = T.SearchConfig(n_processes=n, patience=3, master_seed=seed)
c_cfg = cfg.to_c()
p0, p1 = n * rank // world, n * (rank + 1) // world
inc = None  # (cost, subs, strategy, seed)
last_cost = [0] * n
unchanged = it = steps = 0
slots = (_abi.ProcessConfig * n)()
while True:
    it += 1
    assert O.or_assign_strategies(C.byref(c_cfg), it, n, 0, slots) == 0
    reinit = [0] * n
    if it >= 2 and inc and len(inc[1]) >= 2:
        costs = (C.c_int32 * n)(*last_cost)
        flags = (C.c_uint8 * n)()
        O.or_pick_reinit(costs, n, cfg["reinit_fraction"], flags)
        reinit = list(flags)
    pre, npre = _abi.make_pairs(inc[1] if inc else [])
    local = []
    for p in range(p0, p1):
        rec = _abi.make_record(cap)
        own = C.c_int32()
        rc = O.or_run_process(C.byref(s), C.byref(slots[p]), reinit[p], pre, npre, C.byref(rec), C.byref(own))
        assert rc == 0, O.or_last_error()
        local.append((rec.cost, _abi.record_subs(rec), rec.strategy, rec.seed))
        steps += own.value
    # payload: slice costs + local best (min cost, lowest global id)
    best = min(range(len(local)), key=lambda t: (local[t][0], t)) if local else None
    payload = {"costs": [r[0] for r in local],
               "best": None if best is None else [p0 + best] + list(local[best])}
    parts = [None] * world
    dist.all_gather_object(parts, payload)
    gcost = [c for pl in parts for c in pl["costs"]]
    assert len(gcost) == n
    bp = min(range(n), key=lambda p: (gcost[p], p))
    owner = next(pl for pl in parts if pl["best"] and pl["best"][0] == bp)["best"]
    if inc is None or gcost[bp] < inc[0]:
        inc = (owner[1], [tuple(q) for q in owner[2]], owner[3], owner[4])
        unchanged = 0
    else:
        unchanged += 1
    last_cost = gcost
    if unchanged >= cfg["patience"]:
        break
steps_all = [None] * world
dist.all_gather_object(steps_all, steps)
json.dump({"cost": inc[0], "subs": [list(q) for q in inc[1]], "strategy": inc[2], "seed": inc[3],
           "iterations": it, "steps": sum(steps_all)}, open(out + ".%d" % rank, "w"))
dist.destroy_process_group()
