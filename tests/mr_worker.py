"""Worker for tests/test_gpu_multirank.py: one rank of a 2-rank search on a
shared GPU, exchanging payloads over gloo (host), in one of two transports:
  callback: tcse_set_partition allgather callback (library-driven)
  device:   step_begin/step_end around a caller-run all-gather of device
            buffers (here staged through gloo; NCCL in bench.py)"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2512_13365_b200 as T  # noqa: E402
from helpers import fixture_systems  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
mode, name, n, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
dist.init_process_group("gloo")


def allgather(data):
    t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return [p.numpy().tobytes() for p in parts]


dev = T.Device(0)
systems = fixture_systems(name)
cfg = T.SearchConfig(n_processes=n, patience=3, master_seed=11)
if mode == "callback":
    dev.set_partition(rank, world, allgather)
    st = {}
    res = T.optimize_systems(systems, cfg, [0, 1, 2], device=dev, stats=st)
else:
    dev.set_partition(rank, world, None)
    search = T.Search(systems, cfg, [0, 1, 2], device=dev)
    nb = search.payload_bytes()
    send = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    recv = torch.zeros(nb * world, dtype=torch.uint8, device="cuda")
    while True:
        search.step_begin(send.data_ptr())
        torch.cuda.synchronize()
        parts = [torch.empty(nb, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, send.cpu())
        recv.copy_(torch.cat(parts).cuda())
        torch.cuda.synchronize()
        if search.step_end(recv.data_ptr()) == 0:
            break
    res, st = search.result()
json.dump({"records": [[list(map(list, r.substitutions)), r.cost, r.strategy, r.seed, it] for r, it in res],
           "steps": st["steps"]}, open(out + ".%d" % rank, "w"))
dist.destroy_process_group()
