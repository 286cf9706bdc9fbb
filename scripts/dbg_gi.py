import os, sys, random
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2512_13365_b200 as T
import test_gpu_giforms as G
idx = int(sys.argv[1]); cidx = int(sys.argv[2]) if len(sys.argv) > 2 else -1
rng = random.Random(4242)
syss = G.systems(rng)
allc = []
for s in syss:
    allc.append(G.gi_cfgs(rng, 18))
s = syss[idx]
cfgs = allc[idx] if cidx < 0 else [allc[idx][cidx]]
try:
    T.run_cse(s, cfgs, trace_stride=32)
    print(idx, cidx, "ok", "n_e", len(s[1]), "n_x", s[0])
except Exception as e:
    print(idx, cidx, "FAIL", e, "n_e", len(s[1]), "n_x", s[0])
