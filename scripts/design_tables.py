"""Regenerate the DESIGN.md section 7 tables (per-config bench lines, fixed
wall time) from profiles/ in place: python scripts/design_tables.py"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = lambda f: os.path.join(ROOT, "profiles", f)  # noqa: E731
names = {0: "Strassen 2×2×2:7, forced greedy", 1: "Laderman 3×3×3:23, forced gi", 2: "S⊗S 4×4×4:49, mixed (headline)",
         3: "naive 5×5×5 + 1000 flips, mixed", 4: "S⊗L 6×6×6:161, mixed"}


def M(x):
    return "%.1f M" % (x / 1e6) if x >= 1e6 else ("%.3f M" % (x / 1e6) if x > 0 else "0")


tbl = ["| config | workload | N/component | value (steps/s) | e2e | reference CPU | ratio (e2e) | roofline frac |",
       "|---|---|---:|---:|---:|---:|---:|---:|"]
for c in range(5):
    d = json.load(open(P("r01_bench_cfg%d.json" % c)))
    n = d["config"]["processes_per_gpu"]
    if c == 0:
        tbl.append("| 0 | %s | %d | 0 (no reducible pair; costs 5/5/8 = 18) | 0 | 0 | — | — |" % (names[0], n))
        continue
    v, e, cpu, fr = d["value"], d["e2e"]["value"], d["cpu_baseline"]["value"], d["roofline"]["frac"]
    tbl.append("| %d | %s | %d | %s | %s | %s | %d× | %.1f%% |" % (c, names[c], n, M(v), M(e), M(cpu), round(e / cpu),
                                                                 100 * fr))
rows = json.load(open(P("r01_wall_budget.json")))
wt = ["| scheme | shape | naive | reference total (N, iters, wall s) | GPU total (N, wall s) | GPU, more seeds + "
      "combine within the reference's time | GPU ≤ ref |", "|---|---|---:|---|---|---|---|"]
for r in rows:
    ref, g, cb = r["reference"], r["gpu"], r["gpu_seeds_combined"]
    wt.append("| %s | %s | %d | %d (%d, %d, %.2f) | %d (%d, %.2f) | %d (%d seeds, %.2f s) | %s |" % (
        r["scheme"], r["shape"], sum(r["naive"]), ref["total"], ref["processes"], ref["iterations"], ref["wall_s"],
        g["total"], g["processes"], g["wall_s"], cb["total"], len(cb["seeds"]), cb["wall_s"],
        "yes" if r["gpu_le_reference"] else "no"))
path = os.path.join(ROOT, "DESIGN.md")
s = open(path).read()
for head, new in (("| config | workload | N/component |", tbl), ("| scheme | shape | naive | reference total", wt)):
    a = s.index(head)
    b = s.index("\n\n", a)
    s = s[:a] + "\n".join(new) + s[b:]
open(path, "w").write(s)
print("\n".join(tbl))
print("\n".join(wt))
