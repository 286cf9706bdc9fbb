"""Copy one evidence run (scripts/evidence.sh TAG, ALLCFG=1 WALL=1) from
gpurun_out/ into profiles/: bench lines per config, launch list, ncu summary of
the headline search kernel (+ top lines and regions), DRAM bytes per launch,
fixed-wall-time table.  usage: python scripts/make_profiles.py TAG "note" """
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
G = lambda f: os.path.join(ROOT, "gpurun_out", f)  # noqa: E731
P = lambda f: os.path.join(ROOT, "profiles", f)  # noqa: E731
run = lambda *a: subprocess.run(["python"] + list(a), capture_output=True, text=True, cwd=ROOT).stdout  # noqa: E731

with open(P("r01_%s_launches.txt" % tag), "w") as f:
    f.write(run("scripts/launch_summary.py", G("%s_launches.csv" % tag),
                "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 1 "
                "--no-cpu-baseline (all launches incl. e2e pass)"))
d = json.loads(run("scripts/ncu_summary.py", G("%s_search.ncu-rep" % tag), note))
d["top_source_lines"] = run("scripts/ncu_lines.py", G("%s_search.ncu-rep" % tag), "14").strip().split("\n")
d["regions"] = run("scripts/ncu_regions.py", G("%s_search.ncu-rep" % tag)).strip().split("\n")[:16]
json.dump(d, open(P("r01_%s_search_kernel_ncu.json" % tag), "w"), indent=1)


def nbytes(x):
    v, u = x.split()
    return float(v) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u]


json.dump({"kernel": "search_kernel<1,64,dense> W group (sxs, 16384 processes, iteration 2)",
           "dram_bytes_per_launch": nbytes(d["dram__bytes_read.sum"]) + nbytes(d["dram__bytes_write.sum"]),
           "source": "profiles/r01_%s_search_kernel_ncu.json (ncu --set full; dram__bytes_read.sum + "
                     "dram__bytes_write.sum)" % tag}, open(P("search_kernel_dram.json"), "w"), indent=1)
shutil.copy(G("%s_bench.json" % tag), P("r01_bench_%s.json" % tag))
shutil.copy(G("%s_bench.json" % tag), P("r01_bench_cfg2.json"))
for c in (0, 1, 3, 4):
    if os.path.exists(G("%s_bench_cfg%d.json" % (tag, c))):
        shutil.copy(G("%s_bench_cfg%d.json" % (tag, c)), P("r01_bench_cfg%d.json" % c))
wl = G("%s_wall_budget.log" % tag)
if os.path.exists(wl):
    rows = [json.loads(ln) for ln in open(wl) if ln.startswith("{")]
    if rows:
        json.dump(rows, open(P("r01_wall_budget.json"), "w"), indent=1)
print(json.dumps({k: d[k] for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                                    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum")}))
print(d["stall_share_pct"])
print("\n".join(d["regions"][:10]))
