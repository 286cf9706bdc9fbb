"""Copy one round-2 evidence run (scripts/evidence_r2.sh TAG) from gpurun_out/
into profiles/ as r02_*: bench lines of every config (+ the reference arm of
configs 3 and 4 at the same process count), the headline launch list, ncu
summaries (+ top lines, regions) of the dominant search kernel of configs 2,
1 and 4, DRAM bytes per launch of the headline kernel, pipe peaks.
usage: python scripts/make_profiles_r2.py TAG VERSION "note" """
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, ver, note = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
G = lambda f: os.path.join(ROOT, "gpurun_out", f)  # noqa: E731
P = lambda f: os.path.join(ROOT, "profiles", f)  # noqa: E731
run = lambda *a: subprocess.run(["python"] + list(a), capture_output=True, text=True, cwd=ROOT).stdout  # noqa: E731


def nbytes(x):
    v, u = x.split()
    return float(v.replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u]


with open(P("r02_%s_launches.txt" % ver), "w") as f:
    f.write(run("scripts/launch_summary.py", G("%s_launches.csv" % tag),
                "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 1 "
                "--no-cpu-baseline --no-e2e"))
for rep, out, what in [("%s_search.ncu-rep" % tag, "r02_%s_search_kernel_ncu.json" % ver,
                        "config 2 headline: W group search_kernel<1,64,dense>, sxs 16384 processes, iteration 2"),
                       ("%s_cfg1_search.ncu-rep" % tag, "r02_%s_cfg1_search_kernel_ncu.json" % ver,
                        "config 1: search_kernel<1,32,dense>, laderman forced gi 4096 processes, iteration 2"),
                       ("%s_cfg4_search.ncu-rep" % tag, "r02_%s_cfg4_search_kernel_ncu.json" % ver,
                        "config 4: W group search_kernel<1,256,walk>, sxl 8192 processes, iteration 2")]:
    if not os.path.exists(G(rep)):
        continue
    d = json.loads(run("scripts/ncu_summary.py", G(rep), note))
    d["what"] = what
    d["top_source_lines"] = run("scripts/ncu_lines.py", G(rep), "14").strip().split("\n")
    d["regions"] = run("scripts/ncu_regions.py", G(rep), *([os.environ["TCSE_PROFILED_SRC"]] if os.environ.get("TCSE_PROFILED_SRC") else [])).strip().split("\n")[:16]
    json.dump(d, open(P(out), "w"), indent=1)
    if "cfg" not in out:
        json.dump({"kernel": what, "dram_bytes_per_launch": nbytes(d["dram__bytes_read.sum"]) +
                   nbytes(d["dram__bytes_write.sum"]),
                   "source": "profiles/%s (ncu --set full; dram__bytes_read.sum + dram__bytes_write.sum)" % out},
                  open(P("search_kernel_dram.json"), "w"), indent=1)
for c in range(5):
    src = G("%s_bench.json" % tag) if c == 2 else G("%s_bench_cfg%d.json" % (tag, c))
    if os.path.exists(src):
        shutil.copy(src, P("r02_bench_cfg%d.json" % c))
for c in (2, 3, 4):
    if os.path.exists(G("%s_ref_cfg%d.json" % (tag, c))):
        shutil.copy(G("%s_ref_cfg%d.json" % (tag, c)), P("r02_bench_reference_cfg%d.json" % c))
if os.path.exists(G("%s_pipes.json" % tag)):
    shutil.copy(G("%s_pipes.json" % tag), P("r02_pipe_peaks.json"))
print("ok")
