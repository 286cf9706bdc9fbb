"""Summarise the longest kernel of an ncu --set full report into the JSON kept
under profiles/: python scripts/ncu_summary.py report.ncu-rep note > out.json"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
]
rep, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
kern = [dict(zip(hdr, r)) for r in rows[2:]]


def ms(d):
    v = float(d["gpu__time_duration.sum"].replace(",", ""))
    u = units[hdr.index("gpu__time_duration.sum")]
    return v / 1e6 if u == "ns" else (v / 1e3 if u == "us" else v)


d = max(kern, key=ms)
out = {"Kernel Name": d["Kernel Name"]}
for m in METRICS:
    if m in d:
        u = units[hdr.index(m)]
        out[m] = ("%s %s" % (d[m], u)).strip()
stalls = {}
for h in hdr:
    pre = "smsp__pcsamp_warps_issue_stalled_"
    if h.startswith(pre) and not h.endswith("not_issued"):
        try:
            stalls[h[len(pre):]] = float(d[h].replace(",", ""))
        except ValueError:
            pass
tot = sum(stalls.values()) or 1.0
out["stall_share_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])
                          if v / tot >= 0.005}
lines = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_lines.py"), rep, "12"],
                       capture_output=True, text=True).stdout.splitlines()
out["top_source_lines"] = lines
out["note"] = note
print(json.dumps(out, indent=1))
