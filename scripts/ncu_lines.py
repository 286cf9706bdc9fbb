"""Per-source-line hot spots from an ncu report (source page, cuda,sass view):
python scripts/ncu_lines.py report.ncu-rep [top] [launch_skip launch_count]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
sel = ["--launch-skip", sys.argv[3], "--launch-count", sys.argv[4]] if len(sys.argv) > 4 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + sel,
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
hdr = None
tot_s = tot_i = 0
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or not rec[0].isdigit() or rec[2] != "-":
        continue
    d = dict(zip(hdr[2:], rec[2:]))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"])
        i = int(d["Instructions Executed"])
    except (KeyError, ValueError):
        continue
    tot_s += s
    tot_i += i
    rows.append((s, i, fname, int(rec[0]), rec[1].strip()[:90]))
rows.sort(reverse=True)
print("total samples %d, warp instructions %d" % (tot_s, tot_i))
for s, i, f, ln, src in rows[:top]:
    print("%5.1f%% smp %5.1f%% ins  %s:%d  %s" % (100.0 * s / tot_s, 100.0 * i / max(tot_i, 1), f, ln, src))
