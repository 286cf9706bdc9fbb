"""Aggregate ncu source-page samples/instructions of search.cu by code region
(function line ranges read from the source): python scripts/ncu_regions.py rep"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
src = open(sys.argv[2] if len(sys.argv) > 2 else "paper_2512_13365_b200/csrc/search.cu").read().split("\n")
# region starts: lines declaring a device function / kernel
starts = []
for n, line in enumerate(src, 1):
    m = re.search(r"__device__[^(]*?\b(\w+)\s*\(", line) or re.search(r"__global__[^(]*?\b(\w+)\s*\(", line)
    if m:
        starts.append((n, m.group(1)))
# split the big functions into blocks marked by '// @region name' comments
for n, line in enumerate(src, 1):
    m = re.search(r"// @region (\S+)", line)
    if m:
        starts.append((n, m.group(1)))
starts.sort()


def region(ln):
    r = "?"
    for n, name in starts:
        if n <= ln:
            r = name
        else:
            break
    return r


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
hdr = None
fname = "?"
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] in ("File Path", "File Name"):
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or not rec[0].isdigit() or rec[2] != "-":
        continue
    d = dict(zip(hdr[2:], rec[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        i = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    key = region(int(rec[0])) if fname == "search.cu" else fname
    a = agg.setdefault(key, [0, 0])
    a[0] += s
    a[1] += i
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if s / ts > 0.003:
        print("%6.1f%% smp %6.1f%% ins  %s" % (100.0 * s / ts, 100.0 * i / ti, k))
