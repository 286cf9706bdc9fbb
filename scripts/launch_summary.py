"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-launch lines + per-kernel shares: python scripts/launch_summary.py launches.csv "<command>" """
import collections
import csv
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    ns = float(r["Metric Value"].replace(",", ""))
    if r["Metric Unit"] == "us":
        ns *= 1e3
    elif r["Metric Unit"] == "ms":
        ns *= 1e6
    name = r["Kernel Name"].replace("tcse::", "").replace("(tcse::LaunchDesc)", "").replace("(tcse::XchgLaunch)", "")
    rows.append((name, r["Grid Size"], r["Block Size"], ns / 1e6))
print("# ncu --metrics gpu__time_duration.sum --clock-control none " + (sys.argv[2] if len(sys.argv) > 2 else ""))
print("# (cold-cache, serialised: compare shares)")
for name, g, b, ms in rows:
    print("%s grid=%s block=%s %.3f ms" % (name, g, b, ms))
tot = collections.OrderedDict()
cnt = collections.Counter()
for name, _, _, ms in rows:
    tot[name] = tot.get(name, 0.0) + ms
    cnt[name] += 1
all_ms = sum(tot.values())
print()
for name, ms in sorted(tot.items(), key=lambda x: -x[1]):
    print("%-40s launches=%d total=%.3f ms share=%.1f%%" % (name, cnt[name], ms, 100 * ms / all_ms))
