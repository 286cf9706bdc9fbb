"""Where a kernel's stall_no_inst / long_sb samples sit (SASS address ranges
with the source line of the nearest cuda,sass row): python scripts/ncu_noinst.py rep [col]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "stall_no_inst"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, ic, iall = hdr.index("Address"), hdr.index("Source"), hdr.index(col), hdr.index("Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[ia], 16), r[isrc].strip(), int(r[ic]), int(r[iall])))
    except (ValueError, IndexError):
        pass
base = recs[0][0]
tot = sum(x[2] for x in recs) or 1
tall = sum(x[3] for x in recs) or 1
print("total %s samples %d of %d (%.1f%%), code bytes %d" % (col, tot, tall, 100.0 * tot / tall, recs[-1][0] - base))
# 1 KB buckets
b = {}
for a, s, c, al in recs:
    k = (a - base) // 2048
    b.setdefault(k, [0, 0])
    b[k][0] += c
    b[k][1] += al
for k in sorted(b):
    if b[k][1] > 0.004 * tall:
        print("  +%6d KB  %5.1f%% %s   %5.1f%% all" % (2 * k, 100.0 * b[k][0] / tot, col, 100.0 * b[k][1] / tall))
