"""SASS of one kernel instantiation grouped by search.cu source line (from the
-lineinfo line table): python scripts/sass_lines.py KERNEL_SUBSTR LINE_LO LINE_HI
Extracts the cubins of paper_2512_13365_b200/libtcse.so into /tmp/tcse_cubin."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
kern, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
d = "/tmp/tcse_cubin"
os.makedirs(d, exist_ok=True)
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2512_13365_b200", "libtcse.so")], cwd=d,
               capture_output=True)
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, "search.sm_100a.cubin")], capture_output=True,
                     text=True).stdout.split("\n")
start = next(i for i, l in enumerate(txt) if l.startswith("\t.section") and kern in l and ".text." in l)
end = next((i for i in range(start + 1, len(txt)) if txt[i].startswith("\t.section")), len(txt))
cur = None
for l in txt[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and cur and cur[0] == "search.cu" and lo <= cur[1] <= hi:
        print("%5d  %s  %s" % (cur[1], m.group(1), re.sub(r"\s+", " ", m.group(2))))
