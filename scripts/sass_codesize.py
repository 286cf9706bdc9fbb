"""Code bytes of one kernel by source call site (nvdisasm -gi of a cubin):
python scripts/sass_codesize.py file.sass mangled_fn [outer_line] [top]
Without outer_line: bytes per outermost line (the kernel body); with it: bytes
per next-level line inside that call site."""
import re
import sys

fname, fun = sys.argv[1], sys.argv[2]
outer_sel = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(fname).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text." + fun + ":")][0]
end = start + 1
while end < len(lines) and not lines[end].startswith(".text."):
    end += 1
src = open(sys.argv[5] if len(sys.argv) > 5 else "paper_2512_13365_b200/csrc/search.cu").read().split("\n")
chain, agg, building = None, {}, False
for l in lines[start:end]:
    if "//##" in l:
        # an inline chain comes as consecutive lines, innermost first
        n = int(re.findall(r"line (\d+)", l)[0])
        chain = chain + [n] if building else [n]
        building = True
        continue
    building = False
    if chain and re.search(r"/\*[0-9a-f]{4,}\*/", l):
        if outer_sel is None:
            k = chain[-1]
        elif len(chain) >= 2 and chain[-1] == outer_sel:
            k = chain[-2]
        else:
            continue
        agg[k] = agg.get(k, 0) + 16
tot = sum(agg.values())
print("total bytes", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print("%7d %5.1f%%  %5d  %s" % (v, 100.0 * v / tot, k, src[k - 1].strip()[:90]))
