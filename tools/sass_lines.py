"""Attribute an ncu SASS source page (csv) to CUDA source lines using the
line table of `nvdisasm -g -c` of the same kernel.
    python tools/sass_lines.py NCU_SRC.csv DISASM.txt KERNEL_MANGLED [FILE]"""
import collections
import csv
import re
import sys

src_csv, dis, kern = sys.argv[1:4]
fname = sys.argv[4] if len(sys.argv) > 4 else None
# offset -> (file, line)
lines = {}
cur = None
inside = False
for ln in open(dis):
    if ln.startswith("//----") and ".text." in ln:
        inside = ln.strip().endswith(".text." + kern + " --------------------------") or \
            (".text." + kern + " ") in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), \
    hdr.index("Warp Stall Sampling (All Samples)")
seen = set()
data = []
for r in rows[2:]:
    if len(r) <= iE or not r[iE].isdigit():
        continue
    a = int(r[0], 16)
    if a in seen:
        continue
    seen.add(a)
    data.append((a, int(r[iE]), int(r[iW] or 0), r[iS].strip()))
base = min(a for a, *_ in data)
agg = collections.defaultdict(lambda: [0, 0])
tot_i = sum(n for _, n, _, _ in data)
tot_w = sum(w for _, _, w, _ in data)
miss = 0
for a, n, w, s in data:
    key = lines.get(a - base)
    if key is None:
        miss += n
        continue
    if fname and key[0] != fname:
        key = ("(inlined:" + key[0] + ")", key[1])
    agg[key][0] += n
    agg[key][1] += w
print(f"total inst {tot_i:.4e} stall samples {tot_w} unmapped inst {miss:.3e}")
for (f, l), (n, w) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:60]:
    print(f"{f}:{l:<5d} inst {100*n/tot_i:6.2f}%  stall {100*w/max(tot_w,1):6.2f}%")
