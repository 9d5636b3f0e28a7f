"""Attribute an ncu SASS source page (csv) to the OUTERMOST source line of the
kernel body (the call site, through any depth of inlining) using
`nvdisasm -gi -c` of the same cubin, and sum instructions / stall samples per
call-site line and per named line range.

    python tools/sass_regions.py NCU_SRC.csv DISASM_GI.txt KERNEL_MANGLED \
        [name=lo-hi ...]

    cuobjdump -xelf all paper_2412_03898_b200/csrc/fwd_run.o
    nvdisasm -gi -c fwd_run.sm_100a.cubin > dis.txt
"""
import collections
import csv
import re
import sys

src_csv, dis, kern = sys.argv[1:4]
regions = []
for spec in sys.argv[4:]:
    name, rng = spec.split("=")
    lo, hi = rng.split("-")
    regions.append((name, int(lo), int(hi)))

outer = {}     # offset -> (file, line) outermost frame
inner = {}     # offset -> (file, line) innermost frame
inside = False
chain = []
cur_outer = cur_inner = None
for ln in open(dis):
    if ln.startswith("//----") and ".text." in ln:
        inside = (".text." + kern + " ") in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)( inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        fr = (m.group(1).split("/")[-1], int(m.group(2)))
        if not chain:
            cur_inner = fr
        chain.append(fr)
        if not m.group(3):          # end of the chain: the outermost frame
            cur_outer = fr
            chain = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m and cur_outer:
        off = int(m.group(1), 16)
        outer[off] = cur_outer
        inner[off] = cur_inner

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
tot_i = sum(n for _, n, _, _ in data)
tot_w = sum(w for _, _, w, _ in data)
by_line = collections.defaultdict(lambda: [0, 0])
by_reg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for a, n, w, s in data:
    o = outer.get(a - base)
    if o is None:
        o = ("?", 0)
    by_line[o][0] += n
    by_line[o][1] += w
    name = "other"
    for rn, lo, hi in regions:
        if lo <= o[1] <= hi:
            name = rn
            break
    by_reg[name][0] += n
    by_reg[name][1] += w
    by_reg[name][2][s.split()[0] if s else "?"] += n
print(f"total inst {tot_i:.4e} stall samples {tot_w}")
if regions:
    print("-- regions (outermost line range)")
    for name, (n, w, ops) in sorted(by_reg.items(), key=lambda kv: -kv[1][0]):
        top = ", ".join(f"{k} {100*v/max(n,1):.0f}%" for k, v in ops.most_common(6))
        print(f"{name:<14s} inst {100*n/tot_i:6.2f}%  stall {100*w/max(tot_w,1):6.2f}%   [{top}]")
print("-- call-site lines")
for (f, l), (n, w) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{f}:{l:<5d} inst {100*n/tot_i:6.2f}%  stall {100*w/max(tot_w,1):6.2f}%")
