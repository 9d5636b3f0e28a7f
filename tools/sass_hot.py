"""Summarise an ncu source page (SASS) csv: instructions executed by opcode and
hot address ranges.  python tools/sass_hot.py FILE.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS, iE, iW, iT = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Avg. Threads Executed")
tot = 0; ops = collections.Counter(); stall = collections.Counter()
lines = []
for r in rows[2:]:
    if len(r) <= iE or not r[iE].isdigit(): continue
    src = r[iS].strip(); n = int(r[iE] or 0); w = int(r[iW] or 0)
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    ops[op.split(".")[0]] += n; stall[op.split(".")[0]] += w; tot += n
    lines.append((r[0], src, n, w, r[iT]))
print("total", tot)
for op, n in ops.most_common(30):
    print(f"{op:12s} {n:14d} {100*n/tot:6.2f}%  stall-samples {stall[op]}")
if len(sys.argv) > 2:
    for a, src, n, w, t in lines:
        if n >= int(sys.argv[2]):
            print(f"{a[-5:]} {n:12d} {w:7d} thr{t:>5s}  {src}")
