"""Aggregate an ncu source page (SASS, --csv) by opcode and stall reason.

usage: ncu -i rep --page source --csv --print-source sass --launch-skip N --launch-count 1 > x.csv
       python profiles/ncu_source_summary.py x.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
iS = hdr.index("Warp Stall Sampling (All Samples)")
# the source page may list the SASS more than once: keep the first row per address
ia = hdr.index("Address")
seen = set()
data = []
for r in rows[2:]:
    if len(r) > iS and r[iS].strip().isdigit() and r[ia] not in seen:
        seen.add(r[ia])
        data.append(r)
src = hdr.index("Source")
stall = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iS] or 0) for r in data)
by_op = collections.Counter()
by_reason = collections.Counter()
by_op_reason = collections.defaultdict(collections.Counter)
for r in data:
    s = r[src].strip()
    toks = s.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    n = int(r[iS] or 0)
    by_op[op] += n
    for i, h in stall:
        v = int(r[i] or 0)
        by_reason[h] += v
        by_op_reason[op][h] += v
print(f"total samples {tot}")
print("by reason:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in by_reason.most_common(10)))
for op, n in by_op.most_common(14):
    rs = ", ".join(f"{k[6:]} {v}" for k, v in by_op_reason[op].most_common(3))
    print(f"  {op:10s} {100*n/tot:5.1f}%  ({rs})")
