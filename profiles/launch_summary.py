"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch list:
per-kernel launches, total/avg time and share (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("qcg::", "").replace("v4::", "").split("<")[0]
    v = float(r[iv].replace(",", ""))
    v = v / 1e3 if r[iu] in ("ns", "nsecond") else v * (1e3 if r[iu] in ("ms", "msecond") else 1)
    tot[name] += v
    cnt[name] += 1
S = sum(tot.values())
print(f"{'kernel':30s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}")
for k, v in tot.most_common():
    print(f"{k:30s} {cnt[k]:8d} {v:10.1f} {v / cnt[k]:8.1f} {100 * v / S:5.1f}%")
