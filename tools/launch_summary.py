"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10][1:]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = rows[skip:]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    k = r[4].split("(")[0].split("<")[0].replace("void ", "")
    agg[k][0] += 1
    agg[k][1] += float(r[-1])
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} {v[0]:5d} {v[1] / 1e3:9.1f}us {v[1] / v[0] / 1e3:7.2f}us/launch {100 * v[1] / tot:5.1f}%")
print(f"total {tot / 1e3:.1f} us over {len(rows)} launches")
