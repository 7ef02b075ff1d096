"""Per-CUDA-source-line executed thread instructions (per unit) and stall
samples from `ncu -i R --page source --csv --print-source cuda,sass`.
usage: python tools/src_lines.py MIX.csv UNITS [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2])
N = int(sys.argv[3]) if len(sys.argv) > 3 else 50
fname = hdr = None
stats = collections.defaultdict(lambda: [0.0, 0.0, ""])


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or r[0] == "Function Name" or hdr is None or len(r) < 9:
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    s = stats[(fname, line)]
    s[0] += num(r[4])
    s[1] += num(r[8])
    s[2] = r[1].strip()[:95]
ti = sum(v[1] for v in stats.values())
ts = sum(v[0] for v in stats.values()) or 1.0
print(f"thread instr per unit {ti / units:.1f}")
for (f, l), v in sorted(stats.items(), key=lambda kv: -kv[1][1])[:N]:
    print(f"{v[1] / units:7.1f}  samp {100 * v[0] / ts:4.1f}%  {f}:{l}  {v[2]}")
