"""Instruction mix of one kernel from `ncu -i R --page source --csv --print-source sass`:
executed warp instructions per opcode (and per cell-stage if CELLS is given).
usage: python tools/sass_mix.py SASS.csv [THREAD_INSTR_DIVISOR]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie = h.index("Instructions Executed")
te = h.index("Thread Instructions Executed")
src = h.index("Source")
samp = h.index("Warp Stall Sampling (All Samples)")
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cnt = collections.Counter()
tcnt = collections.Counter()
scnt = collections.Counter()
tot = ttot = 0
for r in rows[2:]:
    if len(r) <= te:
        continue
    op = r[src].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    n = float(r[ie] or 0)
    t = float(r[te] or 0)
    cnt[o] += n
    tcnt[o] += t
    scnt[o] += float(r[samp] or 0)
    tot += n
    ttot += t
ssum = sum(scnt.values())
print(f"total warp instr {tot:.4g}, thread instr {ttot:.4g}, per unit {ttot / div:.1f}")
for o, n in cnt.most_common(30):
    print(f"{o:12s} {100 * n / tot:5.1f}%  {tcnt[o] / div:8.1f}/unit  stall-samples {100 * scnt[o] / ssum:5.1f}%")
