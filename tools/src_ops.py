"""Executed thread instructions per (source line, opcode) from
`ncu --page source --csv --print-source cuda,sass`.
usage: python tools/src_ops.py MIX.csv OPCODE [N] [DIVISOR]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
op_want = sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 20
div = float(sys.argv[4]) if len(sys.argv) > 4 else 134217728.0
cur = None
fname = None
acc = collections.Counter()
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 9:
        continue
    if r[0] not in ("", "Line No"):
        try:
            cur = f"{fname}:{int(r[0])} {r[1].strip()[:70]}"
        except ValueError:
            pass
        continue
    if r[0] == "" and r[2].startswith("0x"):
        op = r[3].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        if o.split(".")[0] != op_want and op_want != "*":
            continue
        try:
            acc[cur] += float(r[8])
        except ValueError:
            pass
for k, v in acc.most_common(N):
    print(f"{v / div:8.1f}/cell  {k}")
