"""Per-CUDA-source-line stall samples and executed instructions from
`ncu -i R --page source --csv --print-source cuda,sass` (all files).
usage: python tools/src_hot.py MIX.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
stats = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    samp = num(r[4])
    ie = num(r[7])
    stats.append((samp, ie, fname, line, r[1].strip()[:90]))
tot_s = sum(s[0] for s in stats)
tot_i = sum(s[1] for s in stats)
stats.sort(reverse=True)
for s, i, f, l, src in stats[:N]:
    print(f"{100 * s / tot_s:5.1f}% samp {100 * i / tot_i:5.1f}% inst  {f}:{l}  {src}")
