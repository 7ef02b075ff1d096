"""Writes the bench's roofline inputs from one `ncu --set full` capture of the
two RK-stage launches of the 3D stage kernel (tools/gpu/prof_stages.sh):
profiles/traffic_cfg4.json (DRAM bytes per launch, averaged over the two
stages) and the fp64-pipe fraction in profiles/fp64_peaks.json.
usage: python tools/roofline_inputs.py REPORT.ncu-rep KERNEL_LABEL"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, label = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]


def col(name):
    i = hdr.index(name)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(units[i], 1)
    return [float(r[i].replace(",", "")) * scale for r in data]


rd, wr = col("dram__bytes_read.sum"), col("dram__bytes_write.sum")
fp = col("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
per = [r + w for r, w in zip(rd, wr)]
src = os.path.basename(rep)
tr = {"kernel": f"{label} (512^3), average of the two RK stage launches",
      "bytes_per_launch": sum(per) / len(per),
      "source": f"ncu --set full, {src}: " + ", ".join(
          f"stage {i + 1} dram read {r / 1e9:.3f} GB + write {w / 1e9:.3f} GB"
          for i, (r, w) in enumerate(zip(rd, wr))) +
                "; algorithmic 2.5 S x 134.2M cells = 13.42 GB"}
json.dump(tr, open(os.path.join(ROOT, "profiles", "traffic_cfg4.json"), "w"), indent=1)
p = os.path.join(ROOT, "profiles", "fp64_peaks.json")
d = json.load(open(p))
d["fv3d_stage_fp64_pipe_frac"] = round(sum(fp) / len(fp) / 100.0, 3)
d["fv3d_stage_fp64_pipe_frac_source"] = (
    f"ncu --set full, sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active, "
    f"{label}, both RK stages ({src})")
json.dump(d, open(p, "w"), indent=1)
print(json.dumps(tr, indent=1))
print("fp64 pipe frac", d["fv3d_stage_fp64_pipe_frac"])
