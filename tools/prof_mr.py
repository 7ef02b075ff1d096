"""Driver for ncu captures of the MR cycle: builds the cfg2 (or cfg3) tree,
runs W warm-up cycles, then K cycles.
    python tools/prof_mr.py [--workload cfg2] [--warmup 2] [--steps 2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_1603_05211_b200 import mr as M  # noqa: E402
from paper_1603_05211_b200 import uniform as U  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--level", type=int, default=None)
a = ap.parse_args()
if a.level is not None:
    w = list(bench.WORKLOADS[a.workload])
    w[3] = a.level
    bench.WORKLOADS[a.workload] = tuple(w)
idx, case, dim, level, cfl, seed, _ = bench.WORKLOADS[a.workload]
o, epsl = bench.mr_options(a.workload)
s = M.MRSolver(dim, level, M.MROptions(epsilon=o["eps"], eps_level=epsl,
                                       min_leaf_level=o["min_leaf"], local_time=o["local_time"],
                                       local_time_level_gap=o["gap"]))
s.build(U.case_fill(case, seed, level))
if a.warmup:
    s.run(a.warmup, cfl=cfl)
l0 = s.kernel_launches()
rep = s.run(a.steps, cfl=cfl)
print("cycles", len(rep.cycles), "updates", rep.updates, "launches", s.kernel_launches() - l0)
