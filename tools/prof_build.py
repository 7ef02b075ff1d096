"""Times MRSolver.build (from_uniform + norms + coarsen) for a workload and
prints the kernel launches it makes: python tools/prof_build.py [--workload cfg2]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_1603_05211_b200 import mr as M  # noqa: E402
from paper_1603_05211_b200 import uniform as U  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
idx, case, dim, level, cfl, seed, _ = bench.WORKLOADS[a.workload]
o, epsl = bench.mr_options(a.workload)
s = M.MRSolver(dim, level, M.MROptions(epsilon=o["eps"], eps_level=epsl,
                                       min_leaf_level=o["min_leaf"], local_time=o["local_time"],
                                       local_time_level_gap=o["gap"]))
init = U.case_fill(case, seed, level)
for r in range(a.reps):
    l0 = s.kernel_launches()
    t0 = time.perf_counter()
    s.build(init)
    t1 = time.perf_counter()
    print(f"build {1e3 * (t1 - t0):.2f} ms, launches {s.kernel_launches() - l0}, "
          f"leaves {s.counts()[0]}")
