"""Run-to-run variability probe: times repeated batches of MR cycles in one
process (python tools/var_mr.py [--workload cfg3] [--reps 4] [--steps 4])."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1603_05211_b200 import mr as M  # noqa: E402
from paper_1603_05211_b200 import uniform as U  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
idx, case, dim, level, cfl, seed, _ = bench.WORKLOADS[a.workload]
o, epsl = bench.mr_options(a.workload)
s = M.MRSolver(dim, level, M.MROptions(epsilon=o["eps"], eps_level=epsl,
                                       min_leaf_level=o["min_leaf"], local_time=o["local_time"],
                                       local_time_level_gap=o["gap"]))
st = torch.cuda.Stream()
s.set_stream(st)
s.build(U.case_fill(case, seed, level))
s.run(3, cfl=cfl)
for r in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    rep = s.run(a.steps, cfl=cfl)
    e1.record(st)
    e1.synchronize()
    print(f"rep {r}: {e0.elapsed_time(e1) / len(rep.cycles):.2f} ms/cycle (gpu), "
          f"{1e3 * (time.perf_counter() - t0) / len(rep.cycles):.2f} ms/cycle (wall), "
          f"updates/cycle {rep.updates / len(rep.cycles):.3e}", flush=True)
