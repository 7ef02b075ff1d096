"""Wall-clock and event time of cfg3 macro-cycles (run(steps) after warm-up),
with and without the bench's stage profiling."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_1603_05211_b200 import mr as M  # noqa: E402
from paper_1603_05211_b200 import uniform as U  # noqa: E402

idx, case, dim, level, cfl, seed, _ = bench.WORKLOADS["cfg3"]
o, epsl = bench.mr_options("cfg3")
s = M.MRSolver(dim, level, M.MROptions(epsilon=o["eps"], eps_level=epsl, min_leaf_level=o["min_leaf"],
                                       local_time=o["local_time"], local_time_level_gap=o["gap"]))
st = torch.cuda.Stream()
s.set_stream(st)
s.build(U.case_fill(case, seed, level))
s.run(4, cfl=cfl)
for prof in (False, True, False):
    s.profile(prof)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record(st)
    rep = s.run(8, cfl=cfl)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"profile={prof}: wall {1e3 * (time.time() - t0) / 4:.2f} ms/macro, events "
          f"{e0.elapsed_time(e1) / 4:.2f} ms/macro, cycles {len(rep.cycles)}", flush=True)
