"""cfg3: device time of run(8) after 4 warm-up steps (CUDA events), per finest
step; run under ncu --cache-control none to get the kernel sum of the same
steps (tools/gpu/c3gap.sh)."""
import os
import sys

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
import time
for rnd in range(int(os.environ.get("ROUNDS", "1"))):
    torch.cuda.synchronize()
    l0 = s.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record(st)
    rep = s.run(8, cfl=cfl)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"device {e0.elapsed_time(e1):.2f} ms (wall {1e3 * (time.time() - t0):.1f}) for 8 finest "
          f"steps ({len(rep.cycles)} cycles, subs {[int(c) for c in rep.cycles[:, 2]]}), "
          f"launches {s.kernel_launches() - l0}", flush=True)
