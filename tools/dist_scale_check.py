"""Full-size check of the MR slab decomposition on one GPU: the cfg3 tree
(2D MRLT, L=13) run as one rank and as N host-thread ranks
(af_comm_create_local), compared bit for bit, with the device memory each
setup takes (windowed arrays map only each rank's rows).
    python tools/dist_scale_check.py [--ranks 8] [--steps 4] [--workload cfg3]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1603_05211_b200 import mr as M  # noqa: E402
from paper_1603_05211_b200 import uniform as U  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--level", type=int, default=None)
a = ap.parse_args()
idx, case, dim, level, cfl, seed, _ = bench.WORKLOADS[a.workload]
level = a.level or level
o, epsl = bench.mr_options(a.workload)
if a.level:
    epsl = ([o['eps'] * 2.0 ** (dim * (l - level)) for l in range(level + 1)]
            if o['eps_scaled'] else None)
opts = M.MROptions(epsilon=o["eps"], eps_level=epsl, min_leaf_level=o["min_leaf"],
                   local_time=o["local_time"], local_time_level_gap=o["gap"])
init = U.case_fill(case, seed, level)
res = {}
for ranks in (1, a.ranks):
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    s = M.MRSolver(dim, level, opts) if ranks == 1 else M.MRGroup(dim, level, ranks, opts)
    torch.cuda.synchronize()
    used = free0 - torch.cuda.mem_get_info()[0]
    t0 = time.perf_counter()
    s.build(init)
    rep = s.run(a.steps, cfl=cfl)
    wall = time.perf_counter() - t0
    keys, u = s.leaves(), s.to_uniform()
    s.close()
    del s
    res[ranks] = (rep, keys, u)
    print(f"ranks={ranks}: device memory at creation {used / 2**30:.2f} GiB "
          f"({used / 2**30 / ranks:.2f} GiB per rank), build+{a.steps} steps {wall:.1f} s, "
          f"{len(rep.cycles)} cycles, {len(keys)} leaves", flush=True)
r1, rN = res[1], res[a.ranks]
same = (np.array_equal(r1[0].cycles, rN[0].cycles) and np.array_equal(r1[1], rN[1]) and
        np.array_equal(r1[2].view(np.uint64), rN[2].view(np.uint64)))
print("bit-identical:", same)
sys.exit(0 if same else 1)
