"""The bench's e2e leg, phase by phase (CUDA events on the solver stream):
device-resident warm-up and timed cycles first, exactly as bench.py runs
them, then build from pinned host memory, K cycles, to_uniform to pinned.
    python tools/e2e_bench_phases.py [--steps 10] [--warmup 3] [--reps 3]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1603_05211_b200 import mr as M  # noqa: E402
from paper_1603_05211_b200 import uniform as U  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
idx, case, dim, level, cfl, seed, _ = bench.WORKLOADS[a.workload]
o, epsl = bench.mr_options(a.workload)
s = M.MRSolver(dim, level, M.MROptions(epsilon=o["eps"], eps_level=epsl,
                                       min_leaf_level=o["min_leaf"], local_time=o["local_time"],
                                       local_time_level_gap=o["gap"]))
st = torch.cuda.Stream()
s.set_stream(st)
init = torch.from_numpy(U.case_fill(case, seed, level)).pin_memory()
out = torch.empty_like(init).pin_memory()
s.build(init.to("cuda"))
s.run(a.warmup, cfl=cfl)
s.profile(True)
s.run(a.steps, cfl=cfl)
s.profile(False)
torch.cuda.synchronize()
for rep in range(a.reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(st)
    s.build(init.numpy())
    ev[1].record(st)
    r = s.run(a.steps, cfl=cfl)
    ev[2].record(st)
    s._check(s._lib.af_mr_to_uniform(s._h, level, C.c_void_p(out.data_ptr())))
    ev[3].record(st)
    ev[3].synchronize()
    print(f"rep {rep}: build {ev[0].elapsed_time(ev[1]):.2f} ms, {len(r.cycles)} cycles "
          f"{ev[1].elapsed_time(ev[2]):.2f} ms, to_uniform {ev[2].elapsed_time(ev[3]):.2f} ms")
