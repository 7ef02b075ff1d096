"""ncu driver for the MR stage kernel on a dense level (cfg3 generator):
    python tools/prof_mr_stage.py [--level 12]
builds the MRLT tree from the noisy quadrant data and runs one cycle."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_05211_b200 import mr as M  # noqa: E402
from paper_1603_05211_b200 import uniform as U  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=12)
a = ap.parse_args()
s = M.MRSolver(2, a.level, M.MROptions(epsilon=1e-3, local_time=True))
s.build(U.case_fill(1, 1, a.level))
rep = s.run(2, cfl=0.5)
print("updates", rep.updates)
