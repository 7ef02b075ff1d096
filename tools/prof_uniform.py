"""Small driver for ncu captures of the uniform stage kernels:
    python tools/prof_uniform.py [--level 9] [--dim 3] [--steps 2]
Uploads the seeded cfg4 (or cfg1) input, runs `steps` CFL steps, syncs."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1603_05211_b200 import uniform as U  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=9)
ap.add_argument("--dim", type=int, default=3)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--limiter", type=int, default=1)
a = ap.parse_args()
kind = 2 if a.dim == 3 else 0
s = U.UniformSolver(a.dim, a.level, scheme=U.SchemeConfig(limiter=a.limiter))
s.upload(U.case_fill(kind, 1, a.level))
rep = s.run(a.steps, cfl=0.4 if a.dim == 3 else 0.5)
print("steps", a.steps, "max_cfl", rep.max_cfl, "launches", s.kernel_launches())
