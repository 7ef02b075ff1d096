"""Runs `steps` RK2 steps of the 3D uniform solver (for ncu captures).
usage: fv3d_one.py LEVEL STEPS [legacy] [tol]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
level, steps = int(sys.argv[1]), int(sys.argv[2])
os.environ["AF_FV3D_TILE"] = "0" if "legacy" in sys.argv else "1"
from paper_1603_05211_b200 import uniform as U  # noqa: E402

s = U.UniformSolver(3, level, scheme=U.SchemeConfig(limiter=1))
if "tol" in sys.argv:
    s.set_numerics(True)
s.upload(U.case_fill(2, 1, level))
s.run(steps, cfl=0.4, collect=False)
s.sync()
print("ok")
