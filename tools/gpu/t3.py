"""Repeats the reflective van Albada tolerance case and prints its relative L1
against the exact run (determinism check)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1603_05211_b200 import uniform as U

def run(tol, level=5, steps=8, bc=[2] * 6, lim=0, flux=0):
    s = U.UniformSolver(3, level, scheme=U.SchemeConfig(limiter=lim, flux=flux), bc=bc)
    if tol:
        s.set_numerics(True)
    s.upload(U.case_fill(2, 1, level))
    rep = s.run(steps, cfl=0.4)
    out = s.download()
    s.close()
    return out, rep

for lim, flux, bc in ((0, 0, [2] * 6), (0, 1, [2] * 6), (1, 0, [2] * 6), (0, 0, None), (0, 0, [2, 2, 0, 0, 0, 0]),
                      (0, 0, [0, 0, 2, 2, 0, 0]), (0, 0, [0, 0, 0, 0, 2, 2])):
    a, ra = run(False, lim=lim, flux=flux, bc=bc)
    for i in range(3):
        t, rt = run(True, lim=lim, flux=flux, bc=bc)
        d = np.abs(t - a).sum(0) / np.maximum(np.abs(a).sum(0), 1e-300)
        print(lim, flux, bc, f"{d.max():.3e}", "fb", ra.fallbacks, rt.fallbacks, flush=True)
